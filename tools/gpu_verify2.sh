cd $GRAFT_REPO_ROOT
for cfg in "bert.qkv 32 1" "bert.o 16 1" "gpt.qkv 64 1"; do NO_MC=1 timeout 300 ./tools/gemm_bench_phases $cfg 1 2>&1 | grep -A1 -E "^(bert|gpt)" | grep -v "S= 1c"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_invariance.py -x -q 2>&1 | tail -2
timeout 600 python tools/linkcode_bench.py resnet50 bert-base gpt2-xl --reps 5 2>&1 | grep -E "dmaz" | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['model'], 'resident', d['resident_ms'], 'cold', d['p50_ms'])"
