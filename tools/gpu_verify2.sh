cd $GRAFT_REPO_ROOT
python tools/cluster_cap.py
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q 2>&1 | tail -2
timeout 600 python tools/linkcode_bench.py resnet50 bert-base gpt2-xl --reps 5 2>&1 | grep -E "dmaz|smz" | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['model'], d['engine'], 'resident', d['resident_ms'], 'cold', d['p50_ms'])"
