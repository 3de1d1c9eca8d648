cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_invariance.py -x -q 2>&1 | tail -2
for v in split nosplit; do if [ $v = nosplit ]; then export FSW_ATTN_NOSPLIT=1; fi; echo $v; timeout 600 python tools/linkcode_bench.py bert-base gpt2-xl --reps 3 2>&1 | grep -E "dmaz" | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['model'], 'resident', d['resident_ms'], 'cold', d['p50_ms'])"; done
unset FSW_ATTN_NOSPLIT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_attention --csv --log-file gpurun_out/attn_ll.csv python tools/profile_target.py bert-base 1 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/attn_ll.csv
