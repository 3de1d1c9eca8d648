cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 0 1; do echo "no_cluster_split=$v"; if [ $v = 1 ]; then export FSW_GEMM_NO_CLUSTER_SPLIT=1; fi; timeout 600 python tools/linkcode_bench.py resnet50 bert-base gpt2-xl --reps 5 2>&1 | grep dmaz | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['model'], 'resident', d['resident_ms'], 'cold dmaz', d['p50_ms'])"; done
