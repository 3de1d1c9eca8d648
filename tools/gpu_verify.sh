set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json
timeout 600 python bench.py --model resnet50 --steps 30 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_resnet.json
timeout 600 python bench.py --model mlp --steps 50 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_mlp.json
timeout 900 python bench.py --model gpt2-xl --steps 10 --no-cpu-baseline --no-variants 2>&1 | tail -1 > gpurun_out/bench_gpt2xl.json
timeout 300 python bench.py --impl reference --steps 3 2>&1 | tail -1 > gpurun_out/bench_reference.json
for f in bench_default bench_resnet bench_mlp bench_gpt2xl; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read());print('$f', {k:d.get(k) for k in ['value','p99_ms','resident_p50_ms','host_to_hbm_gbs','link_wire_gbs','compute_tail_p50_ms','clocks']}, d['config'].get('swap_engine'), {k:v.get('p50_ms') for k,v in d.get('engines',{}).items()}, d['e2e'])"; done
