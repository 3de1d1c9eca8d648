# Round-end check: GPU suite, smoke, the exact default bench commands (product and reference arms).
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err; echo "ref rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/final_bench.json')); print({k:d[k] for k in ['value','p99_ms','resident_p50_ms','link_wire_gbs','gpu_launches','clocks']}, d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline']['value'])
r=json.load(open('gpurun_out/final_bench_reference.json')); print(r['impl'], r['value'], r['unit'])"
