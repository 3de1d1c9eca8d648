# DMAZ decode without head-of-line blocking at copy-group boundaries: tests, ResNet-50 engine probe, timelines, bench.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_litmus.py tests/test_gpu_linkcode.py tests/test_gpu_swap.py -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/resnet_sweep.py resnet50 2>&1 | grep -E 'smz|ctas=  0' > gpurun_out/resnet_sweep_hol.txt; echo "sweep rc=$?"
timeout 300 python tools/timeline.py --model resnet50 --engine 4 --out gpurun_out/timeline_resnet50_dmaz_hol.txt > /dev/null 2>&1; echo "tl rc=$?"
timeout 300 python tools/timeline.py --model bert-base --engine 0 --out gpurun_out/timeline_bert_dmazt_hol.txt > /dev/null 2>&1; echo "tl bert rc=$?"
timeout 600 python bench.py --no-variants --no-extras --no-cpu-baseline > gpurun_out/bench_hol.json 2> gpurun_out/bench_hol.err; echo "bench rc=$?"
cat gpurun_out/resnet_sweep_hol.txt
python -c "
import json
d=json.load(open('gpurun_out/bench_hol.json')); print({k:d[k] for k in ['value','p99_ms','resident_p50_ms','link_wire_gbs','compute_tail_p50_ms']})"
