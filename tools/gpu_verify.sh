set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json; cat gpurun_out/bench_default.json
timeout 600 python bench.py --model resnet50 --steps 30 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_resnet.json
timeout 900 python bench.py --model gpt2-xl --steps 10 --no-cpu-baseline --no-variants 2>&1 | tail -1 > gpurun_out/bench_gpt2xl.json
timeout 300 python bench.py --impl reference --steps 3 2>&1 | tail -1 > gpurun_out/bench_reference.json
