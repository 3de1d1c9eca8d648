set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python tools/linkcode_bench.py mlp resnet50 bert-base --reps 15 2>&1 | tee gpurun_out/linkcode_v2.txt | cut -c1-220
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json; cut -c1-1500 gpurun_out/bench_default.json
