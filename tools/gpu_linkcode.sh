cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_linkcode.py tests/test_gpu_swap.py -x -q 2>&1 | tail -3
for r in 0 1 2 4; do echo "ramp $r"; FSW_DMA_RAMP=$r timeout 600 python tools/linkcode_bench.py mlp resnet50 bert-base --reps 15 2>&1 | tee gpurun_out/linkcode_ramp$r.txt | cut -c1-200; done
