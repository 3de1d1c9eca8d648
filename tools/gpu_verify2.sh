cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_linkcode.py -x -q 2>&1 | tail -3
for c in 16 32; do echo "ctas=$c"; timeout 600 python tools/linkcode_bench.py mlp resnet50 bert-base --reps 15 --ctas $c 2>&1 | tee gpurun_out/linkcode_tma_c$c.txt | grep -E "smz|dmaz" | cut -c1-200; done
