cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_linkcode.py -x -q -k striped 2>&1 | grep -E "Error|assert|^E " | head -20
timeout 900 python -m pytest tests/test_gpu_linkcode.py tests/test_gpu_edges.py tests/test_gpu_parity.py -q 2>&1 | tail -4
timeout 600 python tools/linkcode_bench.py mlp resnet50 bert-base gpt2-xl --reps 15 2>&1 | tee gpurun_out/linkcode_v2c.txt | grep -E "smz|dmaz|\"dma\"" | cut -c1-230
