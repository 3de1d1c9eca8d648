cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_linkcode.py -x -q 2>&1 | tail -2
timeout 900 python tools/dmaz_streams.py 2>&1 | tee gpurun_out/dmaz_streams.txt
