cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_ln_fuse.py -m gpu -q -x 2>&1 | grep -v '^  ' | tail -40

