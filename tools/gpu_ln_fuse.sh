# Folded LayerNorm (FSW_LN_FUSE=1) vs the LN kernels: parity, resident / cold latency, then the GPU suites that
# exercise the transformer plans with the fold on.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
FSW_LN_FUSE=1 FSW_PLAN_VERBOSE=1 timeout 300 python tools/ln_fuse_probe.py bert-tiny 2>&1 | grep -E 'LayerNorm|rel err' | head -8
for f in 0 1; do FSW_LN_FUSE=$f timeout 600 python tools/ln_fuse_probe.py bert-tiny bert-base gpt2-tiny 2>&1 | tail -3; done
FSW_LN_FUSE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm_ws.py tests/test_gpu_edges.py -m gpu -q -x 2>&1 | tail -4
