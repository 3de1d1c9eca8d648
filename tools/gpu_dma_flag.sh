# Copy-group publication A/B (FSW_DMA_FLAG 0 fenced write-value, 1 4-byte D2D copy, 3 4-byte H2D copy, 2 unfenced
# write-value = timing reference only), then the readiness litmus and bit-exact swap tests with modes 1 and 3.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
for i in 1 2; do for m in 0 1 3 2; do FSW_DMA_FLAG=$m timeout 300 python tools/dma_flag_probe.py 2>&1 | grep FLAG; done; done
for m in 1 3; do FSW_DMA_FLAG=$m timeout 1200 python -m pytest tests/test_gpu_litmus.py tests/test_gpu_swap.py tests/test_gpu_linkcode.py -m gpu -q -x 2>&1 | tail -2; done
