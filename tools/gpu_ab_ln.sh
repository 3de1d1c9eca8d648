# Same-box A/B: resident / cold BERT-base with the tree before the folded-LayerNorm code (_ab_old, prebuilt) and HEAD.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
for i in 1 2 3; do
  (cd _ab_old && timeout 300 python tools/ln_fuse_probe.py bert-base 2>&1 | tail -1 | sed 's/^/OLD /')
  timeout 300 python tools/ln_fuse_probe.py bert-base 2>&1 | tail -1 | sed 's/^/NEW /'
done
timeout 900 python -m pytest tests/test_gpu_ln_fuse.py tests/test_gpu_gemm_ws.py -m gpu -q -x 2>&1 | tail -2
