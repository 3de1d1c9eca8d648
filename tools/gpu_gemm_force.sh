# In-graph tiling sweep of k_gemm on the linears k_gemm_ws does not take (BERT QKV / FFN1), current defaults.
cd $GRAFT_REPO_ROOT
for f in "" "16:2:1" "32:2:1" "16:3:1" "32:3:1" "16:4:1" "32:4:1" "64:2:1" "64:3:1"; do
  FSW_GEMM_FORCE=$f timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]" | sed "s/^/[$f] /"
done
