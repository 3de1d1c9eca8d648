# BERT-base resident: FFN1 / FFN2 on the k_gemm_ws ring (smaller CTAs, so FFN2's CTAs can be resident beside FFN1's)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
B=2304:768:64:2,768:768:32:4
for i in 1 2; do
for f in "$B,3072:768:64:2,768:3072:64:8" "$B,3072:768:64:2:3,768:3072:64:8:3" "$B,3072:768:64:2:2,768:3072:64:8:2" "$B,3072:768:64:2,768:3072:64:8:3" "$B,3072:768:64:2:3,768:3072:64:8" "$B,3072:768:64:3:2,768:3072:64:8:2"; do
  echo "FORCE=$f"; FSW_GEMM_WS_FORCE=$f timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]" ; done
done
