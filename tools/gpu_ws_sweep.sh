# Per-shape in-graph sweep of k_gemm_ws tilings on resident BERT-base (the listed shape runs k_gemm_ws with the
# given tt:splits, every other linear k_gemm), early PDL triggers on.
cd $GRAFT_REPO_ROOT
export FSW_EARLY_TRIGGER=3
timeout 100 python tools/ws_quick.py bert-base 2>&1 | tail -1
for f in ${CFGS:-2304:768:16:1 2304:768:32:2 2304:768:64:3 2304:768:128:8 \
         768:768:16:1 768:768:16:2 768:768:16:3 768:768:32:4 768:768:32:6 \
         3072:768:32:2 3072:768:64:3 3072:768:128:4 3072:768:128:6 \
         768:3072:32:6 768:3072:64:8 768:3072:32:8} ; do
  FSW_GEMM_WS=1 FSW_GEMM_WS_FORCE=$f timeout 100 python tools/ws_quick.py bert-base 2>&1 | tail -1
done
FSW_GEMM_WS=1 timeout 100 python tools/ws_quick.py bert-base 2>&1 | tail -1
