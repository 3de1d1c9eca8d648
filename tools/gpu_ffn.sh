# FFN1 / FFN2 co-residency: k_gemm_ws tilings with 12-CTA (non-portable) split-K clusters, resident p50 (BERT-base).
cd $GRAFT_REPO_ROOT
timeout 300 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
for f in "768:768:16:2,768:3072:64:12" "768:768:16:2,3072:768:128:4,768:3072:64:12" "768:768:16:2,3072:768:128:4,768:3072:64:8" \
         "768:768:16:2,3072:768:128:6,768:3072:64:12" "768:768:16:2,768:3072:64:16"; do
  FSW_GEMM_WS=2 FSW_GEMM_WS_FORCE=$f timeout 300 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
done
FSW_PLAN_VERBOSE=1 FSW_GEMM_WS=2 FSW_GEMM_WS_FORCE=768:768:16:2,3072:768:128:4,768:3072:64:12 timeout 300 python tools/ws_quick.py bert-tiny 2>&1 | grep "plan\]" | head -0
