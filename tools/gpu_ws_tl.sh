# A/B of the weight-stationary GEMM (k_gemm_ws), early PDL triggers and L2 prefetch on resident BERT-base:
# device timeline phases of the GEMMs (tracing build) and resident / cold p50 (default build).
cd $GRAFT_REPO_ROOT
FSW_PLAN_VERBOSE=1 FSW_GEMM_WS=1 timeout 60 python tools/ws_quick.py bert-tiny 2>&1 | grep "plan\]" | head -0
FSW_PLAN_VERBOSE=1 FSW_GEMM_WS=1 timeout 100 python tools/ws_quick.py bert-base 2>&1 | grep "plan\]" | head -6
for v in "FSW_X=0" "FSW_EARLY_TRIGGER=3" "FSW_GEMM_WS=1 FSW_EARLY_TRIGGER=3" "FSW_GEMM_WS=1 FSW_EARLY_TRIGGER=3 FSW_GEMM_PF=1" ${EXTRA}; do
  echo "== $v"
  env $v timeout 120 python tools/timeline.py --model bert-base --reps 10 --phases 2>&1 | sed -n "/resident invoke device/,\$p" | grep -v "^ *[0-9]* \(layernorm\|attention\|linear\|embed\) " | head -12
  env $v timeout 120 python tools/ws_quick.py bert-base 2>&1 | tail -1
done
