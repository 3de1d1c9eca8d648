# Bisection of the k_gemm_ws epilogue (profiles/r02/gemm/ws_sweep.txt section 2). The FSW_WS_DEBUG hook it used
# was temporary and has been removed from gemm_ws.cu; kept as the record of how that measurement was taken.
cd $GRAFT_REPO_ROOT
export FSW_EARLY_TRIGGER=3 FSW_GEMM_WS=1 FSW_GEMM_WS_FORCE=2304:768:64:3,768:768:16:2,3072:768:128:4,768:3072:64:8
for d in 0 1 2 3; do
  echo "== FSW_WS_DEBUG=$d"
  FSW_WS_DEBUG=$d timeout 120 python tools/timeline.py --model bert-base --reps 10 --phases 2>&1 | sed -n "/resident invoke device/,\$p" | grep -v "^ *[0-9]* \(layernorm\|attention\|linear\|embed\) " | head -9
done
