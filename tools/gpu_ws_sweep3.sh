cd $GRAFT_REPO_ROOT
FSW_PLAN_VERBOSE=1 FSW_GEMM_WS=2 timeout 300 python tools/ws_quick.py bert-base gpt2-2L 2>&1 | grep "plan\]" | sort -u -t: -k1,1 | head -12
for f in 2304:768:64:3,3072:768:128:4,768:768:16:2,768:3072:64:8 2304:768:64:3,3072:768:64:3,768:768:16:2,768:3072:64:8; do
  FSW_GEMM_WS=2 FSW_GEMM_WS_FORCE=$f timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
done
for f in 4800:1600:64:4 4800:1600:128:6 6400:1600:128:4 1600:6400:64:8; do
  FSW_GEMM_WS=2 FSW_GEMM_WS_FORCE=$f,1600:1600:64:5 timeout 300 python tools/ws_quick.py gpt2-xl 2>&1 | grep "\]"
done
