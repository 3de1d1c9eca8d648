# GPT-2: k_gemm_ws on every width (FSW_GEMM_WS=2) vs the default (narrow linears only), resident p50.
cd $GRAFT_REPO_ROOT
for v in "FSW_X=0" "FSW_GEMM_WS=2"; do env $v timeout 600 python tools/ws_quick.py gpt2-2L gpt2-xl 2>&1 | grep "\]"; done
FSW_PLAN_VERBOSE=1 FSW_GEMM_WS=2 timeout 300 python tools/ws_quick.py gpt2-2L 2>&1 | grep "plan\]" | head -5
