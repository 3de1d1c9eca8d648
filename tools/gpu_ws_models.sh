# Resident / cold p50 per model: round-2 defaults (k_gemm_ws on the narrow linears, early PDL triggers) vs the
# previous defaults (FSW_GEMM_WS=0 FSW_EARLY_TRIGGER=0).
cd $GRAFT_REPO_ROOT
M="bert-tiny gpt2-tiny mlp resnet50 bert-base gpt2-xl"
timeout 600 python tools/ws_quick.py $M 2>&1 | grep "\]"
FSW_GEMM_WS=0 FSW_EARLY_TRIGGER=0 timeout 600 python tools/ws_quick.py $M 2>&1 | grep "\]"
FSW_PLAN_VERBOSE=1 timeout 300 python tools/ws_quick.py gpt2-xl 2>&1 | grep "plan\]" | head -5
