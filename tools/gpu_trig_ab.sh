# A/B of the early PDL release in k_gemm_ws (FSW_WS_TRIGGER 0 / 1 / 2): BERT-base and GPT-2-XL resident
cd $GRAFT_REPO_ROOT
for i in 1 2; do for t in 0 1 2; do
  FSW_WS_TRIGGER=$t timeout 300 python tools/ws_quick.py bert-base 2>&1 | tail -1
done; done
for t in 0 1 2; do FSW_WS_TRIGGER=$t timeout 300 python tools/ws_quick.py gpt2-xl 2>&1 | tail -1; done
