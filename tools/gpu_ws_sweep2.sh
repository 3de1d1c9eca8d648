# After the push reduction: does k_gemm_ws now win the wide linears too?  resident p50, BERT-base (and GPT-2-XL)
cd $GRAFT_REPO_ROOT
timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
for f in 2304:768:32:2 2304:768:64:3 2304:768:64:4 2304:768:128:8 3072:768:64:3 3072:768:128:4 3072:768:128:6 3072:768:32:2; do
  FSW_GEMM_WS=2 FSW_GEMM_WS_FORCE=$f,768:768:16:2,768:3072:64:8 timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
done
FSW_GEMM_WS=2 timeout 300 python tools/ws_quick.py bert-base gpt2-xl 2>&1 | grep "\]"
