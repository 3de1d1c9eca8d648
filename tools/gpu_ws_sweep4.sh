# BERT-base resident with the chain-benchmark winners (QKV 64:2, O-proj 32:4) vs the default tiling
cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
FSW_GEMM_WS_FORCE=2304:768:64:2,768:768:16:2,3072:768:64:2,768:3072:64:8 timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
FSW_GEMM_WS_FORCE=2304:768:64:3,768:768:32:4,3072:768:64:2,768:3072:64:8 timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
FSW_GEMM_WS_FORCE=2304:768:64:2,768:768:32:4,3072:768:64:2,768:3072:64:8 timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]"
done
