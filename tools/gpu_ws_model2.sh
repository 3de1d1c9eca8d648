cd $GRAFT_REPO_ROOT
FSW_PLAN_VERBOSE=1 timeout 300 python tools/ws_quick.py bert-base gpt2-2L 2>&1 | grep "plan\] layer \(2\|4\|6\|7\) " | sort -u | head -12
for i in 1 2; do timeout 300 python tools/ws_quick.py bert-base gpt2-xl resnet50 mlp 2>&1 | grep "\]"; done
