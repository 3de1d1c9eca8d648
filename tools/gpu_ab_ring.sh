# A/B of BERT-base resident: a previous build checked out and built in the worktree _ab_old vs this tree; then GPT-2-XL
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
 (cd _ab_old && timeout 300 python tools/ws_quick.py bert-base 2>&1 | tail -1 | sed 's/^/OLD /')
 timeout 300 python tools/ws_quick.py bert-base 2>&1 | tail -1 | sed 's/^/NEW /'
done
timeout 300 python tools/ws_quick.py gpt2-xl 2>&1 | tail -1 | sed 's/^/NEW /'
