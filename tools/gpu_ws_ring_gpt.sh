# GPT-2-XL resident: FC / MLP projection small enough to co-reside (TT = 64 rings) vs the default rings
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
FSW_PLAN_VERBOSE=1 timeout 300 python tools/ws_quick.py gpt2-xl 2>&1 | grep -E 'fsw plan\] layer (2|4|6|7) ' | head -4
for i in 1 2; do
for f in "4800:1600:128:3:3,1600:1600:64:4,6400:1600:128:2:3,1600:6400:128:8:3" "4800:1600:128:3:3,1600:1600:64:4,6400:1600:64:1:3,1600:6400:64:5:3"; do
  echo "FORCE=$f"; FSW_GEMM_WS_FORCE=$f timeout 300 python tools/ws_quick.py gpt2-xl 2>&1 | grep "\]" | sed 's/.*gpt2-xl/gpt2-xl/'; done
done
