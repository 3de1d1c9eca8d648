cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do timeout 200 python tools/ws_quick.py bert-base gpt2-2L 2>&1 | grep "\]" | sed 's/.*\] //'; done
