# BERT-base resident: QKV tilings beside the FFN rings (FFN1 64:2:3, FFN2 64:8:3)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
F=768:768:32:4,3072:768:64:2:3,768:3072:64:8:3
for i in 1 2; do
for q in 2304:768:64:2 2304:768:64:2:2 2304:768:64:3:2 2304:768:64:3:3 2304:768:32:2:3 2304:768:128:4:2; do
  echo "QKV=$q"; FSW_GEMM_WS_FORCE=$q,$F timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]" | sed 's/.*bert-base/bert-base/'; done
done
