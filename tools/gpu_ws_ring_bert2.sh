# BERT-base resident: variants around FFN1 64:2:3 + FFN2 64:8:3 (ring slots)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
O=768:768:32:4
for i in 1 2; do
for f in "2304:768:64:2,$O,3072:768:64:2,768:3072:64:8" "2304:768:64:2,$O,3072:768:64:2:3,768:3072:64:8:3" "2304:768:64:2,$O,3072:768:64:2:3,768:3072:64:6:3" "2304:768:64:2,$O,3072:768:64:2:2,768:3072:64:8:3" "2304:768:64:2:3,$O,3072:768:64:2:3,768:3072:64:8:3" "2304:768:64:2,$O,3072:768:64:2:3,768:3072:64:8:4"; do
  echo "FORCE=$f"; FSW_GEMM_WS_FORCE=$f timeout 200 python tools/ws_quick.py bert-base 2>&1 | grep "\]" | sed 's/.*bert-base/bert-base/'; done
done
