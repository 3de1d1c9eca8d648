# PDL launch mask (attention launched with programmatic dependent launch or not) x early triggers, resident p50.
cd $GRAFT_REPO_ROOT
for v in "FSW_X=0" "FSW_PDL_MASK=127" "FSW_PDL_MASK=127 FSW_EARLY_TRIGGER=1" "FSW_EARLY_TRIGGER=1" "FSW_EARLY_TRIGGER=2"; do
  env $v timeout 300 python tools/ws_quick.py bert-base gpt2-tiny 2>&1 | grep "\]"
done
