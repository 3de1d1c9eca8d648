# Entropy-coded pieces (format v5): cold latency vs the per-block form (FSW_LINK_HUFF=0), DMAZ / SMZ decode CTAs swept.
cd $GRAFT_REPO_ROOT
timeout 300 python tools/ws_quick.py bert-tiny 2>&1 | grep "\]"
FSW_LINK_HUFF=0 timeout 300 python tools/ws_quick.py resnet50 bert-base 2>&1 | grep "\]"
for c in 96 128 192 256; do FSW_DMAZ_HUFF_CTAS=$c timeout 300 python tools/ws_quick.py bert-base 2>&1 | grep "\]"; done
for c in 32 48 64 80; do FSW_SMZ_HUFF_CTAS=$c timeout 300 python tools/ws_quick.py mlp resnet50 2>&1 | grep "\]"; done
