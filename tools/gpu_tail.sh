# DMAZT with entropy-coded pieces: body decode CTAs with the 64-CTA tail (BERT-base), and GPT-2-XL at the defaults.
cd $GRAFT_REPO_ROOT
for c in 96 128 160; do FSW_DMAZ_HUFF_CTAS=$c timeout 300 python tools/ws_quick.py bert-base 2>&1 | grep "\]"; done
timeout 600 python tools/ws_quick.py gpt2-xl resnet50 2>&1 | grep "\]"
