# Device timelines (tracing build, GEMM phases) of BERT-base with and without the folded LayerNorm.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
for f in 0 1; do FSW_LN_FUSE=$f timeout 300 python tools/timeline.py --model bert-base --phases --out gpurun_out/timeline_bert_lnfuse$f.txt > /dev/null 2>&1; echo "tl $f rc=$?"; done
grep -n 'resident invoke device\|last kernel exit' gpurun_out/timeline_bert_lnfuse*.txt
