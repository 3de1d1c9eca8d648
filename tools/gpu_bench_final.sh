cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_r2i_reference.json 2> gpurun_out/bench_r2i_reference.err; echo "ref rc=$?"
