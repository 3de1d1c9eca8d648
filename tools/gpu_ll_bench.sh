cd $GRAFT_REPO_ROOT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_default_r1c.csv python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "rc=$?"
tail -2 gpurun_out/ncu_bench.log | cut -c1-300
python tools/ncu_summary.py gpurun_out/launches_bench_default_r1c.csv
