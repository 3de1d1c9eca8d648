cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_linkcode.py -x -q 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_swapz -c 1 -o gpurun_out/prof_swapz_dmaz python tools/profile_target.py bert-base 0 dmaz --dmaz-cold > gpurun_out/ncu_dmaz.log 2>&1; echo "ncu dmaz rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_default_r1d.csv python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu bench rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_default_r1d.csv
