# Round-2 (second session) evidence: the default bench line, its ncu launch list, --set full captures of the
# v5 DMAZ decode (k_swapz_tma on the staging buffer) and of the resident BERT-base GEMMs (k_gemm / k_gemm_ws).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
(time timeout 900 python bench.py) > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_r2b.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_default_r2b.csv \
  python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline --no-extras > gpurun_out/ncu_bench_r2b.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_default_r2b.csv > gpurun_out/launches_bench_default_r2b_summary.txt; head -14 gpurun_out/launches_bench_default_r2b_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_swapz -c 1 -o gpurun_out/prof_swapz_dmaz_v5 \
  python tools/profile_target.py bert-base 0 dmaz --dmaz-cold > gpurun_out/ncu_dmaz_v5.log 2>&1; echo "ncu dmaz rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 49 -c 4 -o gpurun_out/prof_gemm_bert_resident_r2b \
  python tools/profile_target.py bert-base 1 sm > gpurun_out/ncu_gemm_r2b.log 2>&1; echo "ncu gemm rc=$?"
for f in prof_swapz_dmaz_v5 prof_gemm_bert_resident_r2b; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null
done
ls -la gpurun_out/*.raw.csv
