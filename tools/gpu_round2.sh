# Round-2 evidence: the final bench line, its ncu launch list, a --set full capture of the dominant kernel
# (the DMAZ decode k_swapz) and of the resident BERT-base GEMMs (tensor-pipe share per GEMM).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2306_03622_b200.build >/dev/null
(time python bench.py --steps 20 --warmup 5) > gpurun_out/bench_r2_final.json 2> gpurun_out/bench_r2_final.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_default_r2.csv \
  python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline --no-extras > gpurun_out/ncu_bench_r2.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_default_r2.csv > gpurun_out/launches_bench_default_r2_summary.txt; head -12 gpurun_out/launches_bench_default_r2_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_swapz -c 1 -o gpurun_out/prof_swapz_dmaz_r2 \
  python tools/profile_target.py bert-base 0 dmaz --dmaz-cold > gpurun_out/ncu_dmaz_r2.log 2>&1; echo "ncu dmaz rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 49 -c 4 -o gpurun_out/prof_gemm_bert_resident_r2 \
  python tools/profile_target.py bert-base 1 sm > gpurun_out/ncu_gemm_r2.log 2>&1; echo "ncu gemm rc=$?"
for f in prof_swapz_dmaz_r2 prof_gemm_bert_resident_r2; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null
done
