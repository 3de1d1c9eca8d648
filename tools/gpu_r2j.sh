# Round-2 final evidence at HEAD (third session, after the FFN rings): bench line and reference arm, the ncu launch
# list of the bench command, --set full captures of the DMAZ decode and of the resident BERT-base GEMMs.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
(time timeout 900 python bench.py) > gpurun_out/bench_r2j.json 2> gpurun_out/bench_r2j.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_r2j.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_r2j_reference.json 2> gpurun_out/bench_r2j_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_default_r2j.csv \
  python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline --no-extras > gpurun_out/ncu_bench_r2j.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_default_r2j.csv > gpurun_out/launches_bench_default_r2j_summary.txt; head -14 gpurun_out/launches_bench_default_r2j_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_swapz -c 1 -o gpurun_out/prof_swapz_dmaz_r2j \
  python tools/profile_target.py bert-base 0 dmaz --dmaz-cold > gpurun_out/ncu_dmaz_v5.log 2>&1; echo "ncu dmaz rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 49 -c 4 -o gpurun_out/prof_gemm_bert_resident_r2j \
  python tools/profile_target.py bert-base 1 sm > gpurun_out/ncu_gemm_r2j.log 2>&1; echo "ncu gemm rc=$?"
for f in prof_swapz_dmaz_r2j prof_gemm_bert_resident_r2j; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null
done
ls -la gpurun_out/*.raw.csv
