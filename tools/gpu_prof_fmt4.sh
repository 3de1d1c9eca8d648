#!/bin/bash
# ncu + sanitizer evidence for link format v4 (two-tier exponent codes).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2306_03622_b200.build >/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_swapz -c 1 -o gpurun_out/prof_swapz_dmaz_fmt4 python tools/profile_target.py bert-base 0 dmaz --dmaz-cold > gpurun_out/ncu_dmaz_fmt4.log 2>&1; echo "ncu dmaz rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,syslts__t_sectors_aperture_sysmem_op_read.sum \
  -k regex:k_swapz -c 1 -o gpurun_out/prof_swapz_smz_fmt4 python tools/profile_target.py bert-base 0 smz > gpurun_out/ncu_smz_fmt4.log 2>&1; echo "ncu smz rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_default_fmt4.csv python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/ncu_bench_fmt4.log 2>&1; echo "ncu bench rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_default_fmt4.csv > gpurun_out/launches_bench_default_fmt4_summary.txt; cat gpurun_out/launches_bench_default_fmt4_summary.txt | head -12
for e in smz dmaz; do
  timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_target.py bert-tiny 1 $e > gpurun_out/memcheck_bert-tiny_${e}_fmt4.log 2>&1; echo "memcheck $e rc=$?"
  timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_target.py mlp-small 1 $e > gpurun_out/racecheck_mlp-small_${e}_fmt4.log 2>&1; echo "racecheck $e rc=$?"
done
