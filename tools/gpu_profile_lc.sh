#!/bin/bash
# ncu evidence for the link-coded engines (no-overlap cold invokes: ncu serialises kernels)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
# SMZ decode kernel alone: full set + PCIe / sysmem counters (coded bytes over the link)
timeout 900 ncu --set full --clock-control none --import-source on --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,syslts__t_sectors_aperture_sysmem_op_read.sum \
  -k regex:k_swapz -c 1 -o gpurun_out/prof_swapz_smz python tools/profile_target.py bert-base 0 smz > gpurun_out/ncu_swapz.log 2>&1; echo "ncu smz rc=$?"
# launch list: one no-overlap DMAZ cold invoke + 2 warm invokes (kernel shares of a step)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bert_dmaz.csv python tools/profile_target.py bert-base 2 dmaz > gpurun_out/ncu_ll.log 2>&1; echo "ncu ll rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bert_smz.csv python tools/profile_target.py bert-base 2 smz > gpurun_out/ncu_ll2.log 2>&1; echo "ncu ll2 rc=$?"
# compute-sanitizer on the coded engines (small models)
for e in smz dmaz; do
  timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_target.py bert-tiny 1 $e > gpurun_out/memcheck_bert-tiny_$e.log 2>&1; echo "memcheck $e rc=$?"
  timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_target.py mlp-small 1 $e > gpurun_out/racecheck_mlp-small_$e.log 2>&1; echo "racecheck $e rc=$?"
done
ls -la gpurun_out
