#!/bin/bash
# ncu captures of the current kernels + compute-sanitizer runs (no-overlap mode: tools serialise kernels)
mkdir -p gpurun_out
# SM swap kernel alone (one no-overlap cold invoke, SM engine forced), full set + PCIe counters
timeout 600 ncu --set full --clock-control none --import-source on --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,syslts__t_sectors_aperture_sysmem_op_read.sum \
  -k regex:k_swap -c 1 -o gpurun_out/prof_swap_sm python tools/profile_target.py bert-base 0 sm > gpurun_out/ncu_swap.log 2>&1
# the top GEMMs of a warm BERT-base invoke
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 6 -c 4 -o gpurun_out/prof_gemm python tools/profile_target.py bert-base 1 > gpurun_out/ncu_gemm.log 2>&1
# attention + layernorm
timeout 600 ncu --set full --clock-control none -k regex:"k_attention|k_layernorm" -s 4 -c 2 -o gpurun_out/prof_attn_ln python tools/profile_target.py bert-base 1 > gpurun_out/ncu_attn.log 2>&1
# compute-sanitizer: memcheck and racecheck on small models (no-overlap cold + warm invokes)
for m in mlp-small bert-tiny resnet-tiny gpt2-tiny; do
  timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_target.py $m 1 > gpurun_out/memcheck_$m.log 2>&1; echo "memcheck $m rc=$?"
done
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_target.py bert-tiny 1 > gpurun_out/racecheck_bert-tiny.log 2>&1; echo "racecheck bert-tiny rc=$?"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/profile_target.py bert-tiny 1 > gpurun_out/synccheck_bert-tiny.log 2>&1; echo "synccheck bert-tiny rc=$?"
