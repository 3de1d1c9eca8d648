cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,syslts__t_sectors_aperture_sysmem_op_read.sum \
  -k regex:k_swapz_tma -c 1 -o gpurun_out/prof_swapz_tma python tools/profile_target.py bert-base 0 smz > gpurun_out/ncu_tma.log 2>&1; echo "ncu rc=$?"
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/profile_target.py mlp-small 1 smz > gpurun_out/${t}_mlp-small_smz_tma.log 2>&1; echo "$t rc=$?"
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_target.py bert-tiny 1 smz > gpurun_out/memcheck_bert-tiny_smz_tma.log 2>&1; echo "memcheck bert rc=$?"
