cd $GRAFT_REPO_ROOT
for cfg in "bert.qkv 128 6" "bert.qkv 64 3" "gpt.qkv 64 5"; do NO_MC=1 timeout 300 ./tools/gemm_bench_phases $cfg 1 2>&1 | grep -A1 -E "^(bert|gpt)" ; done > gpurun_out/gemm_phases2.txt 2>&1; cat gpurun_out/gemm_phases2.txt
NO_MC=1 timeout 900 ./tools/gemm_bench 2>&1 > gpurun_out/gemm_sweep_cz2.txt; grep BEST gpurun_out/gemm_sweep_cz2.txt
