# ncu --set full of our GEMM and cuBLAS's on BERT QKV (M=128, K=768, N=2304), for the next GEMM design.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2306_03622_b200.build >/dev/null
timeout 900 python -m pytest tests/test_gpu_linkcode.py -x -q 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 4 -c 1 -o gpurun_out/prof_cublas_qkv python tools/cublas_one.py 128 768 2304 > gpurun_out/ncu_cublas.log 2>&1; echo "ncu cublas rc=$?"
NO_MC=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 20 -c 1 -o gpurun_out/prof_ours_qkv ./tools/gemm_bench bert.qkv 32 1 > gpurun_out/ncu_ours.log 2>&1; echo "ncu ours rc=$?"
