# k_gemm_ws ring mode (ws_stages) on GPT-2-XL's wide linears, in the isolated 12-GEMM chain vs cuBLAS
cd $GRAFT_REPO_ROOT
timeout 600 python tools/gemm_chain_vs_cublas.py gpt-qkv gpt-fc gpt-proj2 2>&1 | tail -3
for f in 4800:1600:128:3:3 4800:1600:128:3:4 4800:1600:128:2:4 4800:1600:64:1:4 4800:1600:64:1:6; do
  FSW_GEMM_WS_FORCE=$f timeout 300 python tools/gemm_chain_vs_cublas.py gpt-qkv 2>&1 | tail -1; done
for f in 6400:1600:128:2:3 6400:1600:64:1:4 6400:1600:64:1:6; do
  FSW_GEMM_WS_FORCE=$f timeout 300 python tools/gemm_chain_vs_cublas.py gpt-fc 2>&1 | tail -1; done
for f in 1600:6400:128:8:3 1600:6400:128:8:2 1600:6400:64:5:4 1600:6400:64:4:4; do
  FSW_GEMM_WS_FORCE=$f timeout 300 python tools/gemm_chain_vs_cublas.py gpt-proj2 2>&1 | tail -1; done
