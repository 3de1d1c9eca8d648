# k_gemm_ws tilings for QKV / O-proj in the isolated 12-GEMM chain vs cuBLAS (tools/gemm_chain_vs_cublas.py)
cd $GRAFT_REPO_ROOT
for f in 2304:768:64:3 2304:768:32:2 2304:768:64:4 2304:768:128:6 2304:768:128:4 2304:768:64:2; do
  FSW_GEMM_WS_FORCE=$f timeout 300 python tools/gemm_chain_vs_cublas.py qkv 2>&1 | tail -1; done
for f in 768:768:16:2 768:768:32:4 768:768:16:3 768:768:32:6 768:768:64:6 768:768:16:4 768:768:32:3; do
  FSW_GEMM_WS_FORCE=$f timeout 300 python tools/gemm_chain_vs_cublas.py o-proj 2>&1 | tail -1; done
FSW_GEMM_WS=0 timeout 300 python tools/gemm_chain_vs_cublas.py 2>&1 | tail -4
