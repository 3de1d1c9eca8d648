"""One cuBLAS bf16 linear of a batch-1 shape (for an ncu capture next to tools/gemm_bench)."""
import sys
import torch
M, K, N = (int(v) for v in sys.argv[1:4])
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(N, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    torch.nn.functional.linear(a, w, b)
torch.cuda.synchronize()
