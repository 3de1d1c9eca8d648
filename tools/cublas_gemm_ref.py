"""cuBLAS (torch.matmul, bf16, fp32 accumulate) on the batch-1 GEMM shapes of the paper's models,
timed as back-to-back calls captured in a CUDA graph (no launch overhead), for comparison with
tools/gemm_bench.cu (our tcgen05 kernel, back-to-back PDL launches)."""
import torch
shapes = [("bert.qkv", 128, 768, 2304), ("bert.o", 128, 768, 768), ("bert.ffn1", 128, 768, 3072),
          ("bert.ffn2", 128, 3072, 768), ("gpt.qkv", 128, 1600, 4800), ("gpt.fc", 128, 1600, 6400),
          ("gpt.proj2", 128, 6400, 1600), ("rn.s3.1x1", 196, 1024, 256), ("rn.s4.1x1", 49, 2048, 512),
          ("rn.s4.3x3", 49, 4608, 512)]
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
for name, M, K, N in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, device="cuda", dtype=torch.bfloat16)
    outs = []
    for _ in range(3):
        torch.nn.functional.linear(a, w, b)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    reps = 50
    with torch.cuda.graph(g):
        for _ in range(reps):
            torch.nn.functional.linear(a, w, b)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    print(f"{name:12s} M={M:4d} K={K:5d} N={N:5d}  cuBLAS {us:7.2f} us  (W {2*N*K/us/1e3:6.0f} GB/s)", flush=True)
