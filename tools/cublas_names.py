import torch
for (M,K,N) in [(128,768,2304),(128,1600,4800),(128,3072,768)]:
    a=torch.randn(M,K,device="cuda",dtype=torch.bfloat16); w=torch.randn(N,K,device="cuda",dtype=torch.bfloat16); b=torch.randn(N,device="cuda",dtype=torch.bfloat16)
    for _ in range(3): torch.nn.functional.linear(a,w,b)
    torch.cuda.synchronize()
