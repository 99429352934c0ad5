import torch, time
M=1245184
for (N,K) in ((1536,2048),(2048,768)):
    a=torch.randn(M,K,device='cuda').to(torch.bfloat16); b=torch.randn(K,N,device='cuda').to(torch.bfloat16)
    for _ in range(2): c=a@b
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): c=a@b
    e1.record(); e1.synchronize()
    ms=e0.elapsed_time(e1)/10
    print(f"cuBLAS bf16 M={M} N={N} K={K}: {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TFLOP/s")
