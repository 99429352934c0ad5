import torch
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b)/reps
x=torch.empty(10*2**30//2, dtype=torch.bfloat16, device='cuda')
y=torch.empty(5*2**30//2, dtype=torch.bfloat16, device='cuda')
z=torch.empty_like(y)
ms=t(lambda: x.fill_(1.0)); print(f"fill 10 GiB: {ms:.3f} ms {10*2**30/ms/1e6:.0f} GB/s")
ms=t(lambda: z.copy_(y)); print(f"copy 5 GiB: {ms:.3f} ms {10*2**30/ms/1e6:.0f} GB/s (r+w)")
ms=t(lambda: y.sum()); print(f"sum 5 GiB: {ms:.3f} ms {5*2**30/ms/1e6:.0f} GB/s (read)")
