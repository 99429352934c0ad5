import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2605_05899_b200 import kernels
N, H, I, E, k = 5000, 2048, 768, 128, 8
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
arena = (torch.randn(E, 3 * I * H, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
ids = torch.topk(torch.randn(N, E, device="cuda", generator=g), k, dim=1).indices.int()
off, src, pos = kernels.permute_plan(ids, E)
xp = kernels.permute_rows(x, src, N * k)
slot = torch.arange(E, dtype=torch.int32, device="cuda")
h1a, ya = kernels.grouped_swiglu(xp, off, arena, slot, I, fused=False)
h1b, yb = kernels.grouped_swiglu(N * k, off, arena, slot, I, x_rows=x, src_row=src)
torch.cuda.synchronize()
print("equal h1", torch.equal(h1a, h1b), "y", torch.equal(ya, yb), (ya.float()-yb.float()).abs().max().item())
