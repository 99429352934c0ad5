"""Time the non-FFN kernels of a cached C3 layer at batch size R (all inputs resident):
combine_norm, combine, rmsnorm, fused permute, router (+lookahead)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05899_b200 import _lib, kernels

R = int(sys.argv[1]) if len(sys.argv) > 1 else 256
N, H, E, k, L = 1216 * R, 2048, 128, 8, 48
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
y = torch.randn(N * k, H, device="cuda", generator=g).to(torch.bfloat16)
ids = torch.topk(torch.randn(N, E, device="cuda", generator=g), k, dim=1).indices.int()
pos = torch.randperm(N * k, device="cuda", generator=g).int().reshape(N, k)
gates = torch.softmax(torch.randn(N, k, device="cuda", generator=g), 1)
router = (torch.randn(L, E, H, device="cuda", generator=g) / 45).to(torch.bfloat16)
out, xn = torch.empty_like(x), torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
Lb = _lib.lib()
sp = lambda: torch.cuda.current_stream().cuda_stream


def t(name, fn, nbytes):
    ts = []
    for i in range(4):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    ms = sum(ts) / len(ts)
    print(f"{name:28s} {ms:8.3f} ms  {nbytes / ms / 1e6:7.0f} GB/s (algorithmic)", flush=True)


rb = N * H * 2
t("combine_norm", lambda: _lib.check(Lb.vmm_combine_norm(y.data_ptr(), pos.data_ptr(), gates.data_ptr(), x.data_ptr(),
                                                          N, k, H, None, 0, 1e-6, out.data_ptr(), xn.data_ptr(), sp())),
  k * rb + 3 * rb)
t("combine", lambda: kernels.combine(y, pos, gates, x, out=out), k * rb + 2 * rb)
t("rmsnorm", lambda: kernels.rmsnorm(x, out=out), 2 * rb)
xp = torch.empty(N * k, H, dtype=torch.bfloat16, device="cuda")
t("permute (plan+copy)", lambda: kernels.permute(ids, x, E, out=xp), rb + k * rb + N * k * 12)
cnt = torch.zeros(E, dtype=torch.int32, device="cuda")
la = torch.zeros(E, dtype=torch.int32, device="cuda")
t("route+lookahead (2 gates)", lambda: kernels.route_lookahead(x, router, 10, k, cnt, la), rb + N * k * 8)
t("route (1 gate)", lambda: kernels.route_topk(x, router[3], k, counts=cnt), rb + N * k * 8)
