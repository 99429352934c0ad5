"""HBM-bound glue kernels of one cached layer at the R=256 C3 size: permute
(plan + row copy), combine, RMSNorm.  Prints time and algorithmic GB/s.

    python tools/bench_glue.py [n_rows] [H] [E] [k]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05899_b200 import _lib, kernels

N = int(sys.argv[1]) if len(sys.argv) > 1 else 150000
H = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
E = int(sys.argv[3]) if len(sys.argv) > 3 else 128
k = int(sys.argv[4]) if len(sys.argv) > 4 else 8
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
ids = torch.rand(N, E, device=dev, generator=g).topk(k, dim=1).indices.to(torch.int32).contiguous()
gates = torch.rand(N, k, device=dev, generator=g).contiguous()
x = torch.randn(N, H, device=dev).to(torch.bfloat16)
xp = torch.empty(N * k, H, device=dev, dtype=torch.bfloat16)
y = torch.randn(N * k, H, device=dev).to(torch.bfloat16)
out = torch.empty_like(x)
xn = torch.empty_like(x)
bufs = (torch.empty(E + 1, dtype=torch.int32, device=dev), torch.empty(N * k, dtype=torch.int32, device=dev),
        torch.empty(N * k, dtype=torch.int32, device=dev))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
wr = (torch.randn(E, H, device=dev) / H ** 0.5).to(torch.bfloat16)
cnt = torch.zeros(E, dtype=torch.int32, device=dev)
cnt2 = torch.zeros(E, dtype=torch.int32, device=dev)
wr2 = (torch.randn(2, E, H, device=dev) / H ** 0.5).to(torch.bfloat16)


def cuda_ms(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t = 0.0
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        t += a.elapsed_time(b)
    return t / reps


row = H * 2
M = N * k
off, src, pos, _ = kernels.permute(ids, x, E, bufs=bufs, out=xp)
cases = {
    "permute (plan+copy)": (lambda: kernels.permute(ids, x, E, bufs=bufs, out=xp), N * row + M * row),
    "permute_plan": (lambda: kernels.permute_plan(ids, E, bufs=bufs), M * 4 * 3),
    "permute_rows": (lambda: kernels.permute_rows(x, src, M, out=xp), 2 * M * row),
    "combine": (lambda: kernels.combine(y, pos.view(N, k), gates, x, out=out), M * row + 2 * N * row),
    "rmsnorm": (lambda: kernels.rmsnorm(out, out=xn), 2 * N * row),
    "combine_norm": (lambda: _lib.check(_lib.lib().vmm_combine_norm(y.data_ptr(), pos.data_ptr(), gates.data_ptr(),
                                                                     x.data_ptr(), N, k, H, None, 0, 1e-6,
                                                                     out.data_ptr(), xn.data_ptr(), 0)),
                     M * row + 3 * N * row),
    "route": (lambda: kernels.route_topk(xn, wr, k, counts=cnt), N * row + E * row + N * k * 8),
    "route_lookahead": (lambda: kernels.route_lookahead(xn, wr2, 0, k, cnt, cnt2), N * row + 2 * E * row + N * k * 8),
}
only = os.environ.get("GLUE_ONLY")
for name, (fn, bytes_) in cases.items():
    if only and only not in name:
        continue
    ms = cuda_ms(fn)
    print(f"{name:22s} {ms:8.3f} ms  {bytes_ / ms / 1e6:8.0f} GB/s algorithmic ({bytes_ / 1e9:.2f} GB)")
