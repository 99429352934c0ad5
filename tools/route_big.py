"""Router at a prefill batch (default 311 296 rows = R=256 retained tokens): route and
route + lookahead, a few launches each (for ncu captures).

    python tools/route_big.py [rows] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05899_b200 import kernels

N = int(sys.argv[1]) if len(sys.argv) > 1 else 311296
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L, H, E, k = 48, 2048, 128, 8
g = torch.Generator(device="cuda").manual_seed(0)
router = (torch.randn(L, E, H, device="cuda", generator=g) / 45).to(torch.bfloat16)
x = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
counts = torch.zeros(E, dtype=torch.int32, device="cuda")
lac = torch.zeros(E, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for la in (0, 1):
    ts = []
    for i in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if la:
            kernels.route_lookahead(x, router, 3, k, counts, lac)
        else:
            kernels.route_topk(x, router[3], k, counts=counts)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"N={N} lookahead={la}: median {sorted(ts)[len(ts) // 2]:.1f} us -> "
          f"{N * H * 2 / (sorted(ts)[len(ts) // 2] * 1e-6) / 1e12:.2f} TB/s of rows")
