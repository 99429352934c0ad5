"""Phase timeline of the split-K router (CTA 0) in the VMM_PRUNE_PROF dev build
(VMM_BUILD_VARIANT=prof python -m paper_2605_05899_b200.build).

    python tools/route_prof.py [rows=1216] [lookahead=1]
"""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("VMM_LIB", os.path.join(HERE, "paper_2605_05899_b200", "libvismmoe_prof.so"))
sys.path.insert(0, HERE)
import numpy as np
import torch

from paper_2605_05899_b200 import _lib, kernels

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1216
la = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L, H, E, k = 48, 2048, 128, 8
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
router = (torch.randn(L, E, H, device="cuda", generator=g) / 45).to(torch.bfloat16)
counts = torch.zeros(E, dtype=torch.int32, device="cuda")
lac = torch.zeros(E, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
Lb = _lib.lib()
names = ["mainloop", "spill", "cluster barrier", "reduce + top-k", "final barrier"]
acc = np.zeros(5)
tot = []
n = 20
for i in range(n + 3):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    if la:
        kernels.route_lookahead(x, router, 3, k, counts, lac)
    else:
        kernels.route_topk(x, router[3], k, counts=counts)
    b.record()
    torch.cuda.synchronize()
    ts = (ctypes.c_ulonglong * 8)()
    _lib.check(Lb.vmm_route_prof_read(ts))
    if i >= 3:
        acc += np.diff(np.array(ts[:6], dtype=np.float64))
        tot.append(a.elapsed_time(b))
for nm, v in zip(names, acc / n):
    print(f"{nm:16s} {v / 1e3:8.2f} us")
print(f"kernel span (CTA 0) {acc.sum() / n / 1e3:.2f} us; event-timed launch {np.median(tot) * 1e3:.2f} us")
