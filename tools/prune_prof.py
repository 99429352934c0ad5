"""Phase timeline of one prune launch (CTA 0): the VMM_PRUNE_PROF dev build
(VMM_BUILD_VARIANT=prof python -m paper_2605_05899_b200.build).

    python tools/prune_prof.py [requests=1]

Phases: 0 reset/min-max, 1 s_norm, 2 core select, 3 target OR, 4 delta/score,
5 extras select, 6 retained compaction, 7 final cluster barrier.
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

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nv, nt, P, k, E = 2304, 64, 8, 8, 128
T1 = nv + nt
T = T1 * R
rng = np.random.default_rng(R)
dev = torch.device("cuda")
sal = torch.from_numpy(rng.gamma(2.0, 1.0, size=T)).to(dev)
mod = torch.from_numpy(np.tile(np.r_[np.zeros(nv, np.uint8), np.ones(nt, np.uint8)], R)).to(dev)
routes = torch.randint(0, E, (P, T, k), dtype=torch.int32, device=dev)
offs = torch.tensor([r * T1 for r in range(R + 1)], dtype=torch.int32, device=dev)
L = _lib.lib()
names = ["reset/min-max", "s_norm", "core select", "target OR", "delta/score", "extras select", "compaction",
         "final barrier"]
acc = np.zeros(8)
n = 20
for i in range(n + 3):
    kernels.prune(sal, mod, routes, offs, None, None, E, 2.0, alpha=0.1, beta=0.5)
    torch.cuda.synchronize()
    ts = (ctypes.c_ulonglong * 16)()
    _lib.check(L.vmm_prune_prof_read(ts))
    if i >= 3:
        acc += np.diff(np.array(ts[:9], dtype=np.float64))
for nm, v in zip(names, acc / n):
    print(f"{nm:16s} {v / 1e3:8.2f} us")
print(f"{'total':16s} {acc.sum() / n / 1e3:8.2f} us (CTA 0, launch excluded)")
