"""Time the device prune (vmm_prune) at C3 request shapes: R requests of 2304
visual + 64 text tokens, 8 prefix layers, E=128 top-8 (CUDA events, L2 flushed,
median of 20).  Prints one JSON line per R with the achieved HBM rate on the
algorithmic bytes (saliency + modality + prefix routes read, s_norm/delta/score/
flags/retained written)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_05899_b200 import _lib, kernels  # noqa: E402
from paper_2605_05899_b200._lib import ptr  # noqa: E402


def main():
    dev = torch.device("cuda")
    nv, nt, P, k, E = 2304, 64, 8, 8, 128
    T1 = nv + nt
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for R in [int(x) for x in (sys.argv[1:] or ["1", "8", "64", "256"])]:
        rng = np.random.default_rng(R)
        T = T1 * R
        sal = torch.from_numpy(rng.gamma(2.0, 1.0, size=T)).to(dev)
        mod = torch.from_numpy(np.tile(np.r_[np.zeros(nv, np.uint8), np.ones(nt, np.uint8)], R)).to(dev)
        routes = torch.randint(0, E, (P, T, k), dtype=torch.int32, device=dev)
        offs = torch.tensor([r * T1 for r in range(R + 1)], dtype=torch.int32, device=dev)
        out = kernels.prune(sal, mod, routes, offs, None, None, E, 2.0, alpha=0.1, beta=0.5)
        L = _lib.lib()
        st = torch.cuda.current_stream().cuda_stream
        args = [ptr(sal), ptr(mod), ptr(routes), ptr(offs), None, None, 0.1, 0.5, R, T, P, k, E, 2.0,
                ptr(out["s_norm"]), ptr(out["delta"]), ptr(out["score"]), ptr(out["flags"]), ptr(out["retained"]),
                ptr(out["n_retained"]), ptr(out["target"]), ptr(out["status"]), st]
        times = []
        for i in range(25):  # kernel only: the C-ABI launch on preallocated outputs, L2 flushed
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _lib.check(L.vmm_prune(*args))
            b.record()
            b.synchronize()
            if i >= 5:
                times.append(a.elapsed_time(b))
        assert (out["status"].cpu().numpy() == 0).all()
        ms = float(np.median(times))
        nbytes = T * (8 + 1 + P * k * 4) + T * (3 * 8 + 1) + int(out["n_retained"].sum()) * 4
        print(json.dumps({"kernel": "prune_kernel", "requests": R, "tokens": T, "ms": ms,
                          "us_per_request": ms * 1e3 / R, "alg_bytes": nbytes,
                          "gbs": nbytes / (ms * 1e-3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
