"""Router launch time vs K-split count S (VMM_ROUTE_SPLIT forces S at every N).

    python tools/route_split_sweep.py            # parent: one child process per S
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

if len(sys.argv) == 1:
    for S in ["auto", "1", "2", "4", "8"]:
        env = dict(os.environ)
        if S != "auto":
            env["VMM_ROUTE_SPLIT"] = S
        out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(f"S={S}: {out.stdout.strip()} {out.stderr.strip()[-300:] if out.returncode else ''}", flush=True)
    sys.exit(0)

import torch

from paper_2605_05899_b200 import kernels

L, H, E, k = 48, 2048, 128, 8
g = torch.Generator(device="cuda").manual_seed(0)
router = (torch.randn(L, E, H, device="cuda", generator=g) / 45).to(torch.bfloat16)
counts = torch.zeros(E, dtype=torch.int32, device="cuda")
lac = torch.zeros(E, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for N in (8, 1216, 9728, 38912, 311296):
    x = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
    for la in (0, 1):
        ts = []
        for i in range(13):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if la:
                kernels.route_lookahead(x, router, 3, k, counts, lac)
            else:
                kernels.route_topk(x, router[3], k, counts=counts)
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        res.append(f"N={N}{'+la' if la else ''} {ts[len(ts) // 2]:.1f}us")
print("  ".join(res))
