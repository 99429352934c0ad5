"""Repeated 1 GiB pinned->device copies for `secs` seconds on one stream; prints GB/s.
Run two at once (two processes) to see whether the link, or one copy stream, is the limit."""
import sys
import time

import torch

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d.copy_(h)
torch.cuda.synchronize()
t0, k = time.perf_counter(), 0
while time.perf_counter() - t0 < secs:
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    k += 1
dt = time.perf_counter() - t0
print(f"{k * n / dt / 1e9:.1f} GB/s over {dt:.1f} s ({k} copies)")
