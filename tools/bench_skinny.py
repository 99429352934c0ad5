"""Decode-sized grouped SwiGLU (one token, top-8 of 128 experts, C3 shapes): the
skinny weight-streaming kernel alone, L2 flushed before every launch.

    python tools/bench_skinny.py [rows=8]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05899_b200 import kernels

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
H, I, E, k = 2048, 768, 128, 8
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
arena = (torch.randn(E, 3 * I * H, device=dev, generator=g) * 0.02).to(torch.bfloat16)
x = torch.randn(M, H, device=dev, generator=g).to(torch.bfloat16)
# M picks on M distinct experts spread over the arena
off = torch.zeros(E + 1, dtype=torch.int32, device=dev)
sel = torch.randperm(E, generator=torch.Generator().manual_seed(1))[:M].sort().values
cnt = torch.zeros(E, dtype=torch.int32)
cnt[sel] = 1
off[1:] = torch.cumsum(cnt, 0).to(dev)
slot = torch.arange(E, dtype=torch.int32, device=dev)
h1 = torch.empty(M, I, dtype=torch.bfloat16, device=dev)
y = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for i in range(30):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    kernels.grouped_swiglu(x, off, arena, slot, I, h1=h1, y=y)
    b.record()
    b.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
wbytes = M * 3 * I * H * 2
print(f"skinny FFN M={M}: median {ts[len(ts) // 2]:.1f} us, min {ts[0]:.1f} us -> "
      f"{wbytes / (ts[len(ts) // 2] * 1e-6) / 1e12:.2f} TB/s of expert weights ({wbytes / 1e6:.1f} MB)")
if os.environ.get("VMM_LIB", "").endswith("_prof.so"):  # per-CTA phase timestamps (VMM_FFN_PROF build)
    import ctypes
    import numpy as np

    from paper_2605_05899_b200 import _lib
    buf = (ctypes.c_ulonglong * (256 * 24))()
    torch.cuda.synchronize()
    flush.zero_()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    kernels.grouped_swiglu(x, off, arena, slot, I, h1=h1, y=y)
    b.record()
    b.synchronize()
    _lib.lib().vmm_ffn_prof_read(buf, 0)
    c = np.frombuffer(buf, dtype=np.uint64).reshape(256, 24)[:148, 20:24].astype(np.int64)
    t0 = c[:, 0].min()
    r = (c - t0) / 1e3
    print(f"  event {a.elapsed_time(b) * 1e3:.1f} us; CTA start spread {r[:, 0].max():.1f} us; phase1 done "
          f"min/med/max {r[:, 1].min():.1f}/{np.median(r[:, 1]):.1f}/{r[:, 1].max():.1f}; barrier passed max "
          f"{r[:, 2].max():.1f}; end min/med/max {r[:, 3].min():.1f}/{np.median(r[:, 3]):.1f}/{r[:, 3].max():.1f} us")
