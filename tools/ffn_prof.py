"""Where the pair FFN kernel's cycles go: per-CTA wait counters of the
VMM_FFN_PROF build (VMM_BUILD_VARIANT=prof python -m paper_2605_05899_b200.build).

    python tools/ffn_prof.py [rows_per_request=1216] [requests=256]

Slots (cycles, summed over the CTA's tiles; fractions of the CTA's kernel time):
  0 producer: ready-flag / H1-done waits   1 producer: empty-stage waits
  2 MMA: TMEM accumulator free waits        3/4 MMA: full-stage waits (GEMM1 / GEMM2)
  5 epilogue warp 2: TMEM full waits        7 kernel cycles (thread 0)
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

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 1216
R = int(sys.argv[2]) if len(sys.argv) > 2 else 256
H, I, E, k = 2048, 768, 128, 8
N = n_r * R
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
arena = (torch.randn(E, 3 * I * H, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
ids = torch.topk(torch.randn(N, E, device="cuda", generator=g), k, dim=1).indices.int()
off, src, pos = kernels.permute_plan(ids, E)
xp = kernels.permute_rows(x, src, N * k)
slot = torch.arange(E, dtype=torch.int32, device="cuda")
M = N * k
lib = _lib.lib()
buf = (ctypes.c_ulonglong * (256 * 24))()
lib.vmm_ffn_prof_mode(int(os.environ.get("FFN_PROF_MODE", "0")))  # 1: no H1 waits, 2: no stores (wrong results)
for it in range(3):
    torch.cuda.synchronize()
    lib.vmm_ffn_prof_read(buf, 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    if os.environ.get("FFN_PROF_GATHER"):
        kernels.grouped_swiglu(M, off, arena, slot, I, x_rows=x, src_row=src)
    else:
        kernels.grouped_swiglu(xp, off, arena, slot, I)
    b.record()
    b.synchronize()
    lib.vmm_ffn_prof_read(buf, 0)
    ms = a.elapsed_time(b)
c = np.frombuffer(buf, dtype=np.uint64).reshape(256, 24)[:148].astype(np.float64)
tot = c[:, 7]
names = ["prod flag/H1 wait", "prod empty wait", "mma tmem-free wait", "mma full wait G1", "mma full wait G2",
         "epi tmem-full wait"]
print(f"M={M}: {ms:.3f} ms, {6.0 * M * H * I / ms / 1e9:.0f} TFLOP/s; kernel cycles/CTA mean {tot.mean():.3e} "
      f"(-> {tot.mean() / (ms * 1e-3) / 1e9:.2f} GHz)")
n_g2 = (M / 256 + E) * (H // 256) / 74
print(f"  GEMM2 tiles not ready at first check: {c[:, 6].sum() / 148:.0f} per CTA (of ~{n_g2:.0f} GEMM2 tiles)")
print(f"  epi (warp 2) GEMM1 tile-end (bulk wait + fences + release) {(c[:, 12] / tot).mean():.3f}, "
      f"staging+store issue {(c[:, 13] / tot).mean():.3f} of kernel cycles")
for j, nm in enumerate(names):
    f = c[:, j] / tot
    print(f"  {nm:20s} mean {f.mean():6.3f}  min {f.min():6.3f}  max {f.max():6.3f} of kernel cycles")
print(f"  epi (warp 2) bulk_wait_read {(c[:, 14] / tot).mean():.3f}, tmem ld wait {(c[:, 15] / tot).mean():.3f} of kernel cycles")
print(f"  epi (warp 2) busy per tile: GEMM1 {c[:, 16].sum() / c[:, 18].sum():.0f} cycles, "
      f"GEMM2 {c[:, 17].sum() / c[:, 19].sum():.0f} cycles; MMA cycles per k-step at peak ~542 "
      f"(GEMM1 32 k-steps, GEMM2 12)")
lead = c[0::2]
busy = 1 - (lead[:, 2] + lead[:, 3] + lead[:, 4]) / lead[:, 7]
work = lead[:, 8] * 32 + lead[:, 9] * 12  # ~cost units: k-steps (GEMM1 nk=32 per tile... counted per k-step)
t0 = c[:, 10].min()
print("  leader MMA busy frac: min %.3f median %.3f max %.3f" % (busy.min(), np.median(busy), busy.max()))
print("  leader k-steps G1: min %d max %d; G2: min %d max %d" % (lead[:, 8].min(), lead[:, 8].max(), lead[:, 9].min(),
                                                               lead[:, 9].max()))
print("  CTA start skew %.1f us, end spread %.1f us (first end %.1f ms, last %.1f ms)" % (
    (c[:, 10].max() - t0) / 1e3, (c[:, 11].max() - c[:, 11].min()) / 1e3, (c[:, 11].min() - t0) / 1e6,
    (c[:, 11].max() - t0) / 1e6))
