"""Time the fused grouped SwiGLU alone on a C3-shaped layer (all experts resident).

    python tools/bench_ffn.py [rows_per_request=1216] [requests=128]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05899_b200 import kernels

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 1216
R = int(sys.argv[2]) if len(sys.argv) > 2 else 128
H, I, E, k = 2048, 768, 128, 8
N = n_r * R
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
arena = (torch.randn(E, 3 * I * H, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
ids = torch.topk(torch.randn(N, E, device="cuda", generator=g), k, dim=1).indices.int()
off, src, pos = kernels.permute_plan(ids, E)
xp = kernels.permute_rows(x, src, N * k)
slot = torch.arange(E, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
M = N * k
flops = 6.0 * M * H * I
MODES = os.environ.get("FFN_MODES", "gather,fused,split").split(",")
for mode in MODES:
    ts = []
    for i in range(6):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if mode == "gather":
            kernels.grouped_swiglu(M, off, arena, slot, I, x_rows=x, src_row=src)
        else:
            kernels.grouped_swiglu(xp, off, arena, slot, I, fused=(mode == "fused"))
        b.record()
        b.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    ms = sum(ts) / len(ts)
    print(f"{mode:6s} M={M} {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s "
          f"{(E * 3 * I * H * 2 + M * H * 4 + M * I * 4) / ms / 1e6:.0f} GB/s(alg)", flush=True)
