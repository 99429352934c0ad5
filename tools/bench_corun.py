"""Does the HBM-bound glue (permute / combine / norm) co-run with the tcgen05 FFN?

Times, on a C3-shaped half batch (all experts resident): FFN alone, glue alone,
both serially on one stream, and both concurrently on two streams (glue on a
second stream launched right after the FFN).

    python tools/bench_corun.py [tokens=155648]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_05899_b200 import kernels

N = int(sys.argv[1]) if len(sys.argv) > 1 else 155648
H, I, E, k = 2048, 768, 128, 8
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(N, H, device=dev, generator=g).to(torch.bfloat16)
arena = (torch.randn(E, 3 * I * H, device=dev, generator=g) * 0.02).to(torch.bfloat16)
ids = torch.topk(torch.randn(N, E, device=dev, generator=g), k, dim=1).indices.int().contiguous()
gates = torch.rand(N, k, device=dev, generator=g)
M = N * k
bufA = (torch.empty(E + 1, dtype=torch.int32, device=dev), torch.empty(M, dtype=torch.int32, device=dev),
        torch.empty(M, dtype=torch.int32, device=dev))
bufB = tuple(torch.empty_like(b) for b in bufA)
off, src, pos, xp = kernels.permute(ids, x, E, bufs=bufA)
xp2 = torch.empty_like(xp)
slot = torch.arange(E, dtype=torch.int32, device=dev)
h1 = torch.empty(M, I, dtype=torch.bfloat16, device=dev)
y = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
y2 = torch.randn(M, H, device=dev).to(torch.bfloat16)
out = torch.empty_like(x)
xn = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s2 = torch.cuda.Stream()


def ffn(st=None):
    kernels.grouped_swiglu(xp, off, arena, slot, I, h1=h1, y=y, stream=st)


def glue(st=None):
    kernels.combine(y2, pos.view(N, k), gates, x, out=out, stream=st)
    kernels.rmsnorm(out, out=xn, stream=st)
    kernels.permute(ids, xn, E, bufs=bufB, out=xp2, stream=st)


def timed(fn, reps=6):
    ts = []
    for i in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    return sum(ts) / len(ts)


def both_serial():
    ffn()
    glue()


def both_concurrent():
    ffn()
    s2.wait_stream(torch.cuda.current_stream())  # (the flush) -- glue does not depend on the FFN here
    glue(s2)
    torch.cuda.current_stream().wait_stream(s2)


def both_concurrent_glue_first():
    s2.wait_stream(torch.cuda.current_stream())
    glue(s2)
    ffn()
    torch.cuda.current_stream().wait_stream(s2)


for name, fn in (("ffn", ffn), ("glue", glue), ("serial", both_serial), ("concurrent", both_concurrent),
                 ("concurrent(glue first)", both_concurrent_glue_first)):
    print(f"{name:24s} {timed(fn):8.3f} ms", flush=True)
