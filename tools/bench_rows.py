"""Timings for the §8(f) rows 2 and 4: attention saliency, GPU routing
diagnostics (vs the oracle port of moesim.metrics on the host), binary trace I/O."""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import metrics_ref as M
from paper_2605_05899_b200 import metrics
from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.saliency import attention_saliency
from paper_2605_05899_b200.trace import generate_trace, load_trace_bin, save_trace_bin


def cuda_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


w = WORKLOADS["c3_qwen3vl"]
tr = generate_trace(w.trace_config(seed=0))
ids = list(range(tr.num_tokens))
dev_ms = cuda_ms(lambda: metrics.layer_diagnostics(tr, ids, 8))
t0 = time.perf_counter()
for l in range(tr.layers):
    M.working_set(tr.route_experts, tr.experts, ids, l)
    M.topk_coverage(tr.route_experts, tr.experts, ids, l, 8)
    if l + 1 < tr.layers:
        M.interlayer_similarity(tr.route_experts, tr.experts, ids, l)
        M.interlayer_jaccard(tr.route_experts, tr.experts, ids, l)
cpu_ms = (time.perf_counter() - t0) * 1e3
print(f"affinity report C3 (48 layers, {len(ids)} tokens): device {dev_ms:.3f} ms (incl. D2H), "
      f"oracle port (numpy, 1 thread) {cpu_ms:.1f} ms")
for R, Q in ((1, 1), (256, 1), (16, 64)):
    q = torch.randn(R, 16, Q, 72, device="cuda").to(torch.bfloat16)
    k = torch.randn(R, 16, tr.num_tokens, 72, device="cuda").to(torch.bfloat16)
    ms = cuda_ms(lambda: attention_saliency(q, k))
    kb = k.numel() * 2 + q.numel() * 2
    print(f"attention saliency R={R} heads=16 queries={Q} tokens={tr.num_tokens} D=72: {ms:.3f} ms "
          f"({kb / ms / 1e6:.0f} GB/s of Q/K)")
with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "c3.vmm")
    t0 = time.perf_counter()
    save_trace_bin(tr, p)
    t1 = time.perf_counter()
    back = load_trace_bin(p)
    t2 = time.perf_counter()
    print(f"binary trace C3 ({os.path.getsize(p) / 1e6:.1f} MB): save {1e3 * (t1 - t0):.1f} ms, "
          f"load+validate {1e3 * (t2 - t1):.1f} ms")
