"""Sharded-home R=1 step anatomy: host microseconds per phase (pre-sync launches, sync wait,
decisions + copy issue, post launches) over the cached layers, copy count, step time.

    python tools/sharded_r1_host.py [requests=1]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.moe import ExpertStore, MoEStack, ShardedHome, StackConfig
from paper_2605_05899_b200.trace import generate_trace

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = WORKLOADS["c3_qwen3vl"]
cfg = StackConfig.from_workload(w, routing="live", predictor="gate", host_layers=8,
                                transfer_ms=w.expert_bytes / 3.2e12 * 1e3, gpu_ms=0.01)
store = ExpertStore(cfg, seed=1000)
home = ShardedHome(store, 0, 1)
stack = MoEStack(cfg, store=store, home=home)
tr = generate_trace(w.trace_config(seed=0))
T1 = tr.num_tokens
x = torch.randn((T1 * R, w.hidden), device="cuda").to(torch.bfloat16)
sal = torch.from_numpy(np.concatenate([tr.saliency] * R)).cuda()
mod = torch.from_numpy(np.concatenate([tr.device_modality()] * R)).cuda()
offs = [r * T1 for r in range(R + 1)]
for it in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = stack.forward(x, sal, mod, req_off=offs)
    e1.record()
    torch.cuda.synchronize()
print(f"R={R} step {e0.elapsed_time(e1):.1f} ms, copies {res.copies}, copy window {res.h2d_ms:.1f} ms, "
      f"{res.h2d_bytes / max(res.h2d_ms, 1e-9) / 1e6:.0f} GB/s")
print("host us (pre, sync, decide+issue, post) over cached layers:", [round(v) for v in stack.last_host_us])
