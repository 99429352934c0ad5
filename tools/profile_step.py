"""One warm-up + N measured requests of a workload through the live stack (for ncu)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.moe import MoEStack, StackConfig
from paper_2605_05899_b200.trace import generate_trace
from paper_2605_05899_b200 import kernels

name = sys.argv[1] if len(sys.argv) > 1 else "c3_qwen3vl"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = WORKLOADS[name]
cfg = StackConfig.from_workload(w, routing="live", predictor="gate")
stack = MoEStack(cfg, seed=1000)
tr = generate_trace(w.trace_config(seed=0))
x = torch.randn((tr.num_tokens, w.hidden), device="cuda").to(torch.bfloat16)
sal = torch.from_numpy(tr.saliency).cuda(); mod = torch.from_numpy(tr.device_modality()).cuda()
stack.forward(x, sal, mod); torch.cuda.synchronize()
n0 = kernels.LAUNCHES[0]
print("launches_warmup", n0, flush=True)
for _ in range(steps):
    stack.forward(x, sal, mod)
torch.cuda.synchronize()
print("launches_per_step", (kernels.LAUNCHES[0] - n0) // steps, flush=True)
