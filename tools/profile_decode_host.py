"""cProfile of the decode step's host side (C3, trace routing, oracle predictor)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.moe import MoEStack, StackConfig
from paper_2605_05899_b200.trace import generate_trace

w = WORKLOADS["c3_qwen3vl"]
D = 16
tr = generate_trace(w.trace_config(seed=0, decode_steps=D))
T = tr.num_tokens - D
cfg = StackConfig.from_workload(w, routing="trace", predictor="oracle")
stack = MoEStack(cfg, seed=1)
x = torch.randn((T, w.hidden), device="cuda").to(torch.bfloat16)
dtr = dict(routes=torch.from_numpy(tr.route_experts.astype(np.int32)).cuda(),
           gates=torch.from_numpy(tr.route_gates.astype(np.float32)).cuda())
stack.forward(x, torch.from_numpy(tr.saliency[:T]).cuda(), torch.from_numpy(tr.device_modality()[:T]).cuda(),
              trace=dtr, keep_session=True)
toks = torch.randn((D, 1, w.hidden), device="cuda").to(torch.bfloat16)
torch.cuda.synchronize()
stack.decode_step(toks[0], tok=T)
pr = cProfile.Profile()
pr.enable()
for i in range(1, D):
    stack.decode_step(toks[i], tok=T + i)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
