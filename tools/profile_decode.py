"""Prefill one request (trace routing) then N decode steps -- for ncu launch lists of the decode phase.
Prints the library launch count after prefill (use it as ncu -s with the kernel-name filter)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_05899_b200 import _lib
from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.moe import MoEStack, StackConfig
from paper_2605_05899_b200.trace import generate_trace

name = sys.argv[1] if len(sys.argv) > 1 else "c3_qwen3vl"
D = int(sys.argv[2]) if len(sys.argv) > 2 else 4
pred = sys.argv[3] if len(sys.argv) > 3 else "oracle"
w = WORKLOADS[name]
tr = generate_trace(w.trace_config(seed=0, decode_steps=D))
T = tr.num_tokens - D
cfg = StackConfig.from_workload(w, routing="trace", predictor=pred)
stack = MoEStack(cfg, seed=1000)
dtr = dict(routes=torch.from_numpy(tr.route_experts.astype(np.int32)).cuda(),
           gates=torch.from_numpy(tr.route_gates.astype(np.float32)).cuda())
x = torch.randn((T, w.hidden), device="cuda").to(torch.bfloat16)
stack.forward(x, torch.from_numpy(tr.saliency[:T]).cuda(), torch.from_numpy(tr.device_modality()[:T]).cuda(),
              trace=dtr, keep_session=True)
torch.cuda.synchronize()
n0 = _lib.load().vmm_launch_count()
print("launches_after_prefill", n0, flush=True)
for s in range(D):
    stack.decode_step(torch.randn((1, w.hidden), device="cuda").to(torch.bfloat16), tok=T + s)
torch.cuda.synchronize()
print("launches_per_decode_step", (_lib.load().vmm_launch_count() - n0) // D, flush=True)
