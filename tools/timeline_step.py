"""Per-layer timeline of one batched prefill step (FFN events, host phases, copy stream).

    python tools/timeline_step.py [requests] [workload]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.moe import MoEStack, StackConfig
from paper_2605_05899_b200.trace import generate_trace

R = int(sys.argv[1]) if len(sys.argv) > 1 else 128
w = WORKLOADS[sys.argv[2] if len(sys.argv) > 2 else "c3_qwen3vl"]
cfg = StackConfig.from_workload(w, routing="live", predictor="gate", host_layers=8)
stack = MoEStack(cfg, seed=1000)
tr = generate_trace(w.trace_config(seed=0))
T1 = tr.num_tokens
x = torch.randn((T1 * R, w.hidden), device="cuda").to(torch.bfloat16)
rng = np.random.default_rng(0)
sal = torch.from_numpy(np.concatenate([tr.saliency] + [rng.gamma(2.0, 1.0, T1) for _ in range(R - 1)])).cuda()
mod = torch.from_numpy(np.concatenate([tr.device_modality()] * R)).cuda()
offs = [r * T1 for r in range(R + 1)]
ITERS = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for it in range(ITERS):
    stack.profile = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = stack.forward(x, sal, mod, req_off=offs)
    e1.record()
    torch.cuda.synchronize()
    prof = stack.profile
    stack.profile = None
total = e0.elapsed_time(e1)
pre = [p for p in prof if p[4]]
prof = [p for p in prof if not p[4]]
starts = [p[0] for p in prof]
ffn = [p[0].elapsed_time(p[1]) for p in prof]
lp = 0
print(f"R={R} step {total:.1f} ms, copies {res.copies}, h2d {res.h2d_bytes / 1e9:.1f} GB")
print(f"prefix (start -> first cached FFN): {e0.elapsed_time(starts[0]):.1f} ms; prefix FFN launches {len(pre)}, "
      f"sum {sum(p[0].elapsed_time(p[1]) for p in pre):.1f} ms")
per = [starts[i].elapsed_time(starts[i + 1]) for i in range(lp, len(starts) - 1)]
print(f"cached layers: period mean {np.mean(per):.2f} ms, FFN(incl. copy waits) mean {np.mean(ffn[lp:]):.2f} ms,"
      f" non-FFN mean {np.mean(per) - np.mean(ffn[lp:-1]):.2f} ms")
print("host us (pre, sync, decide, post) over cached layers:", [round(v / 1e3, 1) for v in stack.last_host_us])
print(f"copy stream: {res.copies} copies, {res.h2d_bytes / 1e9:.1f} GB, first->last copy {res.h2d_ms:.1f} ms "
      f"= {res.h2d_bytes / res.h2d_ms / 1e6:.1f} GB/s over the copy window")
cm = stack.last_copy_marks
if cm:
    nl = len(cm) // 3
    dem = [cm[3 * i].elapsed_time(cm[3 * i + 1]) for i in range(nl)]
    emi = [cm[3 * i + 1].elapsed_time(cm[3 * i + 2]) for i in range(nl)]
    idle = [cm[3 * (i - 1) + 2].elapsed_time(cm[3 * i]) for i in range(1, nl)]
    print(f"copy stream per cached layer: demand {np.mean(dem):.2f} ms, emission prefetch {np.mean(emi):.2f} ms, "
          f"gap before next demand {np.mean(idle):.2f} ms (mean)")
print("per-layer period:", [round(v, 1) for v in per])
print("per-layer ffn   :", [round(v, 1) for v in ffn])
if cm and len(cm) // 3 == len(prof):
    tail = [cm[3 * i + 1].elapsed_time(prof[i][1]) for i in range(len(prof))]
    lead = [cm[3 * i].elapsed_time(prof[i][0]) for i in range(len(prof))]
    print(f"FFN end after its demand copies done: mean {np.mean(tail):.2f} ms; FFN start after copies start: "
          f"mean {np.mean(lead):.2f} ms")
    print("per-layer tail:", [round(v, 2) for v in tail])
if cm and len(cm) // 3 == len(prof):
    post = [prof[i][1].elapsed_time(cm[3 * (i + 1)]) for i in range(len(prof) - 1)]
    print(f"FFN(l) end -> layer l+1 copies start: mean {np.mean(post):.2f} ms (first-chunk combine/norm/route, "
          f"D2H, host decision, issue)")
