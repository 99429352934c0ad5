"""Debug helper: run the live stack at a given workload shape with overrides."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.moe import MoEStack, StackConfig
from paper_2605_05899_b200.trace import generate_trace, TraceGenConfig

kw = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
w = WORKLOADS[kw.pop("workload", "c3_qwen3vl")]
nv = kw.pop("n_visual", w.n_visual)
routing = kw.get("routing", "live")
cfg = StackConfig.from_workload(w, **{"predictor": "gate", **kw})
print(cfg, flush=True)
stack = MoEStack(cfg)
tr = generate_trace(TraceGenConfig(n_visual=nv, n_text=w.n_text, layers=cfg.layers, experts=w.experts, k=w.k, visual_noise=0.3, seed=0))
x = torch.randn((tr.num_tokens, w.hidden), device="cuda").to(torch.bfloat16)
dtr = dict(routes=torch.from_numpy(tr.route_experts.astype(np.int32)).cuda(), gates=torch.from_numpy(tr.route_gates.astype(np.float32)).cuda())
for i in range(2):
    t = time.time()
    res = stack.forward(x, torch.from_numpy(tr.saliency).cuda(), torch.from_numpy(tr.device_modality()).cuda(), trace=dtr)
    torch.cuda.synchronize()
    print("step", i, time.time() - t, "copies", res.copies, "hit", res.report.hit_rate, flush=True)
