"""Decode-phase measurement.

Prefill one request, then D decode tokens through all layers with the cache
persisting (pipeline.py:723-740); per-token wall time with CUDA events, the
decode hit rate and H2D bytes.  Compares lookahead predictors with
predictor=none (demand-only loading: the no-prefetch baseline).

  live  : live router on synthetic hidden states (router_corr couples the
          gates of consecutive layers; decode tokens follow an AR(1) sequence)
  trace : routes from the reference trace generator incl. its decode tokens
          (rho persistence across layers and steps); oracle predictor allowed

    python tools/bench_decode.py [workload] [D] [pred,pred,...] [live|trace]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.moe import ExpertStore, MoEStack, StackConfig
from paper_2605_05899_b200.trace import generate_trace

name = sys.argv[1] if len(sys.argv) > 1 else "c3_qwen3vl"
D = int(sys.argv[2]) if len(sys.argv) > 2 else 16
preds = sys.argv[3].split(",") if len(sys.argv) > 3 else ["gate", "none"]
routing = sys.argv[4] if len(sys.argv) > 4 else "live"
w = WORKLOADS[name]
tr = generate_trace(w.trace_config(seed=0, decode_steps=D if routing == "trace" else 0))
T = tr.num_tokens - (D if routing == "trace" else 0)
x = torch.randn((T, w.hidden), device="cuda").to(torch.bfloat16)
sal = torch.from_numpy(tr.saliency[:T]).cuda()
mod = torch.from_numpy(tr.device_modality()[:T]).cuda()
dtr = None
if routing == "trace":
    dtr = dict(routes=torch.from_numpy(tr.route_experts.astype(np.int32)).cuda(),
               gates=torch.from_numpy(tr.route_gates.astype(np.float32)).cuda())
store = None
out = {}
for pred in preds:
    cfg = StackConfig.from_workload(w, routing=routing, predictor=pred)
    if store is None:
        store = ExpertStore(cfg, seed=1000)
    stack = MoEStack(cfg, store=store)
    g = torch.Generator(device="cuda").manual_seed(7)
    toks, t = [], torch.randn((1, w.hidden), generator=g, device="cuda")
    for _ in range(D):  # AR(1) decode-token hidden states (consecutive tokens correlate)
        toks.append(t.to(torch.bfloat16))
        t = 0.9 * t + (1 - 0.81) ** 0.5 * torch.randn((1, w.hidden), generator=g, device="cuda")
    res = stack.forward(x, sal, mod, trace=dtr, keep_session=True)
    pre = res.report
    ms, copies, host = [], 0, np.zeros(4)
    ffn = []
    for s, tk in enumerate(toks):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stack.profile = [] if s == D - 1 else None  # FFN events on the last token only
        e0.record()
        r = stack.decode_step(tk, tok=T + s if routing == "trace" else None)
        e1.record()
        e1.synchronize()
        if stack.profile:
            ffn = [p[0].elapsed_time(p[1]) * 1e3 for p in stack.profile]
        stack.profile = None
        ms.append(e0.elapsed_time(e1))
        copies += r.copies
        host += np.asarray(stack.last_host_us)
    rep = stack.end_session()
    dh, dm = rep.hits - pre.hits, rep.misses - pre.misses
    steady = ms[1:] if D > 1 else ms
    out[pred] = dict(decode_ms_per_token=float(np.mean(steady)), decode_tokens_per_s=1e3 / float(np.mean(steady)),
                     decode_hit_rate=dh / max(dh + dm, 1), copies_per_token=copies / D,
                     h2d_bytes_per_token=copies * cfg.slot_bytes / D, ms_first_token=ms[0],
                     ffn_us_per_layer=float(np.mean(ffn)) if ffn else None,
                     host_us_per_token=dict(zip(["launch_pre_sync", "sync_wait", "decisions_copies", "launch_post"],
                                                (host / D).round(1).tolist())))
    print(pred, json.dumps(out[pred]), flush=True)
base = out.get("none")
if base:
    for p in preds:
        if p != "none":
            out[f"speedup_{p}_vs_none"] = base["decode_ms_per_token"] / out[p]["decode_ms_per_token"]
print(json.dumps({"workload": name, "routing": routing, "decode_steps": D, **out}))
