"""Generate golden vectors by running the REAL reference (`moesim`).

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed, small): compress.json, predict.npz + predict.json,
cache_ops.json, engine.json, traces.json.  Traces are stored as generator
configs plus a digest; the product generator regenerates them bit-identically
(pinned by tests/test_trace_golden.py).
"""
from __future__ import annotations

import json
import math
import os
import sys
from dataclasses import asdict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import moesim  # noqa: E402  (reference)
from moesim import (  # noqa: E402
    CompressionConfig, ExpertCache, ExpertRef, Modality, PredictorSpec, RoutingTrace,
    SimConfig, Token, TraceGenConfig, build_plan, compress, generate_trace, simulate,
    simulate_reactive,
)
from moesim.cache import ResidencyClass  # noqa: E402
from moesim.errors import SimulationError  # noqa: E402
from moesim.predictor import (  # noqa: E402
    build_features, build_targets, init_model, predict_topb, routing_histogram, layer_drift,
)

from paper_2605_05899_b200.configs import WORKLOADS  # noqa: E402
from paper_2605_05899_b200.trace import RoutingTrace as MyTrace, trace_digest  # noqa: E402


def digest_ref(tr) -> str:
    return trace_digest(MyTrace.from_reference(tr))


def gen_cfg_dict(c: TraceGenConfig) -> dict:
    d = asdict(c)
    d["saliency_shape"] = list(d["saliency_shape"])
    return d


# ---------------------------------------------------------------------------
def compress_cases():
    out = {"random": [], "frozen": None, "traces": []}
    # frozen instance (test_compress.py:89-100)
    sal = [9, 1, 8, 7, 3, 5]
    routes = [[[0], [0], [1], [2], [1], [3]]]
    out["frozen"] = dict(saliency=sal, routes=routes, experts=4, k=1, alpha=1 / 6, beta=0.5, lam=2.0, prefix=[0])
    rng = np.random.default_rng(11)
    for _ in range(400):
        n = int(rng.integers(1, 11))
        experts = int(rng.integers(2, 7))
        k = int(rng.integers(1, min(2, experts) + 1))
        sal = [float(v) for v in rng.integers(0, 5, size=n)]
        routes = [[sorted(rng.choice(experts, size=k, replace=False).tolist()) for _ in range(n)] for _ in range(2)]
        prefix = [0] if rng.random() < 0.5 else [0, 1]
        beta = float(rng.uniform(0, 1))
        alpha = float(rng.uniform(0, beta))
        lam = float(rng.choice([0.0, 0.5, 1.0, 2.0, 5.0, 0.3, 1.7]))
        tokens = [Token(i, Modality.VISUAL, sal[i], np.zeros(1)) for i in range(n)]
        tr = RoutingTrace(2, experts, k, tokens, np.array(routes, dtype=np.int64), np.full((2, n, k), 1.0 / k))
        p = compress(tr, CompressionConfig(alpha, beta, lam, tuple(prefix)))
        out["random"].append(dict(
            saliency=sal, routes=routes, experts=experts, k=k, alpha=alpha, beta=beta, lam=lam, prefix=prefix,
            core=p.core, keep=p.keep, target=sorted(p.target_experts),
            delta=[[i, p.delta[i]] for i in sorted(p.delta)], score=[[i, p.score[i]] for i in sorted(p.score)],
        ))
    # generated traces, incl. the full C1 and C3 shapes
    specs = []
    for name in ("c1_tiny", "c3_qwen3vl", "c4_dsvl2s"):
        w = WORKLOADS[name]
        specs.append((name, w.trace_config(seed=0), CompressionConfig(w.alpha, w.beta, w.lam, w.prefix_layers)))
    for seed in range(6):
        g = TraceGenConfig(n_visual=40 + 7 * seed, n_text=5, layers=4, experts=16, k=3, cluster_support=6,
                           visual_noise=0.4, seed=100 + seed, decode_steps=seed % 3)
        specs.append((f"small{seed}", g, CompressionConfig(0.1 + 0.02 * seed, 0.5, [0.3, 2.0, 5.0][seed % 3], (0, 1))))
    for name, g, cc in specs:
        tr = generate_trace(g)
        p = compress(tr, cc)
        vis = tr.visual_ids()
        out["traces"].append(dict(
            name=name, gen=gen_cfg_dict(g), digest=digest_ref(tr),
            alpha=cc.alpha, beta=cc.beta, lam=cc.lam, prefix=list(cc.prefix_layers),
            core=p.core, keep=p.keep, target=sorted(p.target_experts), retained=p.retained_ids(tr),
            delta_hex=[float(p.delta[i]).hex() if i in p.delta else None for i in vis],
            score_hex=[float(p.score[i]).hex() if i in p.score else None for i in vis],
            snorm_hex=[float(p.saliency_norm[i]).hex() for i in vis],
        ))
    return out


# ---------------------------------------------------------------------------
def predict_cases():
    cases = []
    rng = np.random.default_rng(22)
    for it in range(30):
        g = TraceGenConfig(
            n_visual=int(rng.integers(2, 30)), n_text=int(rng.integers(1, 6)), layers=int(rng.integers(2, 10)),
            experts=int(rng.choice([4, 8, 13, 64, 128, 200])), k=int(rng.integers(1, 4)),
            clusters=int(rng.integers(1, 4)), cluster_support=4, rho=float(rng.random()),
            visual_noise=float(rng.random() * 0.5), seed=int(rng.integers(100_000)))
        if g.cluster_support > g.experts:
            g.cluster_support = g.experts
        tr = generate_trace(g)
        prefill = tr.prefill_ids()
        for _ in range(3):
            layer = int(rng.integers(0, tr.layers))
            window = int(rng.integers(1, 6))
            gamma = float(rng.choice([0.5, 0.8, 1.0, 0.3]))
            decay = float(rng.choice([0.5, 0.3, 0.0, 0.9, 1.0]))
            size = int(rng.integers(1, len(prefill) + 1))
            ids = sorted(int(i) for i in rng.choice(prefill, size=size, replace=False))
            tgt = build_targets(tr, layer, window, gamma, token_ids=ids)
            hist = routing_histogram(tr, ids, layer, decay)
            cases.append(dict(gen=gen_cfg_dict(g), digest=digest_ref(tr), layer=layer, window=window, gamma=gamma,
                              decay=decay, ids=ids, targets_hex=[float(v).hex() for v in tgt],
                              hist_hex=[float(v).hex() for v in hist],
                              topb=predict_topb(hist, min(tr.experts, 5))))
    # MLP predictor on a small trace (tolerance-level parity: BLAS order)
    g = TraceGenConfig(n_visual=30, n_text=6, layers=6, experts=8, k=2, cluster_support=4, visual_noise=0.2, seed=7)
    tr = generate_trace(g)
    plan = compress(tr, CompressionConfig(0.1, 0.5, 2.0, (0,)))
    model = init_model(8 + 2 * tr.embed_dim, 8, d_hidden=32, d_bottleneck=16, seed=3)
    mlp = moesim.MLPPredictor(model, tr, plan, 0.5)
    pri = [mlp.priorities(l).tolist() for l in range(1, tr.layers)]
    feats = [build_features(tr, plan, l, 0.5).concat().tolist() for l in range(1, tr.layers)]
    drift = [layer_drift(l, tr.embed_dim).tolist() for l in range(tr.layers)]
    mlp_case = dict(gen=gen_cfg_dict(g), digest=digest_ref(tr), alpha=0.1, beta=0.5, lam=2.0, prefix=[0],
                    w1=model.w1.tolist(), b1=model.b1.tolist(), w2=model.w2.tolist(), b2=model.b2.tolist(),
                    wo=model.wo.tolist(), bo=model.bo.tolist(), layers=list(range(1, tr.layers)),
                    features=feats, priorities=pri, drift=drift)
    tb = [dict(y=[0.1, 0.9, 0.5], b=2, out=predict_topb([0.1, 0.9, 0.5], 2)),
          dict(y=[0.5] * 4, b=3, out=predict_topb([0.5] * 4, 3))]
    return dict(cases=cases, mlp=mlp_case, topb=tb)


# ---------------------------------------------------------------------------
def cache_ops():
    out = []
    for seed, policy in ((1, "priority"), (2, "fifo"), (111, "priority")):
        rng = np.random.default_rng(seed)
        cache = ExpertCache(6, policy)
        ops = []
        keys = [ExpertRef(l, e) for l in range(3) for e in range(4)]
        for _ in range(3000):
            before = len(ops)
            r = float(rng.random())
            key = keys[int(rng.integers(len(keys)))]
            try:
                if r < 0.35:
                    pri = float(rng.choice([0.0, 0.5, 1.0, 0.25, math.inf]))
                    cls = [ResidencyClass.REQUIRED, ResidencyClass.SPECULATIVE][int(rng.integers(2))]
                    res = cache.request_load(key, pri, cls)
                    ops.append(["request", list(key), pri if math.isfinite(pri) else "inf", cls.value,
                                res.status.value, res.slab, list(res.evicted) if res.evicted else None])
                elif r < 0.55:
                    e = cache.entry(key)
                    if e is not None and e.state.value == "loading":
                        cache.complete_load(key, 1.0)
                        ops.append(["complete", list(key)])
                elif r < 0.7:
                    e = cache.entry(key)
                    if e is not None and e.state.value == "resident":
                        cache.mark_executed(key)
                        ops.append(["executed", list(key)])
                elif r < 0.8:
                    e = cache.entry(key)
                    if e is not None and e.state.value == "loading":
                        cache.cancel_load(key)
                        ops.append(["cancel", list(key)])
                else:
                    win = [list(k) for k in keys if rng.random() < 0.3]
                    pr = {tuple(k): float(rng.choice([0.1, 0.2, 0.7])) for k in keys if rng.random() < 0.5}
                    grace = int(rng.integers(0, 3))
                    cache.reclassify([ExpertRef(*k) for k in win], grace, {ExpertRef(*k): v for k, v in pr.items()})
                    ops.append(["reclassify", win, grace, [[list(k), v] for k, v in pr.items()]])
            except Exception as exc:  # noqa: BLE001
                ops.append(["error", type(exc).__name__])
            snap = sorted([[s.slab, list(s.key) if s.key else None, s.state.value, s.cls.value,
                            s.priority if math.isfinite(s.priority) else "inf"] for s in cache.slabs if s.key])
            if len(ops) > before:
                ops[-1].append(snap)
        out.append(dict(seed=seed, policy=policy, num_slabs=6, ops=ops, evictions=cache.evictions,
                        victim=cache.select_victim()))
    return out


# ---------------------------------------------------------------------------
def sim_cfg_dict(c: SimConfig) -> dict:
    d = asdict(c)
    for k, v in list(d.items()):
        if isinstance(v, float) and not math.isfinite(v):
            d[k] = "inf"
    return d


def engine_cases():
    out = []
    rng = np.random.default_rng(99)
    n = 0
    while n < 90:
        layers = int(rng.integers(2, 6))
        experts = int(rng.integers(2, 7))
        k = int(rng.integers(1, min(2, experts) + 1))
        decode = int(rng.integers(0, 3))
        g = TraceGenConfig(n_visual=int(rng.integers(1, 5)), n_text=int(rng.integers(1, 3)), layers=layers,
                           experts=experts, k=k, clusters=int(rng.integers(1, 3)),
                           cluster_support=int(rng.integers(k, experts + 1)), rho=float(rng.choice([0.3, 0.8, 1.0])),
                           visual_noise=float(rng.choice([0.0, 0.4])), seed=int(rng.integers(10_000)),
                           decode_steps=decode)
        kind = str(rng.choice(["none", "oracle", "history"]))
        cfg = SimConfig(
            bandwidth_mb_per_ms=1.0, expert_size_mb=float(rng.choice([0.5, 2.0, 10.0, 0.3])),
            gpu_ms_per_expert=float(rng.choice([0.0, 1.0, 3.0, 0.7])), l_pinned=int(rng.integers(1, 3)) if layers > 2 else 1,
            num_slabs=int(rng.integers(2 * k + 2, 12)), decode_steps=decode,
            predictor=PredictorSpec(kind=kind, budget=int(rng.choice([0, 1, 2, 4])), window=int(rng.integers(1, 4)),
                                    gamma=float(rng.choice([0.5, 0.8, 1.0])), history_decay=float(rng.choice([0.5, 0.3]))),
            speculative_grace=int(rng.integers(0, 3)), victim_policy=str(rng.choice(["priority", "fifo"])),
            compress_latency_ms=float(rng.choice([0.0, 1.7])), predictor_bootstrap_ms=float(rng.choice([0.0, 0.9])),
            event_log=True,
        )
        tr = generate_trace(g)
        use_c = bool(rng.random() < 0.5 and tr.visual_ids())
        cc = CompressionConfig(alpha=0.25, beta=0.75, prefix_layers=(0,)) if use_c else None
        reactive = bool(rng.random() < 0.25)
        plan = build_plan(tr, cfg, cc)
        try:
            rep = (simulate_reactive if reactive else simulate)(tr, plan, cfg)
            res = json.loads(rep.to_json())
            res["events"] = [list(e) for e in rep.events]
            err = None
        except SimulationError as exc:
            res, err = None, str(exc)
        out.append(dict(gen=gen_cfg_dict(g), digest=digest_ref(tr), sim=sim_cfg_dict(cfg),
                        compression=None if cc is None else dict(alpha=cc.alpha, beta=cc.beta, lam=cc.lam, prefix=list(cc.prefix_layers)),
                        reactive=reactive, report=res, error=err))
        n += 1
    # named workloads on the reference cost model (expert MB from bf16 bytes)
    for name in ("c1_tiny", "c2_phi2", "c4_dsvl2s", "c3_qwen3vl"):
        w = WORKLOADS[name]
        g = w.trace_config(seed=0, decode_steps=2)
        tr = generate_trace(g)
        cfg = SimConfig(bandwidth_mb_per_ms=55.0, expert_size_mb=w.expert_bytes / 1e6, gpu_ms_per_expert=0.01,
                        l_pinned=w.l_pinned, num_slabs=w.num_slabs, decode_steps=2, shared_experts=w.shared_experts,
                        predictor=PredictorSpec(kind=w.predictor, budget=w.budget, window=w.window, gamma=w.gamma,
                                                history_decay=w.history_decay), event_log=True)
        cc = CompressionConfig(w.alpha, w.beta, w.lam, w.prefix_layers)
        plan = build_plan(tr, cfg, cc)
        rep = simulate(tr, plan, cfg)
        res = json.loads(rep.to_json())
        res["events"] = [list(e) for e in rep.events]
        out.append(dict(name=name, gen=gen_cfg_dict(g), digest=digest_ref(tr), sim=sim_cfg_dict(cfg),
                        compression=dict(alpha=cc.alpha, beta=cc.beta, lam=cc.lam, prefix=list(cc.prefix_layers)),
                        reactive=False, report=res, error=None))
    return out


def main():
    def dump(name, obj):
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(obj, f, separators=(",", ":"))
        print(name, os.path.getsize(os.path.join(HERE, name)))

    dump("compress.json", compress_cases())
    dump("predict.json", predict_cases())
    dump("cache_ops.json", cache_ops())
    dump("engine.json", engine_cases())


if __name__ == "__main__":
    main()
