"""Hot recall of the lookahead predictors (hot_recall,
pkg/src/moesim/predictor.py:443-450): the fraction of layer l+1's activated
experts that are in the predictor's top-B at context l, for B = 10 / 20 / 30.

Part A -- the reference's own acceptance protocol A7 (pkg/tests/
test_acceptance.py:249-279: 20 seeds of rho=0.8 / visual_noise=0.3 traces,
24+6 tokens, 24 layers, 128 experts top-3, compression alpha .1 / beta .5 on
prefix (0, 1), recall over the retained tokens, layers 2..L-2).  Predictors
run on the device: oracle, history, MLP (weights trained OFFLINE with the
reference's own trainer, moesim.predictor.train -- the paper trains its
predictor offline; training is out of scope for the device
path) and the seeded random baseline.

Part B -- the live stack on synthetic hidden states with inter-layer
affinity (C3 shape: router gates of consecutive layers correlated by
router_corr=0.8, hidden states carried by the residual stream through the
MoE layers, decode tokens an AR(1) sequence): per decode token and emitting
layer, top-B of the recorded lookahead scores against the token's routed
experts at l+1 (k=8 of 128).  gate (W_g^{l+1} applied to h_l), history
(decayed routing histogram), random (B/E).

    python tools/predictor_recall.py [D] > profiles/r02_predictor_recall.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

BUDGETS = (10, 20, 30)


def load_moesim():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if os.path.isdir(p):
        sys.path.insert(0, p)
    import moesim
    return moesim


def part_a(seeds=20):
    m = load_moesim()
    from paper_2605_05899_b200 import (CompressionConfig, HistoryPredictor, MLPPredictor, OraclePredictor,
                                       RandomPredictor, compress, hot_recall)
    from paper_2605_05899_b200.trace import RoutingTrace

    rec = {p: {b: [] for b in BUDGETS} for p in ("oracle", "history", "mlp", "random")}
    for seed in range(seeds):
        rtr = m.generate_trace(m.TraceGenConfig(n_visual=24, n_text=6, layers=24, experts=128, k=3, clusters=3,
                                                cluster_support=6, rho=0.8, visual_noise=0.3, seed=seed))
        tr = RoutingTrace.from_reference(rtr)
        ccfg = CompressionConfig(alpha=0.1, beta=0.5, prefix_layers=(0, 1))
        plan = compress(tr, ccfg)  # device prune
        rplan = m.compress(rtr, m.CompressionConfig(alpha=0.1, beta=0.5, prefix_layers=(0, 1)))
        assert plan.keep == rplan.keep
        tokens = plan.retained_ids(tr)
        data = m.build_dataset(rtr, rplan, range(1, rtr.layers - 1))
        model = m.train(data, m.TrainConfig(learning_rate=0.1, epochs=300, batch_size=8, seed=seed))
        preds = dict(oracle=OraclePredictor(tr, tokens), history=HistoryPredictor(tr, tokens),
                     mlp=MLPPredictor(model, tr, plan), random=RandomPredictor(tr.experts, seed=seed))
        for name, p in preds.items():
            for b in BUDGETS:
                p.reset()
                rec[name][b].append(float(np.mean([hot_recall(p.predict(l, b, tokens), tr, l, tokens)
                                                   for l in range(2, tr.layers - 1)])))
    return {name: {f"B={b}": float(np.mean(v)) for b, v in r.items()} for name, r in rec.items()}


def part_b(D=24):
    from paper_2605_05899_b200.configs import WORKLOADS
    from paper_2605_05899_b200.moe import ExpertStore, MoEStack, StackConfig
    from paper_2605_05899_b200.trace import generate_trace

    w = WORKLOADS["c3_qwen3vl"]
    tr = generate_trace(w.trace_config(seed=0))
    T = tr.num_tokens
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((T, w.hidden), generator=g, device="cuda").to(torch.bfloat16)
    sal = torch.from_numpy(tr.saliency).cuda()
    mod = torch.from_numpy(tr.device_modality()).cuda()
    toks, t = [], torch.randn((1, w.hidden), generator=g, device="cuda")
    for _ in range(D):  # AR(1) decode-token inputs
        toks.append(t.to(torch.bfloat16))
        t = 0.9 * t + (1 - 0.81) ** 0.5 * torch.randn((1, w.hidden), generator=g, device="cuda")
    store, out, routes_ref = None, {}, None
    rng = np.random.default_rng(0)
    for pred in ("gate", "history"):
        cfg = StackConfig.from_workload(w, routing="live", predictor=pred)
        store = store or ExpertStore(cfg, seed=1000)
        stack = MoEStack(cfg, store=store)
        stack.forward(x, sal, mod, keep_session=True)
        hits = {b: [] for b in BUDGETS}
        rnd = {b: [] for b in BUDGETS}
        routes_all = []
        for tk in toks:
            r = stack.decode_step(tk, record=True)
            routes = [set(int(e) for e in rt.cpu().numpy().ravel()) for rt in r.routes]
            routes_all.append(routes)
            for ctx, y in r.scores.items():
                if ctx + 1 >= w.layers:
                    continue
                actual = routes[ctx + 1]
                order = np.lexsort((np.arange(len(y)), -np.asarray(y)))  # predict_topb (predictor.py:434-440)
                for b in BUDGETS:
                    top = set(int(e) for e in order[:b] if y[e] > 0)
                    hits[b].append(len(top & actual) / len(actual))
                    rnd[b].append(len(set(rng.choice(w.experts, b, replace=False).tolist()) & actual) / len(actual))
        stack.end_session()
        if routes_ref is None:
            routes_ref = routes_all
        assert routes_all == routes_ref  # live routing does not depend on the predictor
        out[pred] = {f"B={b}": float(np.mean(v)) for b, v in hits.items()}
        out["random"] = {f"B={b}": float(np.mean(v)) for b, v in rnd.items()}
    out["oracle"] = {f"B={b}": 1.0 for b in BUDGETS}  # top-B of the exact next-layer set, B >= k
    return out


def main():
    D = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    res = {"metric": "hot recall (PAPER.md:696, predictor.py:443-450)", "budgets": list(BUDGETS),
           "paper": {"VisMMOE predictor": {"B=10": 0.641, "B=20": 0.819, "B=30": 0.898},
                     "random": {"B=10": 0.078, "B=30": 0.234}},
           "part_a_reference_protocol_A7": part_a(),
           "part_b_live_stack_decode_c3": {"decode_tokens": D, **part_b(D)}}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
