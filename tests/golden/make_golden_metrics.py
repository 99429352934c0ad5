"""Golden vectors for the routing diagnostics, made by the REAL reference
(`moesim.metrics`).  Build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_metrics.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from moesim import TraceGenConfig, generate_trace  # noqa: E402  (reference)
from moesim.metrics import affinity_report  # noqa: E402

from paper_2605_05899_b200.trace import RoutingTrace as MyTrace, trace_digest  # noqa: E402


def gen_dict(c):
    from dataclasses import asdict

    d = asdict(c)
    d["saliency_shape"] = list(d["saliency_shape"])
    return d


def main():
    cases = []
    specs = [
        dict(n_visual=576, n_text=64, layers=8, experts=8, k=2, cluster_support=4, visual_noise=0.3, seed=0),
        dict(n_visual=300, n_text=20, layers=12, experts=64, k=6, seed=5),
        dict(n_visual=2304, n_text=64, layers=48, experts=128, k=8, visual_noise=0.3, seed=1),
        dict(n_visual=40, n_text=8, layers=5, experts=16, k=4, seed=9, visual_noise=1.0),
    ]
    rng = np.random.default_rng(31)
    for spec in specs:
        g = TraceGenConfig(**spec)
        tr = generate_trace(g)
        n = tr.num_tokens
        subsets = {
            "visual": tr.visual_ids(),
            "all": list(range(n)),
            "random": sorted(rng.choice(n, size=max(1, n // 7), replace=False).tolist()),
            "dups": [0, 0, 1, min(2, n - 1)],
        }
        for name, sub in subsets.items():
            for top in (0, 1, min(5, tr.experts), tr.experts):
                rep = affinity_report(tr, sub, top)
                cases.append(dict(gen=gen_dict(g), digest=trace_digest(MyTrace.from_reference(tr)), subset=name,
                                  ids=[int(t) for t in sub], top=top,
                                  working_set=rep.per_layer_working_set,
                                  coverage=[float(v).hex() for v in rep.topk_coverage],
                                  similarity=[float(v).hex() for v in rep.interlayer_similarity],
                                  jaccard=[float(v).hex() for v in rep.interlayer_jaccard],
                                  means=[float(rep.mean_working_set).hex(), float(rep.mean_coverage).hex(),
                                         float(rep.mean_similarity).hex()]))
    with open(os.path.join(HERE, "metrics.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
    print("metrics.json", os.path.getsize(os.path.join(HERE, "metrics.json")), len(cases))


if __name__ == "__main__":
    main()
