"""Oracle harness: the reference's build_plan + simulate wiring, restated.

Glue between the oracle restatements (compress, predictors, engine) that
mirrors `pkg/src/moesim/pipeline.py:173-226` (predictor construction, plan)
and `pipeline.py:768-776` (simulate / simulate_reactive).  Takes plain dicts so
golden fixtures and product-side configs can drive it identically.
"""
from __future__ import annotations

import math

import numpy as np

from . import compress_ref, engine_ref, predictor_ref


def _f(v):
    return math.inf if v == "inf" else float(v)


def decay_table(gamma: float, n: int) -> list[float]:
    # python float pow, exactly as the reference evaluates gamma ** (d - 1)
    return [gamma ** (d - 1) for d in range(1, n + 1)]


def pow_table(decay: float, n: int) -> list[float]:
    return [decay ** j for j in range(n + 1)]


def plan_and_scores(trace, sim: dict, compression: dict | None, y_override=None):
    """-> (retained ids, compress result or None, scores callback or None)."""
    comp = None
    if compression is not None:
        comp = compress_ref.compress(
            trace.saliency, trace.modality, trace.phase_marks, trace.route_experts, trace.experts,
            compression["alpha"], compression["beta"], compression["lam"], compression["prefix"],
        )
        retained = comp["retained"]
    else:
        retained = np.asarray(trace.prefill_ids(), dtype=np.int64)
    p = sim["predictor"]
    kind = p["kind"]
    E, L = trace.experts, trace.layers
    if y_override is not None:
        scores = y_override
    elif kind == "none":
        scores = None
    elif kind == "oracle":
        dt = decay_table(float(p["gamma"]), int(p["window"]))

        def scores(ctx, ids):
            return predictor_ref.oracle_targets(trace.route_experts, L, ctx, int(p["window"]), dt,
                                                np.asarray(ids, dtype=np.int64), E)
    elif kind == "history":
        pt = pow_table(float(p["history_decay"]), L)

        def scores(ctx, ids):
            return predictor_ref.history_histogram(trace.route_experts, ctx, np.asarray(ids, dtype=np.int64), E, pt)
    else:
        raise ValueError(f"oracle harness: unsupported predictor kind {kind}")
    return retained, comp, scores


def simulate(trace, sim: dict, compression: dict | None, reactive: bool, y_override=None, retained=None):
    """`retained` overrides the compressed token set (a batch of requests each
    compressed on its own, merged into one trace: ExecutionPlan with a prebuilt
    compression, pipeline.py:153-170)."""
    ret0, comp, scores = plan_and_scores(trace, sim, compression if retained is None else None, y_override)
    if retained is not None:
        ret0 = np.asarray(retained, dtype=np.int64)
        comp = {"retained": ret0} if compression is not None else None
    retained = ret0
    p = sim["predictor"]
    prefetching = (scores is not None) and int(p["budget"]) > 0 and not reactive
    l_pinned = int(sim["l_pinned"]) if sim.get("l_pinned") is not None else int(sim.get("l_semantic", 1))
    cfg = dict(
        transfer_ms=_f(sim["expert_size_mb"]) / _f(sim["bandwidth_mb_per_ms"]),
        gpu_ms=_f(sim["gpu_ms_per_expert"]),
        num_slabs=int(sim["num_slabs"]),
        fifo=sim["victim_policy"] == "fifo",
        grace=int(sim["speculative_grace"]),
        budget=int(p["budget"]),
        window=int(p["window"]),
        decay_table=decay_table(float(p["gamma"]), int(p["window"])),
        l_pinned=l_pinned,
        shared=int(sim.get("shared_experts", 0)) or int(trace.shared_experts),
        prefetching=prefetching,
        reactive=reactive,
        compress_ms=_f(sim["compress_latency_ms"]) if comp is not None else 0.0,
        bootstrap_ms=_f(sim["predictor_bootstrap_ms"]),
        event_log=bool(sim.get("event_log", False)),
    )
    L, E = trace.layers, trace.experts
    re = trace.route_experts
    prefill_all = np.asarray(trace.prefill_ids(), dtype=np.int64)

    def dset(layer, ids):
        return set(np.flatnonzero(predictor_ref.demand_counts(re, layer, ids, E)).tolist())

    prefill_demand = [dset(l, retained) if l >= l_pinned else None for l in range(L)]
    pinned_demand = [dset(l, prefill_all) if l < l_pinned else None for l in range(L)]
    dec_tokens = trace.phase_marks[: int(sim.get("decode_steps", 0))]
    dec_demand = [[set(int(e) for e in re[l, t]) for l in range(L)] for t in dec_tokens]
    rep = engine_ref.Replay(L, E, cfg, scores if prefetching else None)
    return rep.run(prefill_demand, pinned_demand, retained.tolist(), dec_tokens, dec_demand)
