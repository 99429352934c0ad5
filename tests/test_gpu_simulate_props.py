"""The reference's engine invariants (pkg/tests/test_pipeline.py:188-250),
restated against simulate()/simulate_reactive() on the device + native engine."""
import math

import pytest

from paper_2605_05899_b200 import CompressionConfig, PredictorSpec, SimConfig, build_plan, simulate, simulate_reactive
from paper_2605_05899_b200.trace import TraceGenConfig, generate_trace

pytestmark = pytest.mark.gpu


def gen_trace(seed=0, **kw):
    base = dict(n_visual=12, n_text=4, layers=7, experts=20, k=2, clusters=3, cluster_support=5, rho=0.8,
                visual_noise=0.2, seed=seed, decode_steps=2)
    base.update(kw)
    return generate_trace(TraceGenConfig(**base))


def bare_cfg(**overrides):
    base = dict(bandwidth_mb_per_ms=1.0, expert_size_mb=10.0, gpu_ms_per_expert=2.0, l_pinned=1, num_slabs=8,
                predictor=PredictorSpec(kind="none"), compress_latency_ms=0.0, predictor_bootstrap_ms=0.0)
    base.update(overrides)
    return SimConfig(**base)


def total_needs(trace, plan, cfg):
    tokens = plan.retained_ids(trace)
    needs = sum(len(trace.active_union(l, tokens)) for l in range(plan.l_pinned, trace.layers))
    for tok in trace.phase_marks[: cfg.decode_steps]:
        needs += sum(len(trace.route_set(l, tok)) for l in range(plan.l_pinned, trace.layers))
    return needs


@pytest.mark.parametrize("kind,budget", [("none", 0), ("oracle", 6), ("history", 6)])
def test_work_conservation(kind, budget):
    """test_pipeline.py:212-222: every need is a hit or a miss; misses split into on-demand
    transfers and in-flight waits (no CPU dispatch path here)."""
    trace = gen_trace(seed=11)
    cfg = bare_cfg(num_slabs=24, decode_steps=2, predictor=PredictorSpec(kind=kind, budget=budget))
    plan = build_plan(trace, cfg, CompressionConfig(alpha=0.1, beta=0.5))
    r = simulate(trace, plan, cfg)
    assert r.hits + r.misses == total_needs(trace, plan, cfg)
    assert r.misses == r.on_demand_transfers + r.cpu_dispatches + r.inflight_waits


def test_infinite_bandwidth_makespan_equals_compute():
    """test_pipeline.py:225-234."""
    trace = gen_trace(seed=3)
    cfg = bare_cfg(bandwidth_mb_per_ms=math.inf, num_slabs=140, decode_steps=2,
                   predictor=PredictorSpec(kind="oracle", budget=6))
    plan = build_plan(trace, cfg)
    r = simulate(trace, plan, cfg)
    assert r.makespan == r.total_compute
    rr = simulate_reactive(trace, plan, cfg)
    assert rr.makespan == rr.total_compute


def test_lower_bounds_and_overlap_identity():
    """test_pipeline.py:237-250."""
    for seed in range(6):
        trace = gen_trace(seed=seed)
        cfg = bare_cfg(num_slabs=24, decode_steps=2, predictor=PredictorSpec(kind="history", budget=5))
        plan = build_plan(trace, cfg, CompressionConfig(alpha=0.1, beta=0.6))
        for r in (simulate(trace, plan, cfg), simulate_reactive(trace, plan, cfg)):
            assert r.makespan >= r.total_compute
            if r.total_transfer > 0:
                assert r.makespan >= cfg.transfer_ms
            assert r.exposed_transfer + r.overlapped_transfer == r.total_transfer
            assert 0.0 <= r.exposed_transfer <= r.total_transfer


def test_a6_ablation_ordering():
    """Reference acceptance A6 (pkg/tests/test_acceptance.py:209-246), with the four stacked
    configurations of pipeline.py:793-829 built from simulate()/simulate_reactive(): on 20
    clustered 48x128x8 traces in a bandwidth-bound config, makespans are monotone
    base >= +compression >= +prediction >= full and the full mean is <= 0.7x the base mean."""
    from dataclasses import replace

    base_spans, full_spans = [], []
    for seed in range(20):
        tr = generate_trace(TraceGenConfig(n_visual=64, n_text=16, layers=48, experts=128, k=8, clusters=4,
                                           cluster_support=16, rho=0.85, visual_noise=0.3, seed=seed,
                                           decode_steps=4))
        cfg = SimConfig(bandwidth_mb_per_ms=17.3 / 8.0, expert_size_mb=17.3, gpu_ms_per_expert=2.0, l_pinned=4,
                        num_slabs=256, decode_steps=4, predictor=PredictorSpec(kind="oracle", budget=20, window=5))
        ccfg = CompressionConfig(alpha=0.1, beta=0.5, lam=2.0, prefix_layers=(0, 1, 2, 3))
        base_cfg = replace(cfg, compress_latency_ms=0.0, predictor_bootstrap_ms=0.0)
        b = simulate_reactive(tr, build_plan(tr, replace(base_cfg, predictor=PredictorSpec(kind="none"))),
                              base_cfg).makespan
        comp_cfg = replace(cfg, predictor_bootstrap_ms=0.0)
        c = simulate_reactive(tr, build_plan(tr, replace(comp_cfg, predictor=PredictorSpec(kind="none")), ccfg),
                              comp_cfg).makespan
        pred_cfg = replace(cfg, speculative_grace=0, victim_policy="fifo")
        p = simulate(tr, build_plan(tr, pred_cfg, ccfg), pred_cfg).makespan
        f = simulate(tr, build_plan(tr, cfg, ccfg), cfg).makespan
        assert b >= c >= p >= f, (seed, b, c, p, f)
        base_spans.append(b)
        full_spans.append(f)
    assert sum(full_spans) / len(full_spans) <= 0.7 * sum(base_spans) / len(base_spans)
