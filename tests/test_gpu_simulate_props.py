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
