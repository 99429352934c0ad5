"""The drop-ins run INSIDE the unmodified reference engine.

INTEGRATION.md §1-§3 verbatim: `moesim.pipeline.ExpertCache = ExpertCache`
(native policy), `moesim.pipeline.compress = compress` (device prune) and the
device predictors as `plan.predictor`, each checked by running
`moesim.simulate` / `moesim.simulate_reactive` and requiring the report
(every counter, the per-layer timeline and the event log) to be identical to
the stock reference run.  Scenario generator restated from the reference's
`build_scenario` (pkg/tests/test_pipeline.py:369-414) plus C1-shaped cases
with real eviction pressure.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from moesim_loader import load_moesim

moesim = load_moesim()
pytestmark = pytest.mark.skipif(moesim is None, reason="reference package moesim not importable")


def _scenario(rng):
    """pkg/tests/test_pipeline.py:369-414 (tiny random scenario)."""
    m = moesim
    layers = int(rng.integers(2, 5))
    experts = int(rng.integers(2, 5))
    k = int(rng.integers(1, min(2, experts) + 1))
    decode = int(rng.integers(0, 3))
    trace = m.generate_trace(m.TraceGenConfig(
        n_visual=int(rng.integers(1, 4)), n_text=int(rng.integers(1, 3)), layers=layers, experts=experts, k=k,
        clusters=int(rng.integers(1, 3)), cluster_support=int(rng.integers(k, experts + 1)),
        rho=float(rng.choice([0.3, 0.8, 1.0])), visual_noise=float(rng.choice([0.0, 0.4])),
        seed=int(rng.integers(10_000)), decode_steps=decode))
    kind = str(rng.choice(["none", "oracle", "history", "random"]))
    budget = int(rng.choice([0, 1, 2, 4]))
    cfg = m.SimConfig(
        bandwidth_mb_per_ms=1.0, expert_size_mb=float(rng.choice([0.5, 2.0, 10.0])),
        gpu_ms_per_expert=float(rng.choice([0.0, 1.0, 3.0])), l_pinned=1,
        num_slabs=int(rng.integers(2 * k + 2, 10)), decode_steps=decode,
        predictor=m.PredictorSpec(kind=kind, budget=budget, window=int(rng.integers(1, 4)),
                                  gamma=float(rng.choice([0.5, 0.8, 1.0]))),
        seed=int(rng.integers(100)), speculative_grace=int(rng.integers(0, 2)),
        victim_policy=str(rng.choice(["priority", "fifo"])), compress_latency_ms=float(rng.choice([0.0, 1.7])),
        predictor_bootstrap_ms=float(rng.choice([0.0, 0.9])), event_log=True)
    ccfg = (m.CompressionConfig(alpha=0.25, beta=0.75, prefix_layers=(0,))
            if rng.random() < 0.5 and trace.visual_ids() else None)
    return trace, cfg, ccfg, bool(rng.random() < 0.3)


def _c1_scenario(seed, kind="oracle", slabs=24):
    """C1 shape (BASELINE configs[0]): 576+64 tokens, 8 experts top-2, 8 layers, tight cache."""
    m = moesim
    trace = m.generate_trace(m.TraceGenConfig(n_visual=576, n_text=64, layers=8, experts=8, k=2,
                                              cluster_support=4, visual_noise=0.3, seed=seed, decode_steps=2))
    cfg = m.SimConfig(bandwidth_mb_per_ms=4.0, expert_size_mb=0.79, gpu_ms_per_expert=0.05, l_pinned=2,
                      num_slabs=slabs, decode_steps=2, victim_policy="priority" if seed % 2 == 0 else "fifo",
                      predictor=m.PredictorSpec(kind=kind, budget=4, window=3), event_log=True)
    return trace, cfg, m.CompressionConfig(alpha=0.05, beta=0.25, prefix_layers=(0, 1)), False


def _report(trace, cfg, ccfg, reactive, plan=None):
    m = moesim
    try:
        plan = plan or m.build_plan(trace, cfg, ccfg)
        rep = (m.simulate_reactive if reactive else m.simulate)(trace, plan, cfg)
    except m.SimulationError as exc:  # both sides must fail the same way
        return ("SimulationError", str(exc))
    return rep.to_dict(), rep.events, rep.timeline_csv()


def _cases(n_tiny=60):
    rng = np.random.default_rng(2024)  # test_pipeline.py:451 sample seed
    cases = [_scenario(rng) for _ in range(n_tiny)]
    cases += [_c1_scenario(s, kind) for s in range(4) for kind in ("oracle", "history")]
    return cases


def test_native_expert_cache_inside_moesim_engine(monkeypatch):
    """moesim.pipeline.ExpertCache = ExpertCache."""
    from paper_2605_05899_b200 import ExpertCache

    cases = _cases()
    want = [_report(*c) for c in cases]
    monkeypatch.setattr(moesim.pipeline, "ExpertCache", ExpertCache)
    got = [_report(*c) for c in cases]
    assert sum(1 for w in want if w[0] != "SimulationError") >= 40
    evicting = sum(1 for w in want if w[0] != "SimulationError" and any(e[1] == "evict" for e in w[1]))
    assert evicting >= 5, "scenarios must exercise eviction"
    for i, (w, g) in enumerate(zip(want, got)):
        assert g == w, f"case {i}"


def test_native_cache_returns_the_callers_enum_members():
    from paper_2605_05899_b200 import ExpertCache
    from paper_2605_05899_b200 import cache as own

    ref = moesim.cache
    c = ExpertCache(4, "priority", enums=ref)
    key = moesim.ExpertRef(3, 1)
    assert c.lookup(key).status is ref.LookupStatus.MISS
    r = c.request_load(key, math.inf, ref.ResidencyClass.REQUIRED)
    assert r.status is ref.RequestStatus.ENQUEUED and r.slab == 0
    assert c.entry(key).state is ref.SlabState.LOADING and c.entry(key).cls is ref.ResidencyClass.REQUIRED
    c.set_ready(key, 2.0)
    c.complete_load(key, 2.0)
    assert c.lookup(key) == (ref.LookupStatus.HIT, 2.0)
    assert c.slabs[0].state is ref.SlabState.RESIDENT
    # this package's own enums still work, and are the default outside moesim
    c2 = ExpertCache(2)
    assert c2.lookup((0, 0)).status is own.LookupStatus.MISS
    assert c2.request_load((0, 0), 1.0, ref.ResidencyClass.SPECULATIVE).status is own.RequestStatus.ENQUEUED


@pytest.mark.gpu
def test_device_compress_inside_moesim_build_plan(monkeypatch):
    """moesim.pipeline.compress = compress (device prune, reference config object)."""
    from paper_2605_05899_b200 import compress

    cases = [c for c in _cases(40) if c[2] is not None]
    want = [(_report(*c), moesim.compress(c[0], c[2])) for c in cases]
    monkeypatch.setattr(moesim.pipeline, "compress", compress)
    for i, (c, (w, wp)) in enumerate(zip(cases, want)):
        gp = compress(c[0], c[2])  # reference RoutingTrace + reference CompressionConfig
        assert (gp.core, gp.keep, gp.target_experts) == (wp.core, wp.keep, wp.target_experts), i
        assert gp.delta == wp.delta and gp.score == wp.score and gp.saliency_norm == wp.saliency_norm, i
        assert gp.retained_ids(c[0]) == wp.retained_ids(c[0])
        assert _report(*c) == w, f"case {i}"


@pytest.mark.gpu
def test_device_predictors_and_all_dropins_inside_moesim(monkeypatch):
    """INTEGRATION.md §2 (+ §1, §3 at once): device Oracle/History predictors as
    plan.predictor on reference plans; reports identical to stock moesim."""
    from paper_2605_05899_b200 import ExpertCache, HistoryPredictor, OraclePredictor, compress

    cases = [c for c in _cases(40) if c[1].predictor.kind in ("oracle", "history") and c[1].predictor.budget > 0]
    assert len(cases) >= 10
    want = [_report(*c) for c in cases]

    def device_plan(trace, cfg, ccfg):
        plan = moesim.build_plan(trace, cfg, ccfg)
        ids = plan.retained_ids(trace)
        spec = cfg.predictor
        plan.predictor = (OraclePredictor(trace, ids, spec.window, spec.gamma) if spec.kind == "oracle"
                          else HistoryPredictor(trace, ids, spec.history_decay))
        return plan

    for i, c in enumerate(cases):
        assert _report(*c, plan=device_plan(*c[:3])) == want[i], f"predictor case {i}"
    monkeypatch.setattr(moesim.pipeline, "compress", compress)
    monkeypatch.setattr(moesim.pipeline, "ExpertCache", ExpertCache)
    for i, c in enumerate(cases):
        assert _report(*c, plan=device_plan(*c[:3])) == want[i], f"all drop-ins case {i}"


@pytest.mark.gpu
def test_device_mlp_predictor_on_reference_objects():
    """MLP predictor (predictor.py:521-550) built from the reference's own model and plan."""
    from paper_2605_05899_b200 import MLPPredictor

    m = moesim
    trace, cfg, ccfg, _ = _c1_scenario(3)
    plan = m.build_plan(trace, m.SimConfig(l_pinned=2, num_slabs=24, predictor=m.PredictorSpec(kind="none")), ccfg)
    d_in = trace.experts + 2 * trace.embed_dim
    model = m.predictor.init_model(d_in, trace.experts, seed=5)  # predictor.py:257-280
    ref = m.MLPPredictor(model, trace, plan.compression, 0.5)
    dev = MLPPredictor(model, trace, plan.compression, 0.5)
    ids = plan.retained_ids(trace)
    for layer in range(1, trace.layers - 1):
        np.testing.assert_allclose(dev.priorities(layer, ids), ref.priorities(layer, ids), rtol=1e-12, atol=0)


def test_reference_trace_is_accepted_by_the_device_upload_cache(monkeypatch):
    """moesim.RoutingTrace is unhashable (__eq__ without __hash__, trace.py:66,135):
    the upload cache keys by object identity instead."""
    import gc

    from paper_2605_05899_b200 import device_trace as dtm
    from paper_2605_05899_b200.trace import RoutingTrace

    made = []

    class Stub:
        def __init__(self, tr):
            assert isinstance(tr, RoutingTrace)
            made.append(tr)

    monkeypatch.setattr(dtm, "DeviceTrace", Stub)
    tr = _c1_scenario(0)[0]
    with pytest.raises(TypeError):
        hash(tr)
    a = dtm.device_trace(tr)
    assert dtm.device_trace(tr) is a and len(made) == 1  # cached per object
    conv = made[0]
    assert np.array_equal(conv.route_experts, tr.route_experts) and conv.visual_ids() == tr.visual_ids()
    key = id(tr)
    del tr, a
    gc.collect()
    assert key not in dtm._CACHE  # dropped with the trace
