"""Device predictors: oracle targets / history histogram bit-exact, MLP within tolerance."""
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import predictor_ref
from paper_2605_05899_b200 import CompressionConfig, HistoryPredictor, MLPModel, MLPPredictor, OraclePredictor, compress
from paper_2605_05899_b200 import kernels
from paper_2605_05899_b200.trace import TraceGenConfig, generate_trace, trace_digest

pytestmark = pytest.mark.gpu


def regen(d, digest):
    d = dict(d)
    d["saliency_shape"] = tuple(d["saliency_shape"])
    tr = generate_trace(TraceGenConfig(**d))
    assert trace_digest(tr) == digest
    return tr


def test_targets_and_history_bit_exact():
    for c in load_golden("predict.json")["cases"]:
        tr = regen(c["gen"], c["digest"])
        o = OraclePredictor(tr, c["ids"], c["window"], c["gamma"])
        assert [v.hex() for v in o.priorities(c["layer"], c["ids"]).tolist()] == c["targets_hex"]
        h = HistoryPredictor(tr, c["ids"], c["decay"])
        y = h.priorities(c["layer"], c["ids"])
        assert [v.hex() for v in y.tolist()] == c["hist_hex"]
        assert h.predict(c["layer"], min(tr.experts, 5), c["ids"]) == c["topb"]


def test_history_batched_table_matches_single_calls_c3_scale():
    tr = generate_trace(TraceGenConfig(n_visual=600, n_text=64, layers=48, experts=128, k=8, visual_noise=0.3, seed=2))
    ids = list(range(0, 664, 2))
    h = HistoryPredictor(tr, ids, 0.3)
    table = h.device_table(list(range(8, 47)), ids).cpu().numpy()
    pt = [0.3 ** j for j in range(49)]
    for row, layer in zip(table, range(8, 47)):
        ref = predictor_ref.history_histogram(tr.route_experts, layer, np.asarray(ids), 128, pt)
        assert row.tolist() == ref.tolist()


def test_mlp_predictor_features_exact_outputs_tolerance():
    m = load_golden("predict.json")["mlp"]
    tr = regen(m["gen"], m["digest"])
    plan = compress(tr, CompressionConfig(m["alpha"], m["beta"], m["lam"], tuple(m["prefix"])))
    model = MLPModel(*(np.asarray(m[k], dtype=np.float64) for k in ("w1", "b1", "w2", "b2", "wo", "bo")))
    pred = MLPPredictor(model, tr, plan, 0.5)
    y, feat = pred.device_table(m["layers"], want_features=True)
    np.testing.assert_array_equal(feat.cpu().numpy(), np.asarray(m["features"]))
    # BLAS order differs from the sequential device dot products: tolerance
    np.testing.assert_allclose(y.cpu().numpy(), np.asarray(m["priorities"]), rtol=1e-12, atol=1e-14)


def test_gate_lookahead_exact_on_integer_inputs():
    g = torch.Generator().manual_seed(0)
    x = torch.randint(-4, 5, (300, 512), generator=g).to(torch.bfloat16)
    w = torch.randint(-1, 2, (64, 512), generator=g).to(torch.bfloat16)
    y = kernels.gate_lookahead(x.cuda(), w.cuda(), 6).cpu().numpy()
    ref = predictor_ref.gate_lookahead(x.float().numpy(), w.float().numpy(), 6)
    assert y.tolist() == ref.tolist()


def test_a4_oracle_recall_perfect():
    """Reference acceptance A4 (pkg/tests/test_acceptance.py:153-178): the device oracle's
    top-B reaches hot recall exactly 1.0 whenever the budget covers the next layer's set."""
    from paper_2605_05899_b200.predictor import OraclePredictor

    checked = 0
    for seed in range(12):
        tr = generate_trace(TraceGenConfig(n_visual=10, n_text=4, layers=8, experts=24, k=2, clusters=3,
                                           cluster_support=6, rho=[0.0, 0.5, 0.9, 1.0][seed % 4],
                                           visual_noise=[0.0, 0.3][seed % 2], seed=seed))
        ids = tr.prefill_ids()
        o = OraclePredictor(tr, ids, window=5, gamma=0.8)
        for layer in range(tr.layers - 1):
            actual = tr.active_union(layer + 1, ids)
            for budget in (len(actual), len(actual) + 3, tr.experts):
                if budget > tr.experts:
                    continue
                picks = set(o.predict(layer, budget))
                assert actual <= picks
                checked += 1
    assert checked > 100
