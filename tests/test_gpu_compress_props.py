"""The reference's compress() property tests (pkg/tests/test_compress.py:103-222),
restated against the device path (vmm_prune behind `compress`)."""
import math

import numpy as np
import pytest

from paper_2605_05899_b200 import CompressionConfig, compress
from paper_2605_05899_b200.trace import MOD_TEXT, MOD_VISUAL, RoutingTrace, TraceGenConfig, generate_trace

pytestmark = pytest.mark.gpu


def _active(trace, tok, layers):
    return {int(e) for l in layers for e in trace.route_experts[l, tok]}


def _hand(sal, routes, experts, k, modality):
    routes = np.asarray(routes, dtype=np.int64)
    n = routes.shape[1]
    return RoutingTrace(routes.shape[0], experts, k, routes, np.full(routes.shape, 1.0 / k), np.asarray(sal, float),
                        np.asarray(modality, np.uint8), np.zeros((n, 1)))


def test_budget_exactness_and_core_subset():
    """test_compress.py:128-145: |keep| = floor(beta N_v), |core| = floor(alpha N_v), core in keep,
    target experts within the kept tokens' prefix experts."""
    for seed in range(30):
        tr = generate_trace(TraceGenConfig(n_visual=17, n_text=5, layers=4, experts=12, k=2, clusters=3,
                                           cluster_support=5, visual_noise=0.2, seed=seed))
        cfg = CompressionConfig(alpha=0.23, beta=0.61, prefix_layers=(0, 1))
        p = compress(tr, cfg)
        assert len(p.keep) == math.floor(0.61 * 17) and len(p.core) == math.floor(0.23 * 17)
        assert set(p.core) <= set(p.keep)
        union = set()
        for t in p.keep:
            union |= _active(tr, t, cfg.prefix_layers)
        assert p.target_experts <= union


def test_text_tokens_always_retained_excluded_from_budget():
    """test_compress.py:147-160."""
    mod = [MOD_VISUAL] * 4 + [MOD_TEXT] * 2
    tr = _hand([5, 4, 3, 2, 0, 0], [[[0], [1], [2], [3], [0], [1]]], 4, 1, mod)
    p = compress(tr, CompressionConfig(alpha=0.25, beta=0.5))
    assert len(p.keep) == 2 and set(p.keep) <= {0, 1, 2, 3}
    assert p.retained_ids(tr) == sorted(set(p.keep) | {4, 5})


def test_beta_one_keeps_all_visual():
    """test_compress.py:120-126."""
    tr = generate_trace(TraceGenConfig(n_visual=40, n_text=6, layers=3, experts=16, k=2, seed=3))
    p = compress(tr, CompressionConfig(alpha=0.1, beta=1.0, prefix_layers=(0, 1)))
    assert p.keep == list(range(40))


def test_lambda_zero_reduces_to_saliency_pruning():
    """test_compress.py:103-118: lam = 0 keeps the top-K_keep tokens by (saliency desc, id asc)."""
    for seed in range(10):
        tr = generate_trace(TraceGenConfig(n_visual=64, n_text=8, layers=4, experts=16, k=2, seed=seed))
        cfg = CompressionConfig(alpha=0.1, beta=0.4, lam=0.0, prefix_layers=(0, 1, 2))
        p = compress(tr, cfg)
        s = tr.saliency[:64]
        order = sorted(range(64), key=lambda i: (-s[i], i))[: math.floor(0.4 * 64)]
        assert p.keep == sorted(order)


def test_core_always_kept_for_every_lambda():
    """test_compress.py:211-222 (monotone non-expansion): the salient core is kept, and the keep set
    has its exact budget, for every lambda."""
    tr = generate_trace(TraceGenConfig(n_visual=96, n_text=8, layers=4, experts=32, k=2, seed=7))
    for lam in (0.0, 0.25, 1.0, 4.0):
        p = compress(tr, CompressionConfig(alpha=0.1, beta=0.5, lam=lam, prefix_layers=(0, 1)))
        assert set(p.core) <= set(p.keep)
        assert len(p.keep) == 48


def test_a8_working_set_compaction():
    """Reference acceptance A8 (pkg/tests/test_acceptance.py:282-320) on the device prune:
    at beta=0.5, lambda=2 the retained tokens' mean per-layer working set is >= 15% smaller
    than uniform-random retention at equal budget, and the inactive-expert count exceeds the
    uncompressed set's at every layer (50 seeds)."""
    comp_ws, rand_ws, inactive_kept, inactive_all = [], [], [], []
    rng = np.random.default_rng(777)
    layers = 6
    for seed in range(50):
        tr = generate_trace(TraceGenConfig(n_visual=48, n_text=0, layers=layers, experts=128, k=8, clusters=4,
                                           cluster_support=16, rho=0.9, visual_noise=0.05, seed=seed))
        p = compress(tr, CompressionConfig(alpha=0.07, beta=0.5, lam=2.0, prefix_layers=(0, 1)))
        kept = p.retained_ids(tr)
        rand_keep = sorted(int(i) for i in rng.choice(tr.visual_ids(), size=len(p.keep), replace=False))
        allp = tr.prefill_ids()
        ws_kept = [len(tr.active_union(l, kept)) for l in range(layers)]
        ws_rand = [len(tr.active_union(l, rand_keep)) for l in range(layers)]
        ws_all = [len(tr.active_union(l, allp)) for l in range(layers)]
        comp_ws.append(np.mean(ws_kept))
        rand_ws.append(np.mean(ws_rand))
        inactive_kept.append([tr.experts - w for w in ws_kept])
        inactive_all.append([tr.experts - w for w in ws_all])
    assert float(np.mean(comp_ws)) <= 0.85 * float(np.mean(rand_ws))
    assert np.all(np.mean(np.array(inactive_kept), axis=0) > np.mean(np.array(inactive_all), axis=0))
