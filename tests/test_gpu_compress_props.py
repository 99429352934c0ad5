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
