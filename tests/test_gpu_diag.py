"""GPU routing diagnostics (bit-exact vs the reference's moesim.metrics golden)
and attention-derived saliency (vs the fp64 oracle; parity unpinned, tolerance
rtol 1e-4 / atol 1e-8 on fp32 softmax) feeding the bit-exact prune."""
import math

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import compress_ref, saliency_ref
from paper_2605_05899_b200 import metrics
from paper_2605_05899_b200.saliency import attention_map_saliency, attention_saliency
from paper_2605_05899_b200.trace import RoutingTrace, TraceGenConfig, generate_trace, trace_digest

pytestmark = pytest.mark.gpu

_CACHE = {}


def regen(d, digest):
    if digest not in _CACHE:
        d = dict(d)
        d["saliency_shape"] = tuple(d["saliency_shape"])
        tr = generate_trace(TraceGenConfig(**d))
        assert trace_digest(tr) == digest
        _CACHE[digest] = tr
    return _CACHE[digest]


def test_device_diagnostics_bit_exact_vs_reference():
    for case in load_golden("metrics.json"):
        tr = regen(case["gen"], case["digest"])
        rep = metrics.affinity_report(tr, case["ids"], case["top"])
        assert rep.per_layer_working_set == case["working_set"]
        assert rep.topk_coverage == [float.fromhex(v) for v in case["coverage"]]
        assert rep.interlayer_similarity == [float.fromhex(v) for v in case["similarity"]]
        assert rep.interlayer_jaccard == [float.fromhex(v) for v in case["jaccard"]]
        assert [rep.mean_working_set, rep.mean_coverage, rep.mean_similarity] == \
            [float.fromhex(v) for v in case["means"]]


def test_single_metric_entry_points():
    tr = generate_trace(TraceGenConfig(n_visual=60, n_text=4, layers=4, experts=8, k=2, seed=2))
    ids = list(range(10))
    from oracle import metrics_ref as M

    re = tr.route_experts
    assert metrics.working_set(tr, ids, 1) == M.working_set(re, 8, ids, 1)
    assert metrics.topk_coverage(tr, ids, 2, 3) == M.topk_coverage(re, 8, ids, 2, 3)
    assert metrics.interlayer_similarity(tr, ids, 0) == M.interlayer_similarity(re, 8, ids, 0)
    assert metrics.interlayer_jaccard(tr, ids, 2) == M.interlayer_jaccard(re, 8, ids, 2)
    with pytest.raises(ValueError):
        metrics.topk_coverage(tr, [], 0, 1)
    with pytest.raises(ValueError):
        metrics.interlayer_similarity(tr, ids, 3)


@pytest.mark.parametrize("R,Hh,Q,N,D", [(1, 16, 1, 2368, 72), (2, 4, 16, 600, 128), (3, 2, 70, 97, 64)])
def test_attention_saliency_matches_fp64_oracle(R, Hh, Q, N, D):
    g = torch.Generator().manual_seed(R * 100 + Q)
    q = (torch.randn(R, Hh, Q, D, generator=g) * 2).to(torch.bfloat16)
    k = torch.randn(R, Hh, N, D, generator=g).to(torch.bfloat16)
    s = attention_saliency(q.cuda(), k.cuda()).cpu().numpy()
    ref = saliency_ref.attention_saliency(q.float().numpy(), k.float().numpy(), 1.0 / math.sqrt(D))
    np.testing.assert_allclose(s, ref, rtol=1e-4, atol=1e-8)
    # each softmax row sums to 1, so each request's saliency sums to 1
    np.testing.assert_allclose(s.reshape(R, N).sum(axis=1), 1.0, rtol=1e-5)
    maps = torch.rand(R, Hh * Q, N, generator=g)
    np.testing.assert_allclose(attention_map_saliency(maps.cuda()).cpu().numpy(),
                               maps.double().mean(dim=1).reshape(-1).numpy(), rtol=1e-12)


def test_prune_on_device_saliency_is_bit_exact():
    """The derived saliency enters the decision path at the reference's boundary
    (compress.py:145-148): the device prune on it equals the oracle on it."""
    from paper_2605_05899_b200 import CompressionConfig, compress

    tr = generate_trace(TraceGenConfig(n_visual=576, n_text=64, layers=8, experts=8, k=2, cluster_support=4,
                                       visual_noise=0.3, seed=0))
    g = torch.Generator().manual_seed(7)
    q = torch.randn(1, 8, 1, 64, generator=g).to(torch.bfloat16)
    k = torch.randn(1, 8, tr.num_tokens, 64, generator=g).to(torch.bfloat16)
    sal = attention_saliency(q.cuda(), k.cuda()).cpu().numpy()
    tr2 = RoutingTrace(tr.layers, tr.experts, tr.k, tr.route_experts, tr.route_gates, sal, tr.modality,
                       tr.embedding, tr.cluster, tr.phase_marks, tr.shared_experts)
    cc = CompressionConfig(0.05, 0.25, 2.0, (0, 1))
    p = compress(tr2, cc)
    o = compress_ref.compress(sal, tr.modality, tr.phase_marks, tr.route_experts, tr.experts, 0.05, 0.25, 2.0, [0, 1])
    assert p.keep == o["keep"] and p.core == o["core"]


def test_stack_forward_with_attention_saliency():
    """MoEStack.forward(saliency=None, attn_qk=...) == forward(saliency=derived)."""
    from paper_2605_05899_b200.moe import MoEStack, StackConfig

    cfg = StackConfig(layers=8, hidden=256, experts=8, k=2, inter=512, l_pinned=2, num_slabs=24, alpha=0.05,
                      beta=0.25, predictor="gate", budget=4, window=3, transfer_ms=0.3, gpu_ms=0.02)
    tr = generate_trace(TraceGenConfig(n_visual=576, n_text=64, layers=8, experts=8, k=2, seed=4))
    T = tr.num_tokens
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((2 * T, 256), generator=g, device="cuda").to(torch.bfloat16)
    mod = torch.from_numpy(np.concatenate([tr.device_modality()] * 2)).cuda()
    q = torch.randn(2, 4, 8, 64, generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn(2, 4, T, 64, generator=g, device="cuda").to(torch.bfloat16)
    stack = MoEStack(cfg)
    a = stack.forward(x, None, mod, req_off=[0, T, 2 * T], attn_qk=(q, k))
    ha, ra = a.hidden.clone(), a.retained.copy()
    b = stack.forward(x, attention_saliency(q, k), mod, req_off=[0, T, 2 * T])
    assert np.array_equal(ra, b.retained)
    assert torch.equal(ha, b.hidden)
