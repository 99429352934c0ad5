"""Device compression (vmm_prune) is bit-exact with the reference's compress()."""
import math

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import compress_ref
from paper_2605_05899_b200 import CompressionConfig, compress, kernels
from paper_2605_05899_b200.errors import ValidationError
from paper_2605_05899_b200.trace import RoutingTrace, TraceGenConfig, generate_trace, trace_digest

pytestmark = pytest.mark.gpu


def hand_trace(sal, routes, experts, k, modality=None):
    routes = np.asarray(routes, dtype=np.int64)
    L, n = routes.shape[0], routes.shape[1]
    mod = np.zeros(n, np.uint8) if modality is None else np.asarray(modality, np.uint8)
    return RoutingTrace(L, experts, k, routes, np.full(routes.shape, 1.0 / k), np.asarray(sal, float), mod,
                        np.zeros((n, 1)))


def regen(d, digest):
    d = dict(d)
    d["saliency_shape"] = tuple(d["saliency_shape"])
    tr = generate_trace(TraceGenConfig(**d))
    assert trace_digest(tr) == digest
    return tr


def test_frozen_instance():
    g = load_golden("compress.json")["frozen"]
    tr = hand_trace(g["saliency"], g["routes"], g["experts"], g["k"])
    p = compress(tr, CompressionConfig(g["alpha"], g["beta"], g["lam"], tuple(g["prefix"])))
    assert p.core == [0] and p.keep == [0, 1, 2] and p.target_experts == {0}
    assert p.delta == {1: 0.0, 2: 1.0, 3: 1.0, 4: 1.0, 5: 1.0}
    assert p.score == {1: 0.0, 2: -1.125, 3: -1.25, 4: -1.75, 5: -1.5}


def test_random_instances_match_reference():
    for c in load_golden("compress.json")["random"]:
        tr = hand_trace(c["saliency"], c["routes"], c["experts"], c["k"])
        p = compress(tr, CompressionConfig(c["alpha"], c["beta"], c["lam"], tuple(c["prefix"])))
        assert p.core == c["core"]
        assert p.keep == c["keep"]
        assert sorted(p.target_experts) == c["target"]
        assert [[i, p.delta[i]] for i in sorted(p.delta)] == c["delta"]
        assert [[i, p.score[i]] for i in sorted(p.score)] == c["score"]


def test_generated_traces_full_shapes_match_reference():
    """C1 / C3 (2304+64 tokens, 8 prefix layers, E=128) / C4 and small traces."""
    for c in load_golden("compress.json")["traces"]:
        tr = regen(c["gen"], c["digest"])
        p = compress(tr, CompressionConfig(c["alpha"], c["beta"], c["lam"], tuple(c["prefix"])))
        assert p.core == c["core"], c["name"]
        assert p.keep == c["keep"]
        assert sorted(p.target_experts) == c["target"]
        assert p.retained_ids(tr) == c["retained"]
        vis = tr.visual_ids()
        for i, (dh, sh, nh) in zip(vis, zip(c["delta_hex"], c["score_hex"], c["snorm_hex"])):
            assert p.saliency_norm[i] == float.fromhex(nh)
            if dh is None:
                assert i not in p.delta
            else:
                assert p.delta[i] == float.fromhex(dh) and p.score[i] == float.fromhex(sh)


def test_batched_requests_one_launch_match_oracle():
    """R requests in one launch (one CTA per request), ragged sizes incl. all-text and empty."""
    rng = np.random.default_rng(5)
    specs = [(300, 20), (0, 7), (1, 0), (2304, 64), (57, 3), (5, 5)]
    P, k, E = 3, 4, 64
    sal, mod, routes, offs, kc, kk, exp = [], [], [], [0], [], [], []
    for nv, nt in specs:
        n = nv + nt
        s = rng.integers(0, 6, size=n).astype(float)  # ties
        m = np.r_[np.zeros(nv, np.uint8), np.ones(nt, np.uint8)]
        rng.shuffle(m)
        r = np.stack([np.stack([rng.choice(E, size=k, replace=False) for _ in range(n)]) if n else
                      np.zeros((0, k), int) for _ in range(P)])
        cfg = CompressionConfig(0.1, 0.5, 1.7, (0, 1, 2))
        kcore, kkeep = cfg.budgets(nv)
        o = compress_ref.compress(s, m, [], r, E, 0.1, 0.5, 1.7, [0, 1, 2])
        exp.append(o)
        sal.append(s); mod.append(m); routes.append(r); offs.append(offs[-1] + n); kc.append(kcore); kk.append(kkeep)
    dev = torch.device("cuda")
    out = kernels.prune(torch.from_numpy(np.concatenate(sal)).to(dev), torch.from_numpy(np.concatenate(mod)).to(dev),
                        torch.from_numpy(np.concatenate(routes, axis=1).astype(np.int32)).to(dev),
                        torch.tensor(offs, dtype=torch.int32, device=dev), torch.tensor(kc, dtype=torch.int32, device=dev),
                        torch.tensor(kk, dtype=torch.int32, device=dev), E, 1.7)
    flags = out["flags"].cpu().numpy()
    ret = out["retained"].cpu().numpy()
    nret = out["n_retained"].cpu().numpy()
    assert (out["status"].cpu().numpy() == 0).all()
    for r, o in enumerate(exp):
        a, b = offs[r], offs[r + 1]
        assert ret[a:a + nret[r]].tolist() == o["retained"].tolist()
        keep = np.flatnonzero(flags[a:b] & 2).tolist()
        assert keep == o["keep"]
        assert np.flatnonzero(flags[a:b] & 1).tolist() == o["core"]
        sc = out["score"].cpu().numpy()[a:b]
        for pos, tok in enumerate(o["visual"]):
            if not math.isnan(o["score"][pos]):
                assert sc[tok] == o["score"][pos]


def test_invalid_saliency_raises_validation_error():
    tr = hand_trace([1.0, float("nan"), 2.0], [[[0], [1], [2]]], 4, 1)
    with pytest.raises(ValidationError):
        compress(tr, CompressionConfig(0.3, 0.6))
    tr = hand_trace([1.0, -1.0, 2.0], [[[0], [1], [2]]], 4, 1)
    with pytest.raises(ValidationError):
        compress(tr, CompressionConfig(0.3, 0.6))


def test_gather_rows_compacts_hidden_states():
    x = torch.randn(100, 256, device="cuda").to(torch.bfloat16)
    idx = torch.tensor([0, 5, 7, 99, 42], dtype=torch.int32, device="cuda")
    y = kernels.gather_rows(x, idx)
    assert torch.equal(y, x[idx.long()])


def _batch(rng, specs, P, k, E, ties=True):
    sal, mod, routes, offs = [], [], [], [0]
    for nv, nt in specs:
        n = nv + nt
        s = rng.integers(0, 6, size=n).astype(float) if ties else rng.gamma(2.0, 1.0, size=n)
        m = np.r_[np.zeros(nv, np.uint8), np.ones(nt, np.uint8)]
        rng.shuffle(m)
        r = np.stack([np.stack([rng.choice(E, size=k, replace=False) for _ in range(n)]) if n else
                      np.zeros((0, k), int) for _ in range(P)])
        sal.append(s); mod.append(m); routes.append(r); offs.append(offs[-1] + n)
    dev = torch.device("cuda")
    d = dict(sal=torch.from_numpy(np.concatenate(sal)).to(dev), mod=torch.from_numpy(np.concatenate(mod)).to(dev),
             routes=torch.from_numpy(np.concatenate(routes, axis=1).astype(np.int32)).to(dev),
             offs=torch.tensor(offs, dtype=torch.int32, device=dev))
    return d, sal, mod, routes, offs


@pytest.mark.parametrize("lam", [0.0, 0.5, 1.0, 2.0, 5.0])
def test_batched_device_budgets_both_cta_sizes_match_oracle(lam):
    """R=70 requests (the 256-thread batch variant) and R=5 (the 1024-thread variant),
    budgets floor(alpha n_vis)/floor(beta n_vis) computed on the device, heavy ties
    (integer saliencies, A1 style, pkg/tests/test_acceptance.py:47-78), every lambda of A1;
    the packed global retained list equals the concatenation of the oracle's."""
    rng = np.random.default_rng(int(lam * 10) + 17)
    P, k, E = 2, 3, 40
    for R in (70, 5):
        specs = [(int(rng.integers(0, 400)), int(rng.integers(0, 30))) for _ in range(R)]
        d, sal, mod, routes, offs = _batch(rng, specs, P, k, E, ties=R == 70)
        out = kernels.prune(d["sal"], d["mod"], d["routes"], d["offs"], None, None, E, lam, alpha=0.13, beta=0.55)
        assert (out["status"].cpu().numpy() == 0).all()
        packed, poff = kernels.retained_pack(d["offs"], out["retained"], out["n_retained"])
        flags = out["flags"].cpu().numpy()
        sc, dl = out["score"].cpu().numpy(), out["delta"].cpu().numpy()
        packed, poff = packed.cpu().numpy(), poff.cpu().numpy()
        for r in range(R):
            o = compress_ref.compress(sal[r], mod[r], [], routes[r], E, 0.13, 0.55, lam, list(range(P)))
            a, b = offs[r], offs[r + 1]
            assert np.flatnonzero(flags[a:b] & 1).tolist() == o["core"], (R, r)
            assert np.flatnonzero(flags[a:b] & 2).tolist() == o["keep"], (R, r)
            assert packed[poff[r]:poff[r + 1]].tolist() == (np.asarray(o["retained"]) + a).tolist(), (R, r)
            for pos, tok in enumerate(o["visual"]):
                if not math.isnan(o["score"][pos]):
                    assert sc[a + tok] == o["score"][pos] and dl[a + tok] == o["delta"][pos]


def test_large_request_beyond_old_cap_matches_oracle():
    """20 000 visual tokens in one request (the round-1 kernel refused > 8192) and a
    C3-shaped request (2304 + 64, 8 prefix layers, E=128), both against the oracle."""
    rng = np.random.default_rng(3)
    for nv, nt, P, k, E in ((20000, 100, 2, 4, 64), (2304, 64, 8, 8, 128)):
        d, sal, mod, routes, offs = _batch(rng, [(nv, nt)], P, k, E, ties=False)
        out = kernels.prune(d["sal"], d["mod"], d["routes"], d["offs"], None, None, E, 2.0, alpha=0.1, beta=0.5)
        assert int(out["status"].cpu()[0]) == 0
        o = compress_ref.compress(sal[0], mod[0], [], routes[0], E, 0.1, 0.5, 2.0, list(range(P)))
        flags = out["flags"].cpu().numpy()
        assert np.flatnonzero(flags & 1).tolist() == o["core"]
        assert np.flatnonzero(flags & 2).tolist() == o["keep"]
        n = int(out["n_retained"].cpu()[0])
        assert out["retained"][:n].cpu().numpy().tolist() == list(o["retained"])


def test_prune_status_codes():
    """alpha > beta -> status 3 (ValidationError); an expert id outside [0, E) -> status 4
    (TraceError) instead of an out-of-bounds mask write."""
    from paper_2605_05899_b200.compress import raise_prune_status
    from paper_2605_05899_b200.errors import TraceError

    rng = np.random.default_rng(9)
    d, *_ = _batch(rng, [(50, 5)], 1, 2, 8)
    out = kernels.prune(d["sal"], d["mod"], d["routes"], d["offs"], None, None, 8, 2.0, alpha=0.6, beta=0.3)
    assert int(out["status"].cpu()[0]) == 3
    with pytest.raises(ValidationError):
        raise_prune_status(3)
    bad = d["routes"].clone()
    bad[0, 7, 1] = 200
    out = kernels.prune(d["sal"], d["mod"], bad, d["offs"], None, None, 8, 2.0, alpha=0.1, beta=0.5)
    assert int(out["status"].cpu()[0]) == 4
    with pytest.raises(TraceError):
        raise_prune_status(4)
