"""Oracle: affinity-aware visual-token compression (reference Alg. 1).

Restates `pkg/src/moesim/compress.py:104-185` with numpy.  Every float is an
IEEE fp64 op in the same order as the reference (no fused multiply-add: numpy
never contracts `a - lam * d`), so outputs are bit-identical:

* s_norm  = (s - lo) / (hi - lo), constant -> 0.5              (compress.py:104-114)
* core    = top floor(alpha*n) by (-s_norm, id), sorted         (compress.py:151-157)
* target  = union of core tokens' prefix-layer experts          (compress.py:159-161)
* delta_i = |E_i \\ T| / |E_i|                                  (compress.py:135-139)
* score_i = s_norm_i - lam * delta_i                            (compress.py:172)
* extras  = top (k_keep - k_core) by (-score, -s_norm, id)      (compress.py:174)
* keep    = sorted(core + extras); retained = keep U text ids   (compress.py:63-65,175)
"""
from __future__ import annotations

import math

import numpy as np


class OracleValidationError(ValueError):
    pass


def normalize(sal: np.ndarray) -> np.ndarray:
    s = np.asarray(sal, dtype=np.float64)
    if s.size and (not np.all(np.isfinite(s)) or np.any(s < 0)):
        raise OracleValidationError("saliency entries must be finite and >= 0")
    if s.size == 0:
        return s
    lo, hi = float(s.min()), float(s.max())
    if hi == lo:
        return np.full_like(s, 0.5)
    return (s - lo) / (hi - lo)


def prefix_masks(route_experts: np.ndarray, tokens: np.ndarray, prefix_layers, experts: int) -> np.ndarray:
    """bool [n, E]: expert e active for token in any prefix layer (compress.py:125-132)."""
    m = np.zeros((tokens.size, experts), dtype=bool)
    rows = np.arange(tokens.size)[:, None]
    for l in prefix_layers:
        m[rows, route_experts[l][tokens]] = True
    return m


def compress(saliency, modality, phase_marks, route_experts, experts, alpha, beta, lam, prefix_layers):
    """Returns dict(core, keep, target, delta, score, s_norm, retained).

    `modality` u8 per token (0 visual, 1 text); phase_marks are decode ids.
    delta/score/s_norm are dense arrays indexed by visual position.
    """
    n_tok = len(saliency)
    dec = np.zeros(n_tok, dtype=bool)
    if len(phase_marks):
        dec[np.asarray(phase_marks, dtype=np.int64)] = True
    modality = np.asarray(modality)
    visual = np.flatnonzero((modality == 0) & ~dec)
    text = np.flatnonzero((modality == 1) & ~dec)
    n = visual.size
    s = normalize(np.asarray(saliency, dtype=np.float64)[visual])
    k_core = math.floor(alpha * n)
    k_keep = math.floor(beta * n)
    if k_keep < k_core:
        raise OracleValidationError("beta budget smaller than alpha budget")
    pos = np.arange(n)
    core_pos = np.sort(np.lexsort((pos, -s))[:k_core])
    masks = prefix_masks(route_experts, visual, prefix_layers, experts)
    target = masks[core_pos].any(axis=0)
    is_core = np.zeros(n, dtype=bool)
    is_core[core_pos] = True
    rest = np.flatnonzero(~is_core)
    sz = masks[rest].sum(axis=1)
    outside = (masks[rest] & ~target).sum(axis=1)
    delta = np.full(n, np.nan)
    score = np.full(n, np.nan)
    delta[rest] = outside.astype(np.float64) / sz.astype(np.float64)
    score[rest] = s[rest] - lam * delta[rest]
    order = np.lexsort((rest, -s[rest], -score[rest]))
    extra_pos = rest[order[: k_keep - k_core]]
    keep_pos = np.sort(np.concatenate([core_pos, extra_pos]))
    keep = visual[keep_pos]
    retained = np.union1d(keep, text)
    return dict(
        core=visual[core_pos].tolist(),
        keep=keep.tolist(),
        target=np.flatnonzero(target).tolist(),
        delta=delta,
        score=score,
        s_norm=s,
        visual=visual,
        retained=retained.astype(np.int64),
        k_core=k_core,
        k_keep=k_keep,
    )
