"""Oracle: lookahead predictors and top-B selection.

Restates `pkg/src/moesim/predictor.py` in numpy:

* demand counts / sets                  predictor.py:115-117, trace.py:102-107
* decayed oracle targets                predictor.py:120-148 (exact)
* decayed routing histogram (History)   predictor.py:63-75 (exact: per expert the
  weight w_past is added count times in ascending past-layer order, then the
  vector is normalised by numpy's pairwise sum, replicated in `pairwise_sum`)
* top-B by (-y, id)                     predictor.py:434-440 (exact)
* MLP features + forward + sigmoid      predictor.py:36-112,196-202,542-547
  (BLAS order -> tolerance only, "parity unpinned" beyond 1e-12 relative)
* gate-reuse lookahead (new; no reference): counts of experts in the top-k of
  layer l+1's gate applied to layer l hidden states, normalised by N*k.
"""
from __future__ import annotations

import numpy as np


def demand_counts(route_experts: np.ndarray, layer: int, ids: np.ndarray, experts: int) -> np.ndarray:
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size == 0:
        return np.zeros(experts, dtype=np.int64)
    return np.bincount(route_experts[layer][ids].ravel(), minlength=experts).astype(np.int64)


def oracle_targets(route_experts, layers, layer, window, decay_table, ids, experts) -> np.ndarray:
    """g_e = max_{d<=W, layer+d<=L-1} decay_table[d-1]*[e active at layer+d]."""
    g = np.zeros(experts, dtype=np.float64)
    for d in range(1, window + 1):
        fut = layer + d
        if fut > layers - 1:
            break
        w = decay_table[d - 1]
        act = demand_counts(route_experts, fut, ids, experts) > 0
        g = np.where(act & (w > g), w, g)
    return g


def pairwise_sum(a: np.ndarray) -> float:
    """numpy's float64 add.reduce for a contiguous vector (pairwise, 8-way unrolled)."""
    n = a.shape[0]
    if n < 8:
        res = 0.0
        for i in range(n):
            res += float(a[i])
        return res
    if n <= 128:
        r = [float(a[j]) for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def history_histogram(route_experts, layer, ids, experts, pow_table) -> np.ndarray:
    """pow_table[j] = decay**j (host-computed, as the reference's `decay ** (layer-past)`)."""
    acc = np.zeros(experts, dtype=np.float64)
    for past in range(layer + 1):
        w = pow_table[layer - past]
        if w == 0.0 and past < layer:
            continue
        c = demand_counts(route_experts, past, ids, experts)
        for e in np.flatnonzero(c):
            x = acc[e]
            for _ in range(int(c[e])):
                x += w
            acc[e] = x
    total = pairwise_sum(acc)
    return acc / total if total > 0 else acc


def topb(y, budget: int) -> list[int]:
    y = np.asarray(y, dtype=np.float64)
    order = np.lexsort((np.arange(y.shape[0]), -y))
    return [int(e) for e in order[:budget]]


def mlp_forward(w1, b1, w2, b2, wo, bo, x):
    a1 = np.maximum(x @ w1.T + b1, 0.0)
    a2 = np.maximum(a1 @ w2.T + b2, 0.0)
    return a2 @ wo.T + bo


def mlp_priorities(model, feats: np.ndarray) -> np.ndarray:
    logits = mlp_forward(model["w1"], model["b1"], model["w2"], model["b2"], model["wo"], model["bo"], feats)
    return 1.0 / (1.0 + np.exp(-logits))


def mlp_features(route_experts, embedding, drift_row, layer, ids, experts, pow_table, h_v):
    """[h_r; mean(emb[ids] + drift); h_v]  (predictor.py:86-112)."""
    ids = np.asarray(ids, dtype=np.int64)
    h_r = history_histogram(route_experts, layer, ids, experts, pow_table)
    h_h = (embedding[ids] + drift_row).mean(axis=0)
    return np.concatenate([h_r, h_h, h_v])


def gate_lookahead(x: np.ndarray, w_next: np.ndarray, k: int) -> np.ndarray:
    """Per-expert share of top-k picks when layer l+1's gate scores h_l (fp64 logits)."""
    logits = x.astype(np.float64) @ w_next.astype(np.float64).T
    n, e = logits.shape
    ids = np.lexsort((np.broadcast_to(np.arange(e), (n, e)), -logits), axis=1)[:, :k]
    c = np.bincount(ids.ravel(), minlength=e).astype(np.float64)
    return c / float(n * k) if n else c
