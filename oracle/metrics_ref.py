"""Oracle (test infrastructure only): CPU restatement of the reference's
routing diagnostics, `pkg/src/moesim/metrics.py`:

* _histogram            metrics.py:17-22  (float64 counts, duplicates counted)
* working_set           metrics.py:25-27  (|active_union|)
* topk_coverage         metrics.py:30-40  (top by (-count, expert), / (|subset| k))
* interlayer_similarity metrics.py:43-54  (cosine; 1.0 if both empty, 0.0 if one)
* interlayer_jaccard    metrics.py:57-66  (1.0 if the union is empty)

Pinned by tests/golden/metrics.json (made by the real reference).
"""
from __future__ import annotations

import numpy as np


def histogram(routes: np.ndarray, experts: int, subset, layer: int) -> np.ndarray:
    # the reference adds 1.0 per (token, slot) in a Python loop; integer counts
    # are exact in float64, so a bincount gives the same array
    sub = np.asarray(list(subset), dtype=np.int64)
    return np.bincount(routes[layer, sub].ravel(), minlength=experts).astype(np.float64)


def working_set(routes, experts, subset, layer) -> int:
    return int(np.count_nonzero(histogram(routes, experts, subset, layer)))


def topk_coverage(routes, experts, subset, layer, top) -> float:
    subset = list(subset)
    k = routes.shape[2]
    counts = histogram(routes, experts, subset, layer)
    order = sorted(range(experts), key=lambda e: (-counts[e], e))
    covered = sum(counts[e] for e in order[:top])
    return covered / (len(subset) * k)


def interlayer_similarity(routes, experts, subset, layer) -> float:
    a = histogram(routes, experts, subset, layer)
    b = histogram(routes, experts, subset, layer + 1)
    na, nb = float(np.linalg.norm(a)), float(np.linalg.norm(b))
    if na == 0.0 and nb == 0.0:
        return 1.0
    if na == 0.0 or nb == 0.0:
        return 0.0
    return float(np.dot(a, b) / (na * nb))


def interlayer_jaccard(routes, experts, subset, layer) -> float:
    a = set(np.flatnonzero(histogram(routes, experts, subset, layer)).tolist())
    b = set(np.flatnonzero(histogram(routes, experts, subset, layer + 1)).tolist())
    union = a | b
    if not union:
        return 1.0
    return len(a & b) / len(union)
