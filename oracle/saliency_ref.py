"""Oracle (test infrastructure only): fp64 restatement of attention-derived
saliency, s = Mean_h(A^h) of Algorithm 1, with A the
softmax(q k^T * scale) rows of the CLS/text queries over a request's tokens.
The reference has no implementation (it reads saliency from the trace,
trace.py:49): parity unpinned, checked by tolerance.
"""
from __future__ import annotations

import numpy as np


def attention_saliency(q: np.ndarray, k: np.ndarray, scale: float) -> np.ndarray:
    """q [R, Hh, Q, D], k [R, Hh, N, D] (any float dtype) -> f64 [R*N]."""
    q = q.astype(np.float64)
    k = k.astype(np.float64)
    logits = np.einsum("rhqd,rhnd->rhqn", q, k) * scale
    logits -= logits.max(axis=-1, keepdims=True)
    p = np.exp(logits)
    p /= p.sum(axis=-1, keepdims=True)
    R, Hh, Q, N = p.shape
    return p.reshape(R, Hh * Q, N).mean(axis=1).reshape(-1)
