"""Attention-derived visual-token saliency on the GPU.

VisMMOE's Algorithm 1 starts from s = Mean_h(A^h), the head-averaged
attention each visual token receives (VisionZip-style
CLS or text->visual attention); the reference simulator reads it precomputed
from the trace (`trace.py:49`, `SPEC.md:170`).  Here it is computed from the
vision encoder's query/key projections without materialising more than one
fp32 probability row per (request, head, query), and feeds `vmm_prune`
directly (MoEStack.forward(..., attn_qk=(q, k))).
"""
from __future__ import annotations

import math

import torch

from . import _lib, kernels
from ._lib import check, ptr, stream_ptr
from .errors import ValidationError


def attention_saliency(q, k, scale: float | None = None, stream=None, probs=None):
    """q bf16 [R, Hh, Q, D] (CLS / text query rows), k bf16 [R, Hh, N, D] (the
    request's tokens) -> saliency f64 [R*N]: mean over heads and queries of
    softmax(q k^T * scale), summed in ascending (head, query) order."""
    if q.dim() == 3:
        q, k = q.unsqueeze(0), k.unsqueeze(0)
    R, Hh, Q, D = (int(s) for s in q.shape)
    if tuple(k.shape[:2]) != (R, Hh) or int(k.shape[3]) != D:
        raise ValidationError("q [R,Hh,Q,D] and k [R,Hh,N,D] disagree")
    N = int(k.shape[2])
    scale = 1.0 / math.sqrt(D) if scale is None else float(scale)
    q = q.contiguous().to(torch.bfloat16)
    k = k.contiguous().to(torch.bfloat16)
    probs = torch.empty(R * Hh * Q, N, dtype=torch.float32, device=q.device) if probs is None else probs
    s = torch.empty(R * N, dtype=torch.float64, device=q.device)
    kernels._n(3)
    check(_lib.lib().vmm_attn_saliency(ptr(q), ptr(k), R, Hh, Q, N, D, scale, ptr(probs), ptr(s), stream_ptr(stream)))
    return s


def attention_map_saliency(maps, stream=None):
    """maps f32 [R, HQ, N] (attention rows already computed) -> f64 [R*N]."""
    if maps.dim() == 2:
        maps = maps.unsqueeze(0)
    R, HQ, N = (int(s) for s in maps.shape)
    maps = maps.contiguous().to(torch.float32)
    s = torch.empty(R * N, dtype=torch.float64, device=maps.device)
    kernels._n(1)
    check(_lib.lib().vmm_attn_map_saliency(ptr(maps), R, HQ, N, ptr(s), stream_ptr(stream)))
    return s
