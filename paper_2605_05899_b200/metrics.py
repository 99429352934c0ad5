"""Routing diagnostics on the GPU.

Same names and definitions as the reference's `moesim.metrics`
(`pkg/src/moesim/metrics.py:25-139`): working set, top-K coverage,
inter-layer cosine similarity and Jaccard index of a token subset, and the
`AffinityReport` over all layers.  The per-layer expert histograms come from
the same demand-count kernel the hot path uses (`vmm_demand_counts`), the
derived metrics from `vmm_routing_diagnostics` -- one launch each for the
whole stack instead of L x |subset| x k Python set operations.  Counts are
integers, so the results are bit-identical to the reference's.
"""
from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels
from ._lib import check, ptr, stream_ptr
from .device_trace import device_trace
from .errors import ValidationError


def _subset(dt, subset):
    subset = list(subset)
    if not subset:
        raise ValidationError("subset must be non-empty")
    return subset, dt.ids(subset)


def layer_diagnostics(trace, subset, top: int) -> np.ndarray:
    """f64 [L, 4]: working set, top-`top` coverage, cosine(l, l+1), jaccard(l, l+1) (NaN at L-1)."""
    dt = device_trace(trace)
    subset, ids = _subset(dt, subset)
    if not 0 <= top <= dt.E:
        raise ValidationError("top must lie in [0, experts]")
    counts = kernels.demand_counts(dt.routes, dt.all_layers, ids, dt.E)
    out = torch.empty(dt.L, 4, dtype=torch.float64, device=dt.device)
    kernels._n(1)
    check(_lib.lib().vmm_routing_diagnostics(ptr(counts), dt.L, dt.E, len(subset), dt.k, top, ptr(out),
                                             stream_ptr()))
    return out.cpu().numpy()


def working_set(trace, subset, layer: int) -> int:
    """Number of distinct experts the subset activates at the layer (metrics.py:25-27)."""
    return int(layer_diagnostics(trace, subset, 0)[layer, 0])


def topk_coverage(trace, subset, layer: int, top: int) -> float:
    """Fraction of activations captured by the `top` most-activated experts (metrics.py:30-40)."""
    return float(layer_diagnostics(trace, subset, top)[layer, 1])


def interlayer_similarity(trace, subset, layer: int) -> float:
    """Cosine similarity of the activation histograms at layer and layer+1 (metrics.py:43-54)."""
    if layer + 1 >= device_trace(trace).L:
        raise ValidationError("layer+1 must be a valid layer")
    return float(layer_diagnostics(trace, subset, 0)[layer, 2])


def interlayer_jaccard(trace, subset, layer: int) -> float:
    """|A & B| / |A | B| of the working sets at layer and layer+1 (metrics.py:57-66)."""
    if layer + 1 >= device_trace(trace).L:
        raise ValidationError("layer+1 must be a valid layer")
    return float(layer_diagnostics(trace, subset, 0)[layer, 3])


@dataclass
class AffinityReport:
    """Field-for-field the reference's AffinityReport (metrics.py:69-119)."""

    per_layer_working_set: list
    inactive_experts: list
    topk_coverage: list
    interlayer_similarity: list
    interlayer_jaccard: list
    top: int

    @property
    def mean_working_set(self) -> float:
        return float(np.mean(self.per_layer_working_set))

    @property
    def mean_inactive(self) -> float:
        return float(np.mean(self.inactive_experts))

    @property
    def mean_coverage(self) -> float:
        return float(np.mean(self.topk_coverage))

    @property
    def mean_similarity(self) -> float:
        return float(np.mean(self.interlayer_similarity)) if self.interlayer_similarity else 1.0

    def to_json(self) -> str:
        return json.dumps(
            {
                "top": self.top,
                "per_layer_working_set": self.per_layer_working_set,
                "inactive_experts": self.inactive_experts,
                "topk_coverage": self.topk_coverage,
                "interlayer_similarity": self.interlayer_similarity,
                "interlayer_jaccard": self.interlayer_jaccard,
                "mean_working_set": self.mean_working_set,
                "mean_inactive": self.mean_inactive,
                "mean_coverage": self.mean_coverage,
                "mean_similarity": self.mean_similarity,
            },
            indent=2,
        )


def affinity_report(trace, subset, top: int) -> AffinityReport:
    """All layers in two launches (metrics.py:122-139)."""
    d = layer_diagnostics(trace, subset, top)
    L = d.shape[0]
    E = device_trace(trace).E
    ws = [int(v) for v in d[:, 0]]
    return AffinityReport(
        per_layer_working_set=ws,
        inactive_experts=[E - w for w in ws],
        topk_coverage=[float(v) for v in d[:, 1]],
        interlayer_similarity=[float(v) for v in d[: L - 1, 2]],
        interlayer_jaccard=[float(v) for v in d[: L - 1, 3]],
        top=top,
    )
