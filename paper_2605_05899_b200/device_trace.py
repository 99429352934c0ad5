"""HBM-resident copy of a routing trace (uploaded once, reused by every op).

Layout in HBM: routes i32 [L, T, k] (layer-major so one
layer's picks are contiguous), saliency f64 [T], modality u8 [T] (0 visual,
1 text, 2 decode), embeddings f64 [T, D].
"""
from __future__ import annotations

import weakref

import numpy as np
import torch

_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


class DeviceTrace:
    def __init__(self, trace, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.trace = trace
        self.device = dev
        self.L, self.E, self.k = trace.layers, trace.experts, trace.k
        self.T = trace.num_tokens
        self.routes = torch.from_numpy(np.ascontiguousarray(trace.route_experts, dtype=np.int32)).to(dev)
        self.saliency = torch.from_numpy(np.ascontiguousarray(trace.saliency)).to(dev)
        self.modality = torch.from_numpy(trace.device_modality()).to(dev)
        self._emb = None
        self.all_layers = torch.arange(self.L, dtype=torch.int32, device=dev)

    @property
    def embeddings(self):
        if self._emb is None:
            self._emb = torch.from_numpy(np.ascontiguousarray(self.trace.embedding)).to(self.device)
        return self._emb

    def ids(self, token_ids) -> torch.Tensor:
        a = np.asarray(list(token_ids) if not isinstance(token_ids, np.ndarray) else token_ids, dtype=np.int32)
        return torch.from_numpy(a).to(self.device)


def as_trace(trace):
    """Accept the reference's RoutingTrace (or any duck-typed equivalent)."""
    from .trace import RoutingTrace

    return trace if isinstance(trace, RoutingTrace) else RoutingTrace.from_reference(trace)


def device_trace(trace) -> DeviceTrace:
    dt = _CACHE.get(trace)
    if dt is None:
        dt = DeviceTrace(as_trace(trace))
        _CACHE[trace] = dt
    return dt
