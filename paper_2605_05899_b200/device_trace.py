"""HBM-resident copy of a routing trace (uploaded once, reused by every op).

Layout in HBM: routes i32 [L, T, k] (layer-major so one
layer's picks are contiguous), saliency f64 [T], modality u8 [T] (0 visual,
1 text, 2 decode), embeddings f64 [T, D].

The upload is cached per trace OBJECT (keyed by `id`, dropped by a
`weakref.finalize` when the trace dies): the reference's `RoutingTrace`
defines `__eq__` without `__hash__` (pkg/src/moesim/trace.py:66,135), so it
cannot key a dict, and equal-but-distinct traces must not share an upload
anyway.  The cached entry holds no strong reference to the trace.
"""
from __future__ import annotations

import weakref

import numpy as np
import torch

_CACHE: dict[int, tuple["weakref.ref", "DeviceTrace"]] = {}


class DeviceTrace:
    def __init__(self, trace, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.L, self.E, self.k = trace.layers, trace.experts, trace.k
        self.T = trace.num_tokens
        self.routes = torch.from_numpy(np.ascontiguousarray(trace.route_experts, dtype=np.int32)).to(dev)
        self.saliency = torch.from_numpy(np.ascontiguousarray(trace.saliency)).to(dev)
        self.modality = torch.from_numpy(trace.device_modality()).to(dev)
        # f64 [T, D] on the host (small); uploaded on first use by the MLP features
        self._emb_host = np.ascontiguousarray(trace.embedding, dtype=np.float64)
        self._emb = None
        self.all_layers = torch.arange(self.L, dtype=torch.int32, device=dev)

    @property
    def embeddings(self):
        if self._emb is None:
            self._emb = torch.from_numpy(self._emb_host).to(self.device)
        return self._emb

    def ids(self, token_ids) -> torch.Tensor:
        a = np.asarray(list(token_ids) if not isinstance(token_ids, np.ndarray) else token_ids, dtype=np.int32)
        return torch.from_numpy(a).to(self.device)


def as_trace(trace):
    """Accept the reference's RoutingTrace (or any duck-typed equivalent)."""
    from .trace import RoutingTrace

    return trace if isinstance(trace, RoutingTrace) else RoutingTrace.from_reference(trace)


def _drop(key: int) -> None:
    _CACHE.pop(key, None)


def device_trace(trace) -> DeviceTrace:
    key = id(trace)
    hit = _CACHE.get(key)
    if hit is not None and hit[0]() is trace:
        return hit[1]
    dt = DeviceTrace(as_trace(trace))
    try:
        ref = weakref.ref(trace)
    except TypeError:  # not weak-referenceable: convert without caching
        return dt
    _CACHE[key] = (ref, dt)
    weakref.finalize(trace, _drop, key)
    return dt
