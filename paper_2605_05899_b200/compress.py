"""Affinity-aware visual-token compression on the device (drop-in for
`moesim.compress`, pkg/src/moesim/compress.py:24-185).

`compress(trace, cfg)` has the reference's signature and returns the same
`CompressionPlan` (core/keep sorted id lists, target expert set, delta/score
dicts over non-core visual tokens, saliency_norm over visual tokens).  The
selection itself runs in one sm_100a kernel (`vmm_prune`): fp64 min-max
normalisation, bitonic top-k with exact tie keys, expert-bitmask marginal
expansion and stream compaction of the retained ids, bit-identical to the
reference.  `compress_device` is the batched, sync-free form used inside the
layer stack.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels
from .device_trace import device_trace
from .errors import TraceError, ValidationError

DEFAULT_TRADEOFF = 2.0  # compress.py:21


@dataclass(frozen=True)
class CompressionConfig:
    alpha: float
    beta: float
    lam: float = DEFAULT_TRADEOFF
    prefix_layers: tuple[int, ...] = (0,)

    def validate(self, layers: int | None = None) -> None:  # compress.py:31-43
        if not 0.0 <= self.alpha <= 1.0:
            raise ValidationError("alpha must lie in [0, 1]")
        if not 0.0 <= self.beta <= 1.0:
            raise ValidationError("beta must lie in [0, 1]")
        if self.alpha > self.beta:
            raise ValidationError("alpha must not exceed beta")
        if self.lam < 0.0:
            raise ValidationError("lam must be >= 0")
        if not self.prefix_layers:
            raise ValidationError("prefix_layers must be non-empty")
        if layers is not None and any(not 0 <= l < layers for l in self.prefix_layers):
            raise ValidationError("prefix_layers must all be valid layer indices")

    def budgets(self, n_visual: int) -> tuple[int, int]:
        k_core = math.floor(self.alpha * n_visual)  # compress.py:151-152
        k_keep = math.floor(self.beta * n_visual)
        if k_keep < k_core:
            raise ValidationError("beta budget smaller than alpha budget")
        return k_core, k_keep


@dataclass
class CompressionPlan:
    core: list[int]
    keep: list[int]
    target_experts: set[int]
    delta: dict[int, float]
    score: dict[int, float]
    saliency_norm: dict[int, float]
    config: CompressionConfig

    def retained_ids(self, trace) -> list[int]:
        return sorted(set(self.keep) | set(trace.text_ids()))

    def to_json(self) -> str:
        obj = {
            "core": sorted(self.core),
            "keep": sorted(self.keep),
            "target_experts": sorted(self.target_experts),
            "delta": {str(i): self.delta[i] for i in sorted(self.delta)},
            "score": {str(i): self.score[i] for i in sorted(self.score)},
            "saliency_norm": {str(i): self.saliency_norm[i] for i in sorted(self.saliency_norm)},
            "config": {"alpha": self.config.alpha, "beta": self.config.beta, "lam": self.config.lam,
                       "prefix_layers": list(self.config.prefix_layers)},
        }
        return json.dumps(obj, indent=2)

    @classmethod
    def from_json(cls, text: str) -> "CompressionPlan":
        o = json.loads(text)
        c = o["config"]
        return cls(
            core=list(o["core"]), keep=list(o["keep"]), target_experts=set(o["target_experts"]),
            delta={int(i): v for i, v in o["delta"].items()}, score={int(i): v for i, v in o["score"].items()},
            saliency_norm={int(i): v for i, v in o["saliency_norm"].items()},
            config=CompressionConfig(c["alpha"], c["beta"], c["lam"], tuple(c["prefix_layers"])),
        )


def compress_device(saliency, modality, prefix_routes, req_off, k_core, k_keep, experts, lam, stream=None):
    """Batched device compression (no host sync); see kernels.prune."""
    return kernels.prune(saliency, modality, prefix_routes, req_off, k_core, k_keep, experts, lam, stream)


_STATUS = {1: (ValidationError, "saliency entries must be finite and >= 0"),
           3: (ValidationError, "beta budget smaller than alpha budget"),
           4: (TraceError, "prefix route expert id outside [0, experts)")}


def raise_prune_status(status: int) -> None:
    """Map a vmm_prune status to the reference's exception (compress.py:104-154)."""
    if status:
        cls, msg = _STATUS.get(status, (ValidationError, f"prune failed with status {status}"))
        raise cls(msg)


def compress(trace, cfg: CompressionConfig) -> CompressionPlan:
    """Run the full selection policy over the trace's visual tokens (on the GPU)."""
    cfg.validate(trace.layers)
    visual = trace.visual_ids()
    # budgets inline (compress.py:151-154): `cfg` may be the reference's own
    # CompressionConfig, which has only alpha/beta/lam/prefix_layers + validate()
    k_core = math.floor(cfg.alpha * len(visual))
    k_keep = math.floor(cfg.beta * len(visual))
    if k_keep < k_core:
        raise ValidationError("beta budget smaller than alpha budget")
    dt = device_trace(trace)
    dev = dt.device
    layers = torch.tensor(list(cfg.prefix_layers), dtype=torch.long, device=dev)
    prefix = dt.routes.index_select(0, layers).contiguous()
    req_off = torch.tensor([0, dt.T], dtype=torch.int32, device=dev)
    kc = torch.tensor([k_core], dtype=torch.int32, device=dev)
    kk = torch.tensor([k_keep], dtype=torch.int32, device=dev)
    out = kernels.prune(dt.saliency, dt.modality, prefix, req_off, kc, kk, trace.experts, cfg.lam)
    raise_prune_status(int(out["status"].cpu()[0]))
    flags = out["flags"].cpu().numpy()
    s_norm = out["s_norm"].cpu().numpy()
    delta = out["delta"].cpu().numpy()
    score = out["score"].cpu().numpy()
    tmask = out["target"].cpu().numpy().view(np.uint64)[0]
    vis = np.asarray(visual, dtype=np.int64)
    core_ids = vis[(flags[vis] & 1) != 0]
    keep_ids = vis[(flags[vis] & 2) != 0]
    rest = vis[(flags[vis] & 1) == 0]
    target = {w * 64 + b for w in range(4) for b in range(64) if (int(tmask[w]) >> b) & 1}
    return CompressionPlan(
        core=core_ids.tolist(),
        keep=keep_ids.tolist(),
        target_experts=target,
        delta={int(i): float(delta[i]) for i in rest},
        score={int(i): float(score[i]) for i in rest},
        saliency_norm={int(i): float(s_norm[i]) for i in vis},
        config=cfg,
    )
