"""Lookahead expert-demand predictors on the device (drop-in for the
predictor protocol of `pkg/src/moesim/predictor.py:469-550`).

Every predictor exposes the reference's duck-typed protocol
`priorities(layer, token_ids) -> float64[E]`, `predict(layer, budget,
token_ids)` and `reset()`, plus `device_table(ctx_layers, ids)` returning the
scores for many context layers in one batched launch (what `simulate` and the
layer stack use).

  OraclePredictor   decayed future-demand targets (build_targets :120-148), exact
  HistoryPredictor  decayed routing histogram (routing_histogram :63-75), exact
  MLPPredictor      features + bottleneck MLP + sigmoid (:86-112, :196-202, :542-547)
  RandomPredictor   the reference's seeded uniform baseline (:486-502); its
                    draws are generated host-side as synthetic input
  GatePredictor     new: layer l+1's gate applied to layer l hidden states
                    (top-k pick shares), see moe.py for the live version
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels
from .device_trace import device_trace
from .errors import ContractError, ValidationError

DEFAULT_WINDOW = 5
DEFAULT_GAMMA = 0.8
DEFAULT_BUDGET = 20
DEFAULT_HISTORY_DECAY = 0.5
MODEL_VERSION = 1
_DRIFT_SEED = 0x0D121F7  # predictor.py:31
_DRIFT_STEP = 0.05


def predict_topb(y, budget: int) -> list[int]:
    """Expert ids of the `budget` highest scores, descending, ties to lower id (predictor.py:434-440)."""
    y = np.asarray(y, dtype=np.float64)
    if budget > y.shape[0]:
        raise ValidationError("budget must not exceed the expert count")
    order = np.lexsort((np.arange(y.shape[0]), -y))
    return [int(e) for e in order[:budget]]


def decay_table(gamma: float, window: int) -> list[float]:
    """gamma ** (d - 1) for d = 1..W, evaluated by CPython as the reference does."""
    return [gamma ** (d - 1) for d in range(1, window + 1)]


def pow_table(decay: float, n: int) -> list[float]:
    return [decay ** j for j in range(n + 1)]


def drift_table(layers: int, dim: int) -> np.ndarray:
    """Cumulative per-layer hidden-state drift of the synthetic hidden-state
    model (predictor.py:36-44); row l = steps[:l+1].sum(axis=0)."""
    rng = np.random.default_rng(_DRIFT_SEED)
    steps = rng.normal(0.0, _DRIFT_STEP, size=(layers, dim))
    return np.stack([steps[: l + 1].sum(axis=0) for l in range(layers)]) if layers else np.zeros((0, dim))


class _DevicePredictor:
    trace = None

    def reset(self) -> None:
        pass

    def priorities(self, layer: int, token_ids=None) -> np.ndarray:
        ids = list(token_ids) if token_ids is not None else self.token_ids
        return self.device_table([layer], ids)[0].cpu().numpy()

    def predict(self, layer: int, budget: int, token_ids=None) -> list[int]:
        return predict_topb(self.priorities(layer, token_ids), budget)


class OraclePredictor(_DevicePredictor):
    def __init__(self, trace, token_ids=None, window: int = DEFAULT_WINDOW, gamma: float = DEFAULT_GAMMA):
        if window < 1:
            raise ValidationError("window must be >= 1")
        if not 0.0 < gamma <= 1.0:
            raise ValidationError("gamma must lie in (0, 1]")
        self.trace = trace
        self.token_ids = list(token_ids) if token_ids is not None else trace.prefill_ids()
        self.window = window
        self.gamma = gamma

    def device_table(self, ctx_layers, token_ids):
        dt = device_trace(self.trace)
        counts = kernels.demand_counts(dt.routes, dt.all_layers, dt.ids(token_ids), dt.E)
        dec = torch.tensor(decay_table(self.gamma, self.window), dtype=torch.float64, device=dt.device)
        ctx = torch.tensor(list(ctx_layers), dtype=torch.int32, device=dt.device)
        return kernels.oracle_targets(counts, ctx, self.window, dec)


class HistoryPredictor(_DevicePredictor):
    def __init__(self, trace, token_ids=None, decay: float = DEFAULT_HISTORY_DECAY):
        self.trace = trace
        self.token_ids = list(token_ids) if token_ids is not None else trace.prefill_ids()
        self.decay = decay

    def device_table(self, ctx_layers, token_ids):
        dt = device_trace(self.trace)
        counts = kernels.demand_counts(dt.routes, dt.all_layers, dt.ids(token_ids), dt.E)
        pw = torch.tensor(pow_table(self.decay, dt.L), dtype=torch.float64, device=dt.device)
        ctx = torch.tensor(list(ctx_layers), dtype=torch.int32, device=dt.device)
        return kernels.history(counts, ctx, pw)


class RandomPredictor:
    """Uniform scores from the reference's seeded PCG64 stream (host draws)."""

    def __init__(self, n_experts: int, seed: int = 0):
        self.n_experts = n_experts
        self.seed = seed
        self.rng = np.random.default_rng(seed)

    def reset(self) -> None:
        self.rng = np.random.default_rng(self.seed)

    def priorities(self, layer: int, token_ids=None) -> np.ndarray:
        return self.rng.random(self.n_experts)

    def predict(self, layer: int, budget: int, token_ids=None) -> list[int]:
        return predict_topb(self.priorities(layer), budget)


@dataclass
class MLPModel:
    """Bottleneck MLP weights (predictor.py:181-248); JSON format unchanged."""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    wo: np.ndarray
    bo: np.ndarray
    dropout_rate: float = 0.0
    final_loss: float = math.nan

    @property
    def dims(self) -> tuple[int, int, int, int]:
        return (self.w1.shape[1], self.w1.shape[0], self.w2.shape[0], self.wo.shape[0])

    def save(self, path: str) -> None:
        obj = {
            "version": MODEL_VERSION, "dims": list(self.dims), "dropout_rate": self.dropout_rate,
            "final_loss": self.final_loss,
            "weights": {k: np.asarray(getattr(self, k)).ravel().tolist() for k in ("w1", "b1", "w2", "b2", "wo", "bo")},
        }
        with open(path, "w", encoding="utf-8", newline="\n") as f:
            json.dump(obj, f)
            f.write("\n")

    @classmethod
    def load(cls, path: str) -> "MLPModel":
        with open(path, encoding="utf-8") as f:
            obj = json.load(f)
        d_in, d_h, d_b, n_out = obj["dims"]
        w = obj["weights"]
        a = lambda k, *s: np.asarray(w[k], dtype=np.float64).reshape(*s)  # noqa: E731
        return cls(a("w1", d_h, d_in), a("b1", d_h), a("w2", d_b, d_h), a("b2", d_b), a("wo", n_out, d_b),
                   a("bo", n_out), float(obj.get("dropout_rate", 0.0)), float(obj.get("final_loss", math.nan)))

    @classmethod
    def from_reference(cls, m) -> "MLPModel":
        return cls(*(np.asarray(getattr(m, k), dtype=np.float64) for k in ("w1", "b1", "w2", "b2", "wo", "bo")),
                   float(getattr(m, "dropout_rate", 0.0)), float(getattr(m, "final_loss", math.nan)))

    def to_device(self, device):
        return {k: torch.from_numpy(np.ascontiguousarray(getattr(self, k), dtype=np.float64)).to(device)
                for k in ("w1", "b1", "w2", "b2", "wo", "bo")}


class MLPPredictor(_DevicePredictor):
    def __init__(self, model, trace, plan=None, decay: float = DEFAULT_HISTORY_DECAY):
        self.model = model if isinstance(model, MLPModel) else MLPModel.from_reference(model)
        self.trace = trace
        self.plan = plan
        self.decay = decay
        dt = device_trace(trace)
        kept_visual = sorted(plan.keep) if plan is not None else trace.visual_ids()
        if kept_visual:
            # static mean of kept visual embeddings (visual_summary, predictor.py:78-83):
            # numpy reduces axis 0 row by row -> same order on the device
            self._h_v = _rowwise_mean(dt.embeddings, kept_visual)
        else:
            self._h_v = torch.zeros(trace.embed_dim, dtype=torch.float64, device=dt.device)
        self._w = self.model.to_device(dt.device)
        self._drift = torch.from_numpy(drift_table(trace.layers, trace.embed_dim)).to(dt.device)
        if self.model.dims[0] != trace.experts + 2 * trace.embed_dim:
            raise ValidationError(f"input dim {trace.experts + 2 * trace.embed_dim} != model dim {self.model.dims[0]}")
        self.token_ids = plan.retained_ids(trace) if plan is not None else trace.prefill_ids()

    def device_table(self, ctx_layers, token_ids=None, want_features=False):
        ids = list(token_ids) if token_ids is not None else self.token_ids
        if not ids:
            raise ContractError("retained token set must be non-empty")
        if self.plan is not None and self.plan.config.prefix_layers and min(ctx_layers) < max(self.plan.config.prefix_layers):
            raise ContractError("features need the full pinned prefix realized")
        dt = device_trace(self.trace)
        d_ids = dt.ids(ids)
        counts = kernels.demand_counts(dt.routes, dt.all_layers, d_ids, dt.E)
        pw = torch.tensor(pow_table(self.decay, dt.L), dtype=torch.float64, device=dt.device)
        ctx = torch.tensor(list(ctx_layers), dtype=torch.int32, device=dt.device)
        hist = kernels.history(counts, ctx, pw)
        y, feat = kernels.mlp_predict(hist, dt.embeddings, self._drift, d_ids, self._h_v, ctx, self._w,
                                      want_features=want_features)
        return (y, feat) if want_features else y


def _rowwise_mean(emb: torch.Tensor, rows) -> torch.Tensor:
    """Column means accumulated row by row (numpy's axis-0 add.reduce order)."""
    sel = emb.index_select(0, torch.as_tensor(list(rows), dtype=torch.long, device=emb.device))
    acc = torch.zeros(emb.shape[1], dtype=torch.float64, device=emb.device)
    for r in range(sel.shape[0]):
        acc = acc + sel[r]
    # divide by a device tensor: torch turns division by a CPU scalar into a
    # reciprocal multiply, which is not the correctly rounded quotient numpy computes
    return acc / torch.full_like(acc, float(sel.shape[0]))


def build_targets(trace, layer: int, window: int = DEFAULT_WINDOW, gamma: float = DEFAULT_GAMMA, token_ids=None):
    ids = list(token_ids) if token_ids is not None else trace.prefill_ids()
    return OraclePredictor(trace, ids, window, gamma).priorities(layer, ids)


def routing_histogram(trace, token_ids, layer: int, decay: float):
    return HistoryPredictor(trace, list(token_ids), decay).priorities(layer, list(token_ids))


def hot_recall(predicted, trace, layer: int, token_ids=None) -> float:
    ids = list(token_ids) if token_ids is not None else trace.prefill_ids()
    actual = trace.active_union(layer + 1, ids)
    if not actual:
        return 1.0
    return len(set(predicted) & actual) / len(actual)
