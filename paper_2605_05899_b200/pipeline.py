"""Planning, the logical-clock engine driver and reports (drop-in for
`pkg/src/moesim/pipeline.py`).

`simulate` / `simulate_reactive` keep the reference signatures and return a
`SimReport` with the same fields.  The per-layer work is split the B200 way:

  * demand sets for every layer (`active_union`) come from ONE device launch
    of `vmm_demand_counts` over the retained tokens (plus one for the pinned
    prefix over all prefill tokens, one per decode token);
  * predictor scores for every emission come from ONE batched device launch
    (`device_table`: oracle targets / history histogram / MLP);
  * the cache policy and transfer channel run in the native engine
    (csrc/engine.cpp), which reproduces the reference's decisions exactly.

Hybrid CPU dispatch (pipeline.py:587-628, `simulate_hybrid`) is out of scope:
the device path has no CPU fallback, so a finite hybrid threshold is rejected.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib, kernels
from ._lib import EngineConfig, EngineEvent, EngineReport, check
from .compress import CompressionConfig, CompressionPlan, compress
from .device_trace import device_trace
from .errors import PlanningError, SimulationError, ValidationError
from .predictor import (
    DEFAULT_BUDGET, DEFAULT_GAMMA, DEFAULT_HISTORY_DECAY, DEFAULT_WINDOW, HistoryPredictor, MLPPredictor,
    OraclePredictor, RandomPredictor, decay_table,
)
from .trace import ExpertRef

DEFAULT_COMPRESS_MS = 14.70  # pipeline.py:47-48
DEFAULT_PREDICTOR_BOOTSTRAP_MS = 2.72


@dataclass(frozen=True)
class PrefixPlan:
    lo: int
    hi: int
    chosen: int


def plan_prefix(m_avail_mb, s_layer_mb, c_safe_mb, l_semantic, override=None) -> PrefixPlan:
    """Eq. 9 pinned-prefix interval (pipeline.py:63-90)."""
    if s_layer_mb <= 0 or m_avail_mb <= 0 or c_safe_mb < 0:
        raise PlanningError("memory quantities must be positive")
    if l_semantic < 0:
        raise PlanningError("l_semantic must be >= 0")
    hi = math.floor((m_avail_mb - c_safe_mb) / s_layer_mb)
    if hi < l_semantic:
        raise PlanningError("insufficient memory for semantic prefix")
    chosen = l_semantic
    if override is not None:
        if not l_semantic <= override <= hi:
            raise PlanningError(f"prefix override {override} outside valid interval [{l_semantic}, {hi}]")
        chosen = override
    return PrefixPlan(lo=l_semantic, hi=hi, chosen=chosen)


@dataclass
class MemoryBudget:
    m_avail_mb: float
    c_safe_mb: float
    static_resident_mb: float = 0.0


@dataclass
class PredictorSpec:
    kind: str = "oracle"  # oracle | random | history | mlp | none
    budget: int = DEFAULT_BUDGET
    window: int = DEFAULT_WINDOW
    gamma: float = DEFAULT_GAMMA
    history_decay: float = DEFAULT_HISTORY_DECAY


@dataclass
class SimConfig:
    bandwidth_mb_per_ms: float = 10.0
    expert_size_mb: float = 17.3
    gpu_ms_per_expert: float = 1.0
    cpu_ms_per_expert: float = math.inf
    hybrid_threshold_ms: float = math.inf
    memory: MemoryBudget | None = None
    l_semantic: int = 1
    l_pinned: int | None = None
    predictor: PredictorSpec = field(default_factory=PredictorSpec)
    num_slabs: int | None = None
    decode_steps: int = 0
    seed: int = 0
    speculative_grace: int = 1
    victim_policy: str = "priority"
    compress_latency_ms: float = DEFAULT_COMPRESS_MS
    predictor_bootstrap_ms: float = DEFAULT_PREDICTOR_BOOTSTRAP_MS
    shared_experts: int = 0
    event_log: bool = False

    def validate(self) -> None:  # pipeline.py:130-146
        if not self.bandwidth_mb_per_ms > 0:
            raise ValidationError("bandwidth_mb_per_ms must be > 0")
        if not self.expert_size_mb > 0:
            raise ValidationError("expert_size_mb must be > 0")
        if self.gpu_ms_per_expert < 0:
            raise ValidationError("gpu_ms_per_expert must be >= 0")
        if self.cpu_ms_per_expert <= 0:
            raise ValidationError("cpu_ms_per_expert must be > 0")
        if self.decode_steps < 0:
            raise ValidationError("decode_steps must be >= 0")
        if self.speculative_grace < 0:
            raise ValidationError("speculative_grace must be >= 0")
        if self.victim_policy not in ("priority", "fifo"):
            raise ValidationError("victim_policy must be 'priority' or 'fifo'")
        if self.compress_latency_ms < 0 or self.predictor_bootstrap_ms < 0:
            raise ValidationError("bootstrap latencies must be >= 0")

    @property
    def transfer_ms(self) -> float:
        return self.expert_size_mb / self.bandwidth_mb_per_ms


@dataclass
class ExecutionPlan:
    l_pinned: int
    num_slabs: int
    compression: CompressionPlan | None = None
    predictor: object | None = None

    def pinned_keys(self, trace) -> set:
        return {ExpertRef(l, e) for l in range(self.l_pinned) for e in range(trace.experts)}

    def retained_ids(self, trace) -> list[int]:
        if self.compression is None:
            return trace.prefill_ids()
        return self.compression.retained_ids(trace)


def build_predictor(trace, plan: ExecutionPlan, cfg: SimConfig, model=None):
    spec = cfg.predictor
    tokens = plan.retained_ids(trace)
    if spec.kind == "none":
        return None
    if spec.kind == "oracle":
        return OraclePredictor(trace, tokens, spec.window, spec.gamma)
    if spec.kind == "random":
        return RandomPredictor(trace.experts, cfg.seed)
    if spec.kind == "history":
        return HistoryPredictor(trace, tokens, spec.history_decay)
    if spec.kind == "mlp":
        if model is None:
            raise ValidationError("mlp predictor requires a trained model")
        return MLPPredictor(model, trace, plan.compression, spec.history_decay)
    raise ValidationError(f"unknown predictor kind '{spec.kind}'")


def build_plan(trace, cfg: SimConfig, compression_cfg: CompressionConfig | None = None, model=None) -> ExecutionPlan:
    """Resolve prefix depth, slab count, compression and predictor (pipeline.py:191-226)."""
    cfg.validate()
    if cfg.memory is not None:
        s_layer = trace.experts * cfg.expert_size_mb
        prefix = plan_prefix(cfg.memory.m_avail_mb, s_layer, cfg.memory.c_safe_mb, cfg.l_semantic, cfg.l_pinned)
        l_pinned = prefix.chosen
        num_slabs = cfg.num_slabs
        if num_slabs is None:
            num_slabs = math.floor(cfg.memory.c_safe_mb / cfg.expert_size_mb)
        if l_pinned * s_layer + cfg.memory.c_safe_mb > cfg.memory.m_avail_mb:
            raise PlanningError("pinned prefix plus cache reserve exceeds available memory")
    else:
        l_pinned = cfg.l_pinned if cfg.l_pinned is not None else cfg.l_semantic
        if cfg.num_slabs is None:
            raise PlanningError("num_slabs required when no memory budget is given")
        num_slabs = cfg.num_slabs
    if not 0 <= l_pinned <= trace.layers:
        raise PlanningError("pinned prefix depth outside the trace's layer range")
    if num_slabs < 1:
        raise PlanningError("cache needs at least one slab")
    comp = compress(trace, compression_cfg) if compression_cfg is not None else None
    plan = ExecutionPlan(l_pinned=l_pinned, num_slabs=num_slabs, compression=comp)
    plan.predictor = build_predictor(trace, plan, cfg, model)
    if plan.predictor is not None and l_pinned < 1 and cfg.predictor.kind != "random":
        raise PlanningError("lookahead prediction needs at least one pinned layer of context")
    return plan


# ---------------------------------------------------------------------------
# reports
# ---------------------------------------------------------------------------
@dataclass
class LayerStat:
    phase: str
    step: int
    layer: int
    start: float
    end: float
    stall_ms: float
    transfers: int
    hits: int


REPORT_COLUMNS = [
    "makespan", "total_compute", "total_transfer", "exposed_transfer", "overlapped_transfer", "hits", "misses",
    "hit_rate", "stalls", "rejected_loads", "cpu_dispatches", "on_demand_transfers", "inflight_waits", "evictions",
    "prefill_ms", "decode_steps",
]


@dataclass
class SimReport:
    makespan: float
    total_compute: float
    total_transfer: float
    exposed_transfer: float
    hits: int
    misses: int
    stalls: int
    rejected_loads: int
    cpu_dispatches: int
    on_demand_transfers: int
    inflight_waits: int
    evictions: int
    prefill_ms: float
    decode_ms_per_step: list[float]
    per_layer: list[LayerStat]
    events: list[tuple] = field(default_factory=list)

    @property
    def hit_rate(self) -> float:
        total = self.hits + self.misses
        return self.hits / total if total else 1.0

    @property
    def overlapped_transfer(self) -> float:
        return self.total_transfer - self.exposed_transfer

    def to_dict(self) -> dict:
        return {
            "makespan": self.makespan, "total_compute": self.total_compute, "total_transfer": self.total_transfer,
            "exposed_transfer": self.exposed_transfer, "overlapped_transfer": self.overlapped_transfer,
            "hits": self.hits, "misses": self.misses, "hit_rate": self.hit_rate, "stalls": self.stalls,
            "rejected_loads": self.rejected_loads, "cpu_dispatches": self.cpu_dispatches,
            "on_demand_transfers": self.on_demand_transfers, "inflight_waits": self.inflight_waits,
            "evictions": self.evictions, "prefill_ms": self.prefill_ms, "decode_ms_per_step": self.decode_ms_per_step,
            "per_layer": [[s.phase, s.step, s.layer, s.start, s.end, s.stall_ms, s.transfers, s.hits]
                          for s in self.per_layer],
        }

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, indent=2)


_EV_KIND = {0: "issue", 1: "complete", 2: "evict"}


class Engine:
    """Owning wrapper of the native logical-clock engine (one request)."""

    def __init__(self, layers, experts, cfg: SimConfig, num_slabs, l_pinned, shared, prefetching, reactive,
                 boot_ms):
        self._L = _lib.load()
        w = cfg.predictor.window
        self._decay = np.asarray(decay_table(cfg.predictor.gamma, max(w, 1)), dtype=np.float64)
        c = EngineConfig(
            layers=layers, experts=experts, num_slabs=num_slabs, victim_fifo=int(cfg.victim_policy == "fifo"),
            speculative_grace=cfg.speculative_grace, budget=cfg.predictor.budget, window=w, l_pinned=l_pinned,
            shared=shared, prefetching=int(prefetching), reactive=int(reactive), event_log=int(cfg.event_log),
            transfer_ms=cfg.transfer_ms, gpu_ms=cfg.gpu_ms_per_expert, boot_ms=boot_ms,
            decay=self._decay.ctypes.data_as(C.POINTER(C.c_double)),
        )
        self._cfg = c
        h = C.c_void_p()
        check(self._L.vmm_engine_create(C.byref(c), C.byref(h)))
        self._h = h
        self.layers = layers
        self.experts = experts

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.vmm_engine_destroy(h)
            self._h = None

    @staticmethod
    def _y(y):
        if y is None:
            return None, None
        a = np.ascontiguousarray(y, dtype=np.float64)
        return a, a.ctypes.data

    def begin(self, y=None):
        a, p = self._y(y)
        check(self._L.vmm_engine_begin(self._h, p))

    def emits(self, layer: int, phase: int) -> bool:
        return bool(self._L.vmm_engine_emits(self._h, layer, phase))

    def layer(self, layer: int, demand, phase: int, step: int, y=None):
        d = np.ascontiguousarray(demand, dtype=np.int32)
        a, p = self._y(y)
        check(self._L.vmm_engine_layer(self._h, layer, d.ctypes.data, len(d), phase, step, p))

    def end_step(self):
        check(self._L.vmm_engine_end_step(self._h))

    def copies(self) -> np.ndarray:
        out = []
        buf = np.empty((4096, 3), dtype=np.int32)
        while True:
            n = self._L.vmm_engine_copies(self._h, buf.ctypes.data, 4096)
            if n <= 0:
                break
            out.append(buf[:n].copy())
        return np.concatenate(out) if out else np.zeros((0, 3), dtype=np.int32)

    def slab_of(self, layer: int, expert: int) -> int:
        return self._L.vmm_engine_slab_of(self._h, layer, expert)

    def events(self) -> list[tuple]:
        n = self._L.vmm_engine_pending_events(self._h)
        if n <= 0:
            return []
        buf = (EngineEvent * n)()
        m = self._L.vmm_engine_events(self._h, buf, n)
        return [(buf[i].t, _EV_KIND[buf[i].kind], buf[i].layer, buf[i].expert) for i in range(m)]

    def finish(self, with_events: bool) -> SimReport:
        r = EngineReport()
        check(self._L.vmm_engine_finish(self._h, C.byref(r)))
        rows = self.__dict__.setdefault("_rows", [])  # drained rows accumulate: finish() may be called again
        buf = np.empty((1024, 8), dtype=np.float64)
        while True:
            n = self._L.vmm_engine_layer_stats(self._h, buf.ctypes.data, 1024)
            if n <= 0:
                break
            rows.extend(buf[:n].tolist())
        dec = np.empty(max(r.decode_steps, 1), dtype=np.float64)
        nd = self._L.vmm_engine_decode_ms(self._h, dec.ctypes.data, len(dec))
        per_layer = [LayerStat("prefill" if int(x[0]) == 0 else "decode", int(x[1]), int(x[2]), x[3], x[4], x[5],
                               int(x[6]), int(x[7])) for x in rows]
        return SimReport(
            makespan=r.makespan, total_compute=r.total_compute, total_transfer=r.total_transfer,
            exposed_transfer=r.exposed_transfer, hits=r.hits, misses=r.misses, stalls=r.stalls,
            rejected_loads=r.rejected_loads, cpu_dispatches=0, on_demand_transfers=r.on_demand_transfers,
            inflight_waits=r.inflight_waits, evictions=r.evictions, prefill_ms=r.prefill_ms,
            decode_ms_per_step=dec[:nd].tolist(), per_layer=per_layer,
            events=self.events() if with_events else [],
        )


def _demand_lists(counts: np.ndarray) -> list[np.ndarray]:
    return [np.flatnonzero(row).astype(np.int32) for row in counts]


class _Scores:
    """Predictor scores for every emission, batched on the device when possible."""

    def __init__(self, predictor, ctx_layers, ids):
        self.pred = predictor
        self.table = None
        if predictor is not None and hasattr(predictor, "device_table") and ctx_layers:
            self.table = predictor.device_table(list(ctx_layers), ids).cpu().numpy()
            self.index = {c: i for i, c in enumerate(ctx_layers)}

    def get(self, ctx, ids):
        if self.table is not None and ctx in self.index:
            return self.table[self.index[ctx]]
        return self.pred.priorities(ctx, ids)


def _run(trace, plan: ExecutionPlan, cfg: SimConfig, reactive: bool) -> SimReport:
    cfg.validate()
    if math.isfinite(cfg.cpu_ms_per_expert) and math.isfinite(cfg.hybrid_threshold_ms):
        raise ValidationError("hybrid CPU dispatch is out of scope for the device path (no CPU fallback)")
    if plan.l_pinned > trace.layers:
        raise SimulationError("plan pins more layers than the trace has")
    predictor = plan.predictor if not reactive else None
    if predictor is not None and hasattr(predictor, "reset"):
        predictor.reset()
    prefetching = predictor is not None and cfg.predictor.budget > 0
    L, E = trace.layers, trace.experts
    lp = plan.l_pinned
    shared = cfg.shared_experts or trace.shared_experts
    boot = (cfg.compress_latency_ms if plan.compression is not None else 0.0) + (
        cfg.predictor_bootstrap_ms if prefetching else 0.0)
    eng = Engine(L, E, cfg, plan.num_slabs, lp, shared, prefetching, reactive, boot)

    dt = device_trace(trace)
    retained = plan.retained_ids(trace)
    all_prefill = trace.prefill_ids()
    counts_ret = kernels.demand_counts(dt.routes, dt.all_layers, dt.ids(retained), E)
    counts_pre = kernels.demand_counts(dt.routes, dt.all_layers, dt.ids(all_prefill), E) if lp > 0 else None
    ctx_prefill = ([lp - 1] if lp > 0 else []) + [l for l in range(max(lp, 0), L - 1)]
    scores = _Scores(predictor if prefetching else None, ctx_prefill if prefetching else [], retained)
    dem_ret = _demand_lists(counts_ret.cpu().numpy())
    dem_pre = _demand_lists(counts_pre.cpu().numpy()) if counts_pre is not None else None

    try:
        eng.begin(scores.get(lp - 1, retained) if prefetching and lp > 0 else None)
        for layer in range(L):
            dem = dem_pre[layer] if layer < lp else dem_ret[layer]
            y = scores.get(layer, retained) if eng.emits(layer, 0) else None
            eng.layer(layer, dem, 0, -1, y)
        steps = trace.phase_marks[: cfg.decode_steps]
        for s, tok in enumerate(steps):
            c = kernels.demand_counts(dt.routes, dt.all_layers, dt.ids([tok]), E).cpu().numpy()
            dscores = _Scores(predictor if prefetching else None,
                              [l for l in range(L) if eng.emits(l, 1)] if prefetching else [], [tok])
            for layer in range(L):
                y = dscores.get(layer, [tok]) if eng.emits(layer, 1) else None
                eng.layer(layer, np.flatnonzero(c[layer]).astype(np.int32), 1, s, y)
            eng.end_step()
    except SimulationError:
        raise
    return eng.finish(with_events=cfg.event_log)


def simulate(trace, plan: ExecutionPlan, cfg: SimConfig) -> SimReport:
    """Pipelined run with lookahead prefetch if a predictor is attached (pipeline.py:768-771)."""
    return _run(trace, plan, cfg, reactive=False)


def simulate_reactive(trace, plan: ExecutionPlan, cfg: SimConfig) -> SimReport:
    """No-prefetch control: every miss transfers serially before its compute (pipeline.py:774-776)."""
    return _run(trace, plan, cfg, reactive=True)
