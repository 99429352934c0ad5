"""Routing-trace data contract and synthetic input source.

The trace is the router -> compressor/cache contract of the reference
(`pkg/src/moesim/trace.py:65-147`): ``route_experts[l, t]`` holds the k
distinct experts token ``t`` activates at layer ``l`` and ``route_gates`` the
matching positive gate weights that sum to one.  This module keeps that layout
but stores token metadata column-wise (structure of arrays) so it can be
uploaded to HBM in one copy per field:

    saliency   f64 [N]      attention-derived importance (trace.py:49)
    modality   u8  [N]      0 visual, 1 text                (trace.py:33-35)
    embedding  f64 [N, D]   synthetic token embedding       (trace.py:50)
    cluster    i64 [N]      generator latent cluster        (trace.py:51)

`generate_trace` is the CPU-side synthetic input source.  It consumes one
seeded PCG64 stream in exactly the order the reference generator does
(`trace.py:265-348`), so a given config yields byte-identical arrays; this is
pinned against fixtures produced by the reference (tests/golden).  It is input
synthesis, not part of the device hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import NamedTuple

import numpy as np

from .errors import ValidationError

TRACE_VERSION = 1
_SUPPORT_DECAY = 0.6  # trace.py:29
_EMBED_NOISE = 0.15  # trace.py:30

MOD_VISUAL = 0
MOD_TEXT = 1
MOD_DECODE = 2  # device-side tag: token belongs to the decode phase


class Modality(str, Enum):
    VISUAL = "visual"
    TEXT = "text"


class ExpertRef(NamedTuple):
    """(layer, expert) identity of one expert's weights (trace.py:38-42)."""

    layer: int
    expert: int


@dataclass(eq=False)
class Token:
    """Row view of one token (trace.py:46-62); built on demand."""

    id: int
    modality: Modality
    saliency: float
    embedding: np.ndarray
    cluster: int = -1


class RoutingTrace:
    """Per-layer, per-token routes plus column-wise token metadata."""

    def __init__(
        self,
        layers: int,
        experts: int,
        k: int,
        route_experts: np.ndarray,
        route_gates: np.ndarray,
        saliency: np.ndarray,
        modality: np.ndarray,
        embedding: np.ndarray,
        cluster: np.ndarray | None = None,
        phase_marks=(),
        shared_experts: int = 0,
    ):
        self.layers = int(layers)
        self.experts = int(experts)
        self.k = int(k)
        self.route_experts = np.ascontiguousarray(route_experts, dtype=np.int64)
        self.route_gates = np.ascontiguousarray(route_gates, dtype=np.float64)
        self.saliency = np.ascontiguousarray(saliency, dtype=np.float64)
        self.modality = np.ascontiguousarray(modality, dtype=np.uint8)
        self.embedding = np.ascontiguousarray(embedding, dtype=np.float64)
        n = self.saliency.shape[0]
        self.cluster = (
            np.full(n, -1, dtype=np.int64) if cluster is None else np.asarray(cluster, dtype=np.int64)
        )
        self.phase_marks = [int(m) for m in phase_marks]
        self.shared_experts = int(shared_experts)
        self._tokens = None

    # -- geometry ------------------------------------------------------------
    @property
    def num_tokens(self) -> int:
        return int(self.saliency.shape[0])

    @property
    def embed_dim(self) -> int:
        return int(self.embedding.shape[1]) if self.embedding.ndim == 2 and self.num_tokens else 0

    # -- id lists (trace.py:109-127) ----------------------------------------
    def _decode_mask(self) -> np.ndarray:
        m = np.zeros(self.num_tokens, dtype=bool)
        if self.phase_marks:
            m[np.asarray(self.phase_marks, dtype=np.int64)] = True
        return m

    def device_modality(self) -> np.ndarray:
        """u8 tag per token for the device: visual / text / decode."""
        tag = self.modality.copy()
        tag[self._decode_mask()] = MOD_DECODE
        return tag

    def prefill_ids(self) -> list[int]:
        return np.flatnonzero(~self._decode_mask()).tolist()

    def visual_ids(self) -> list[int]:
        return np.flatnonzero((self.modality == MOD_VISUAL) & ~self._decode_mask()).tolist()

    def text_ids(self) -> list[int]:
        return np.flatnonzero((self.modality == MOD_TEXT) & ~self._decode_mask()).tolist()

    # -- route queries (trace.py:96-107) --------------------------------------
    def route(self, layer: int, token: int) -> np.ndarray:
        return self.route_experts[layer, token]

    def route_set(self, layer: int, token: int) -> set[int]:
        return set(int(e) for e in self.route_experts[layer, token])

    def active_union(self, layer: int, token_ids) -> set[int]:
        ids = np.asarray(list(token_ids), dtype=np.int64)
        if ids.size == 0:
            return set()
        return set(np.unique(self.route_experts[layer, ids]).tolist())

    def embeddings(self) -> np.ndarray:
        return self.embedding

    @property
    def tokens(self) -> list[Token]:
        if self._tokens is None:
            self._tokens = [
                Token(
                    id=i,
                    modality=Modality.VISUAL if self.modality[i] == MOD_VISUAL else Modality.TEXT,
                    saliency=float(self.saliency[i]),
                    embedding=self.embedding[i],
                    cluster=int(self.cluster[i]),
                )
                for i in range(self.num_tokens)
            ]
        return self._tokens

    # -- interop -------------------------------------------------------------
    @classmethod
    def from_reference(cls, ref) -> "RoutingTrace":
        """Wrap a reference ``moesim.RoutingTrace`` (or any duck-typed object
        with ``tokens``/``route_experts``/``route_gates``).  Token ids must be
        their list positions, as every reference constructor produces."""
        toks = list(ref.tokens)
        for i, t in enumerate(toks):
            if int(t.id) != i:
                raise ValidationError("token ids must equal their positions")
        n = len(toks)
        d = int(toks[0].embedding.shape[0]) if n else 0
        emb = np.zeros((n, d), dtype=np.float64)
        for i, t in enumerate(toks):
            emb[i] = t.embedding
        mod = np.array(
            [MOD_VISUAL if getattr(t.modality, "value", t.modality) == "visual" else MOD_TEXT for t in toks],
            dtype=np.uint8,
        )
        return cls(
            ref.layers, ref.experts, ref.k, ref.route_experts, ref.route_gates,
            np.array([float(t.saliency) for t in toks], dtype=np.float64), mod, emb,
            np.array([int(getattr(t, "cluster", -1)) for t in toks], dtype=np.int64),
            list(ref.phase_marks), int(getattr(ref, "shared_experts", 0)),
        )

    __hash__ = object.__hash__  # identity hash: device copies are cached per object

    def __eq__(self, other):
        if not isinstance(other, RoutingTrace):
            return NotImplemented
        return (
            (self.layers, self.experts, self.k, self.shared_experts, self.phase_marks)
            == (other.layers, other.experts, other.k, other.shared_experts, other.phase_marks)
            and np.array_equal(self.route_experts, other.route_experts)
            and np.array_equal(self.route_gates, other.route_gates)
            and np.array_equal(self.saliency, other.saliency)
            and np.array_equal(self.modality, other.modality)
            and np.array_equal(self.embedding, other.embedding)
        )


def validate_trace(trace: RoutingTrace) -> list[str]:
    """Invariant violations (trace.py:351-387), vectorised."""
    out: list[str] = []
    sal = trace.saliency
    bad = ~np.isfinite(sal) | (sal < 0)
    for t in np.flatnonzero(bad)[:5]:
        out.append(f"token {int(t)}: saliency must be finite and >= 0")
    re = trace.route_experts
    if re.shape != (trace.layers, trace.num_tokens, trace.k):
        out.append("routes: table shape disagrees with header geometry")
        return out
    if re.size:
        srt = np.sort(re, axis=2)
        dup = (srt[:, :, 1:] == srt[:, :, :-1]).any(axis=2)
        for l, t in np.argwhere(dup)[:5]:
            out.append(f"layer {int(l)} token {int(t)}: route has duplicate experts")
        oor = ((re < 0) | (re >= trace.experts)).any(axis=2)
        for l, t in np.argwhere(oor)[:5]:
            out.append(f"layer {int(l)} token {int(t)}: expert id out of range")
        g = trace.route_gates
        gbad = (~np.isfinite(g) | (g <= 0)).any(axis=2)
        for l, t in np.argwhere(gbad)[:5]:
            out.append(f"layer {int(l)} token {int(t)}: gates must be finite and > 0")
        gs = np.abs(g.sum(axis=2) - 1.0) > 1e-6
        for l, t in np.argwhere(gs & ~gbad)[:5]:
            out.append(f"layer {int(l)} token {int(t)}: gates must sum to 1")
    for m in trace.phase_marks:
        if not 0 <= m < trace.num_tokens:
            out.append(f"phase mark {m}: token id out of range")
    return out


# ---------------------------------------------------------------------------
# Synthetic generator (input source; same draw order as trace.py:208-348)
# ---------------------------------------------------------------------------


@dataclass
class TraceGenConfig:
    n_visual: int
    n_text: int
    layers: int
    experts: int
    k: int
    clusters: int = 4
    cluster_support: int = 8
    rho: float = 0.8
    visual_noise: float = 0.0
    saliency_shape: tuple[float, float] = (2.0, 1.0)
    embed_dim: int = 16
    decode_steps: int = 0
    seed: int = 0
    shared_experts: int = 0

    def validate(self) -> None:
        c = self
        checks = [
            (c.n_visual >= 0, "n_visual must be >= 0"),
            (c.n_text >= 0, "n_text must be >= 0"),
            (c.n_visual + c.n_text >= 1, "n_visual + n_text must be >= 1"),
            (c.layers >= 1, "layers must be >= 1"),
            (c.experts >= 1, "experts must be >= 1"),
            (1 <= c.k <= c.experts, "k must satisfy 1 <= k <= experts"),
            (c.clusters >= 1, "clusters must be >= 1"),
            (c.k <= c.cluster_support <= c.experts, "cluster_support must satisfy k <= cluster_support <= experts"),
            (0.0 <= c.rho <= 1.0, "rho must lie in [0, 1]"),
            (0.0 <= c.visual_noise <= 1.0, "visual_noise must lie in [0, 1]"),
            (c.saliency_shape[0] > 0 and c.saliency_shape[1] > 0, "saliency_shape parameters must be > 0"),
            (c.embed_dim >= 1, "embed_dim must be >= 1"),
            (c.decode_steps >= 0, "decode_steps must be >= 0"),
            (c.shared_experts >= 0, "shared_experts must be >= 0"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValidationError(msg)


class _Preference:
    """One latent cluster: a decaying categorical over `support` experts."""

    __slots__ = ("n_experts", "support", "cdf", "support_set")

    def __init__(self, rng: np.random.Generator, n_experts: int, size: int):
        self.n_experts = n_experts
        self.support = [int(e) for e in rng.choice(n_experts, size=size, replace=False)]
        w = _SUPPORT_DECAY ** np.arange(size)
        self.cdf = np.cumsum(w / w.sum())

    def sample(self, rng: np.random.Generator, taken) -> int:
        support, cdf = self.support, self.cdf
        for _ in range(64):
            e = support[int(np.searchsorted(cdf, rng.random()))]
            if e not in taken:
                return e
        for e in support:
            if e not in taken:
                return e
        return _uniform_excluding(rng, self.n_experts, taken)


def _uniform_excluding(rng: np.random.Generator, n: int, taken) -> int:
    while True:
        e = int(rng.integers(n))
        if e not in taken:
            return e


def _advance_route(rng, prev: list[int], pref: _Preference, rho: float, noise: float, n: int) -> list[int]:
    k = len(prev)
    survive = [rng.random() < rho for _ in range(k)]
    nxt = [p if s else -1 for p, s in zip(prev, survive)]
    present = {e for e in nxt if e >= 0}
    for j in range(k):
        if nxt[j] < 0:
            e = pref.sample(rng, present)
            nxt[j] = e
            present.add(e)
    if noise > 0.0:
        for j in range(k):
            if survive[j] and rng.random() < noise:
                rest = {e for i, e in enumerate(nxt) if i != j}
                e = _uniform_excluding(rng, n, rest)
                present.discard(nxt[j])
                nxt[j] = e
                present.add(e)
    return nxt


def generate_trace(cfg: TraceGenConfig) -> RoutingTrace:
    """Deterministic synthetic trace; same config -> same arrays as the reference."""
    cfg.validate()
    rng = np.random.default_rng(cfg.seed)
    L, E, k = cfg.layers, cfg.experts, cfg.k
    n_pre = cfg.n_visual + cfg.n_text
    n_all = n_pre + cfg.decode_steps

    prefs = [_Preference(rng, E, cfg.cluster_support) for _ in range(cfg.clusters)]
    cl = rng.integers(0, cfg.clusters, size=n_pre).astype(np.int64)
    dec_cl = int(rng.integers(0, cfg.clusters)) if cfg.decode_steps else 0
    cluster = np.concatenate([cl, np.full(cfg.decode_steps, dec_cl, dtype=np.int64)])

    shape, scale = cfg.saliency_shape
    saliency = rng.gamma(shape, scale, size=n_all)
    centers = rng.normal(size=(cfg.clusters, cfg.embed_dim))
    centers /= np.linalg.norm(centers, axis=1, keepdims=True)
    emb = centers[cluster] + _EMBED_NOISE * rng.normal(size=(n_all, cfg.embed_dim))

    routes = np.zeros((L, n_all, k), dtype=np.int64)
    gates = np.zeros((L, n_all, k), dtype=np.float64)
    ones = np.ones(k)

    def chain(t: int, noise: float) -> None:
        pref = prefs[int(cluster[t])]
        r: list[int] = []
        for _ in range(k):
            r.append(pref.sample(rng, set(r)))
        routes[0, t] = r
        gates[0, t] = rng.dirichlet(ones)
        for l in range(1, L):
            r = _advance_route(rng, r, pref, cfg.rho, noise, E)
            routes[l, t] = r
            gates[l, t] = rng.dirichlet(ones)

    for t in range(n_pre):
        chain(t, cfg.visual_noise if t < cfg.n_visual else 0.0)
    for s in range(cfg.decode_steps):
        t = n_pre + s
        if s == 0:
            chain(t, 0.0)
            continue
        pref = prefs[dec_cl]
        for l in range(L):
            routes[l, t] = _advance_route(rng, [int(e) for e in routes[l, t - 1]], pref, cfg.rho, 0.0, E)
            gates[l, t] = rng.dirichlet(ones)

    modality = np.where(np.arange(n_all) < cfg.n_visual, MOD_VISUAL, MOD_TEXT).astype(np.uint8)
    return RoutingTrace(
        L, E, k, routes, gates, saliency, modality, emb.astype(np.float64), cluster,
        list(range(n_pre, n_all)), cfg.shared_experts,
    )


def trace_digest(trace: RoutingTrace) -> str:
    """sha256 over every array of the trace (fixture pinning)."""
    import hashlib

    h = hashlib.sha256()
    for a in (trace.route_experts, trace.route_gates, trace.saliency, trace.modality, trace.embedding, trace.cluster):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(repr((trace.layers, trace.experts, trace.k, trace.phase_marks, trace.shared_experts)).encode())
    return h.hexdigest()


# ---------------------------------------------------------------------------
# Binary trace ingest: replaces the JSON-Lines format of
# trace.py:390-503 for the device path.  One little-endian file:
#   magic b"VMMTRACE" | u32 version | u32 L, E, k, N, D, shared, n_marks
#   | i32 phase_marks[n_marks] | u8 modality[N] | f64 saliency[N]
#   | i64 cluster[N] | f64 embedding[N*D] | i32 route_experts[L*N*k]
#   | f64 route_gates[L*N*k]
# Arrays are stored in the device layout (routes layer-major i32), so loading is
# a few np.fromfile reads (memory-mapped on request) and one H2D per array,
# instead of ~L*N JSON records.  Gates keep full fp64 (exact round trip).
# ---------------------------------------------------------------------------
BIN_MAGIC = b"VMMTRACE"
BIN_VERSION = 1


def save_trace_bin(trace: RoutingTrace, path: str) -> None:
    hdr = np.array([BIN_VERSION, trace.layers, trace.experts, trace.k, trace.num_tokens, trace.embed_dim,
                    trace.shared_experts, len(trace.phase_marks)], dtype="<u4")
    with open(path, "wb") as f:
        f.write(BIN_MAGIC)
        f.write(hdr.tobytes())
        f.write(np.asarray(trace.phase_marks, dtype="<i4").tobytes())
        f.write(np.ascontiguousarray(trace.modality, dtype="u1").tobytes())
        f.write(np.ascontiguousarray(trace.saliency, dtype="<f8").tobytes())
        f.write(np.ascontiguousarray(trace.cluster, dtype="<i8").tobytes())
        f.write(np.ascontiguousarray(trace.embedding, dtype="<f8").tobytes())
        f.write(np.ascontiguousarray(trace.route_experts, dtype="<i4").tobytes())
        f.write(np.ascontiguousarray(trace.route_gates, dtype="<f8").tobytes())


def load_trace_bin(path: str, mmap: bool = False) -> RoutingTrace:
    """Parse a binary trace; ParseError on a malformed file, ValidationError on
    invariant violations (the same checks as the reference's load_trace)."""
    from .errors import ParseError

    with open(path, "rb") as f:
        head = f.read(8 + 4 * 8)
    if len(head) < 40 or head[:8] != BIN_MAGIC:
        raise ParseError(f"{path}: not a VMMTRACE file")
    ver, L, E, k, N, D, shared, nm = (int(v) for v in np.frombuffer(head[8:], dtype="<u4"))
    if ver != BIN_VERSION:
        raise ParseError(f"{path}: unsupported version {ver}")
    sizes = [("marks", "<i4", nm), ("modality", "u1", N), ("saliency", "<f8", N), ("cluster", "<i8", N),
             ("embedding", "<f8", N * D), ("routes", "<i4", L * N * k), ("gates", "<f8", L * N * k)]
    total = 40 + sum(np.dtype(dt).itemsize * n for _, dt, n in sizes)
    import os

    if os.path.getsize(path) != total:
        raise ParseError(f"{path}: size {os.path.getsize(path)} != {total} implied by the header")
    arrs, off = {}, 40
    for name, dt, n in sizes:
        if mmap:
            arrs[name] = np.memmap(path, dtype=dt, mode="r", offset=off, shape=(n,))
        else:
            arrs[name] = np.fromfile(path, dtype=dt, count=n, offset=off)
        off += np.dtype(dt).itemsize * n
    if arrs["modality"].size and int(arrs["modality"].max()) > 1:
        raise ParseError(f"{path}: modality code out of range")
    tr = RoutingTrace(L, E, k, arrs["routes"].reshape(L, N, k), arrs["gates"].reshape(L, N, k), arrs["saliency"],
                      arrs["modality"], arrs["embedding"].reshape(N, D), arrs["cluster"],
                      [int(m) for m in arrs["marks"]], shared)
    bad = validate_trace(tr)
    if bad:
        raise ValidationError("; ".join(bad[:5]))
    return tr


__all__ = [
    "ExpertRef", "Modality", "RoutingTrace", "Token", "TraceGenConfig", "generate_trace",
    "validate_trace", "trace_digest", "MOD_VISUAL", "MOD_TEXT", "MOD_DECODE", "TRACE_VERSION",
    "save_trace_bin", "load_trace_bin",
]
