"""The live VL-MoE layer stack on one B200: router -> prune -> lookahead
predictor -> expert cache (+ real H2D prefetch) -> permute -> grouped SwiGLU
(tcgen05) -> combine, layer by layer.

This is the device realisation of the reference's per-layer engine
(`pkg/src/moesim/pipeline.py:695-760`).  Decisions are made by the native
logical-clock engine exactly as the reference makes them (so the cache
hit/miss/eviction/issue sequence of a run can be replayed bit-exactly by the
reference's `simulate` on the routes the run produced); execution follows the
decided schedule on real streams:

  compute stream : route / predictor / permute / FFN / combine kernels
  copy streams   : one cudaMemcpyAsync per decided expert transfer (pinned
                   host pool -> HBM slab), issued in decision order round-robin
                   over two copy streams, each followed by a ready-flag write;
                   per-slab write-after-read / write-after-write events
                   (vmm_xfer_*).

HBM layout (SURVEY §8(d), C3 numbers):
  arena   bf16 [l_pinned*E + num_slabs, 3*I*H]  -- slot = [W13 (2I x H,
          64-row gate/up interleave) | W2 (H x I)], 9.44 MB per slot; the
          first l_pinned*E slots hold the pinned prefix layers permanently,
          the rest are the cache slabs (826 x 9.44 MB = 7.8 GB at C3)
  router  bf16 [L, E, H]   (always resident, 0.5 MB per layer)
  tokens  bf16 [T, H] -> retained [N_r, H] after prune; permuted [N_r*k, H]
Host: pinned pool bf16 [host_layers*E, 3*I*H] (layer l is served from pool
layer l % host_layers so pinned RAM stays bounded; bytes moved are real).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace

import os

import numpy as np
import torch

from . import _lib, kernels
from ._lib import check
from .configs import Workload
from .errors import ContractError, ValidationError
from .pipeline import Engine, PredictorSpec, SimConfig, SimReport
from .predictor import decay_table, pow_table


@dataclass
class StackConfig:
    layers: int
    hidden: int
    experts: int
    k: int
    inter: int
    l_pinned: int
    num_slabs: int
    alpha: float = 0.1
    beta: float = 0.5
    lam: float = 2.0
    predictor: str = "history"  # history | gate | oracle | mlp | none
    budget: int = 20
    window: int = 5
    gamma: float = 0.8
    history_decay: float = 0.5
    speculative_grace: int = 1
    victim_policy: str = "priority"
    routing: str = "live"  # live | trace
    host_layers: int = 8
    transfer_ms: float = 0.17  # logical clock: 9.44 MB at ~55 GB/s (measured pinned H2D)
    gpu_ms: float = 0.002      # logical clock: per-expert FFN time
    compress_ms: float = 0.0
    bootstrap_ms: float = 0.0
    shared_experts: int = 0
    router_corr: float = 0.8   # synthetic router weights: correlation between consecutive layers' gates

    @classmethod
    def from_workload(cls, w: Workload, **kw) -> "StackConfig":
        base = dict(layers=w.layers, hidden=w.hidden, experts=w.experts, k=w.k, inter=w.inter,
                    l_pinned=w.l_pinned, num_slabs=w.num_slabs, alpha=w.alpha, beta=w.beta, lam=w.lam,
                    predictor=w.predictor, budget=w.budget, window=w.window, gamma=w.gamma,
                    history_decay=w.history_decay, speculative_grace=w.grace,
                    shared_experts=w.shared_experts)
        base.update(kw)
        return cls(**base)

    @property
    def slot_elems(self) -> int:
        return 3 * self.inter * self.hidden

    @property
    def slot_bytes(self) -> int:
        return 2 * self.slot_elems

    def sim_config(self) -> SimConfig:
        """The reference SimConfig whose simulate() replays this stack's decisions."""
        bw = 1.0
        return SimConfig(
            bandwidth_mb_per_ms=bw, expert_size_mb=self.transfer_ms * bw, gpu_ms_per_expert=self.gpu_ms,
            l_pinned=self.l_pinned, num_slabs=self.num_slabs,
            predictor=PredictorSpec(kind=self.predictor if self.predictor != "gate" else "oracle",
                                    budget=self.budget, window=self.window, gamma=self.gamma,
                                    history_decay=self.history_decay),
            speculative_grace=self.speculative_grace, victim_policy=self.victim_policy,
            compress_latency_ms=self.compress_ms, predictor_bootstrap_ms=self.bootstrap_ms,
            shared_experts=self.shared_experts,
        )


class ExpertStore:
    """Expert weights: pinned host pool + HBM slot arena + router weights.

    Under a multi-rank process group the host pool is ONE shared-memory
    segment per node, page-locked in every rank (dist.SharedHostPool,
    SURVEY 8(e) mode DP); alone, or when /dev/shm cannot hold it, each rank
    pins its own (`self.host_pool_kind` says which)."""

    def __init__(self, cfg: StackConfig, seed: int = 0, device=None, share_host_pool: bool = True):
        self.cfg = cfg
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        E, H, I, L = cfg.experts, cfg.hidden, cfg.inter, cfg.layers
        self.host_layers = max(1, min(cfg.host_layers, L))
        n_host = self.host_layers * E
        g = torch.Generator(device=dev).manual_seed(seed)
        self._shared = None
        if share_host_pool:
            from . import dist as vdist

            tag = f"{os.environ.get('MASTER_PORT', '0')}_{os.getppid()}_{seed}_{n_host}_{cfg.slot_bytes}"
            self._shared = vdist.SharedHostPool.create(n_host * cfg.slot_bytes, tag, dev)
        if self._shared is not None:
            self.pool = torch.frombuffer(self._shared.mm, dtype=torch.bfloat16).view(n_host, cfg.slot_elems)
            self.host_pool_kind = "shared (one page-locked shm pool per node)"
            fill = self._shared.filler
        else:
            self.pool = torch.empty((n_host, cfg.slot_elems), dtype=torch.bfloat16, pin_memory=True)
            self.host_pool_kind = "pinned per rank"
            fill = True
        chunk = max(1, (512 << 20) // (cfg.slot_bytes))
        for s0 in range(0, n_host, chunk):
            s1 = min(n_host, s0 + chunk)
            w = torch.randn((s1 - s0, cfg.slot_elems), generator=g, device=dev, dtype=torch.float32)
            w[:, : 2 * I * H] *= 1.0 / math.sqrt(H)
            w[:, 2 * I * H:] *= 1.0 / math.sqrt(I)
            if fill:
                self.pool[s0:s1].copy_(w.to(torch.bfloat16))
        if self._shared is not None:
            torch.cuda.synchronize(dev)
            self._shared.ready()  # the filler's weights are in the segment before any rank reads it
        self.n_pinned_slots = cfg.l_pinned * E
        S = cfg.shared_experts
        # arena: [pinned prefix experts | cache slabs | always-resident shared experts (L*S)]
        self.arena = torch.empty((self.n_pinned_slots + cfg.num_slabs + L * S, cfg.slot_elems),
                                 dtype=torch.bfloat16, device=dev)
        for l in range(cfg.l_pinned):
            h = l % self.host_layers
            self.arena[l * E:(l + 1) * E].copy_(self.pool[h * E:(h + 1) * E], non_blocking=True)
        base = self.n_pinned_slots + cfg.num_slabs
        for s0 in range(0, L * S, chunk):
            s1 = min(L * S, s0 + chunk)
            w = torch.randn((s1 - s0, cfg.slot_elems), generator=g, device=dev, dtype=torch.float32)
            w[:, : 2 * I * H] *= 1.0 / math.sqrt(H)
            w[:, 2 * I * H:] *= 1.0 / math.sqrt(I)
            self.arena[base + s0: base + s1].copy_(w.to(torch.bfloat16))
        self.shared_slot_of = (torch.arange(base, base + L * S, dtype=torch.int32, device=dev).reshape(L, S)
                               if S else None)
        # router: W[l] = rho W[l-1] + sqrt(1-rho^2) noise, so consecutive layers route
        # alike (the inter-layer affinity lookahead prediction relies on; rho=0 -> independent)
        rho = cfg.router_corr
        r = torch.randn((L, E, H), generator=g, device=dev)
        for l in range(1, L):
            r[l] = rho * r[l - 1] + math.sqrt(1.0 - rho * rho) * r[l]
        self.router = (r / math.sqrt(H)).to(torch.bfloat16)
        self.pinned_slot_of = (torch.arange(self.n_pinned_slots, dtype=torch.int32, device=dev).reshape(cfg.l_pinned, E)
                               if cfg.l_pinned else None)
        torch.cuda.synchronize(dev)

    def expert(self, layer: int, expert: int):
        """(w_gate [I,H], w_up [I,H], w_down [H,I]) of (layer, expert) from the host pool (for checks)."""
        c = self.cfg
        I, H = c.inter, c.hidden
        slot = self.pool[(layer % self.host_layers) * c.experts + expert]
        w13 = slot[: 2 * I * H].reshape(I // 64, 2, 64, H)
        return w13[:, 0].reshape(I, H), w13[:, 1].reshape(I, H), slot[2 * I * H:].reshape(H, I)


def route(x, w_gate, k: int, counts=None, stream=None):
    """Router entry point (no reference equivalent): (ids i32 [N,k], gates f32 [N,k])."""
    ids, gates, _ = kernels.route_topk(x, w_gate, k, counts=counts, stream=stream)
    return ids, gates


def moe_layer_forward(x, ids, gates, arena, slot_of, inter: int, experts: int, resid=True, stream=None,
                      bufs: dict | None = None, xn=None):
    """One MoE layer on resident experts: permute -> grouped SwiGLU -> combine (+ residual).

    x: residual rows; xn: the normalised rows the router/experts see (default x)."""
    N = int(x.shape[0])
    k = int(ids.shape[1])
    xn = x if xn is None else xn
    off, src, pos = kernels.permute_plan(ids, experts, stream=stream,
                                         bufs=None if bufs is None else (bufs["off"], bufs["src"], bufs["pos"]))
    xp = kernels.permute_rows(xn, src, N * k, stream=stream, out=None if bufs is None else bufs["xp"][: N * k])
    h1, y = kernels.grouped_swiglu(xp, off, arena, slot_of, inter, stream=stream,
                                   h1=None if bufs is None else bufs["h1"][: N * k],
                                   y=None if bufs is None else bufs["y"][: N * k])
    out = kernels.combine(y, pos, gates, x if resid else None, stream=stream,
                          out=None if bufs is None else bufs["out"][:N])
    return out


@dataclass
class StackResult:
    hidden: torch.Tensor            # [N_r, H] bf16 output of the last layer (retained tokens)
    retained: np.ndarray            # retained token ids (ascending)
    report: SimReport               # decisions / logical-clock report
    prefix_routes: torch.Tensor     # [l_pinned, T, k] routes of the pinned prefix
    routes: list                    # per post-prefix layer: ids [N_r, k] (device)
    scores: dict                    # context layer -> predictor y (np.float64[E])
    copies: int                     # expert transfers issued
    h2d_bytes: float
    retained_offsets: np.ndarray = None  # [R+1] rows of each request in `hidden`
    h2d_ms: float = 0.0                  # copy stream: first copy issued -> last copy landed (events)


@dataclass
class DecodeResult:
    hidden: torch.Tensor            # [1, H] output of the last layer
    copies: int                     # expert transfers issued during the step
    h2d_bytes: float
    routes: list                    # per layer ids [1, k] (device) when recorded
    scores: dict = None             # context layer -> predictor y of this step's emissions


class ShardedHome:
    """Home copies of every expert sharded over the ranks' HBM (SURVEY §8(e)
    mode "sharded cache"): expert (l, e) lives on rank e % world.  A cache miss
    on any rank is one copy-engine pull of the 9.44 MB slot from its home --
    local D2D, or a peer GPU's HBM over NVLink (IPC-mapped, peer access
    enabled) -- instead of a PCIe transfer from the pinned host pool.  No
    collective on the critical path; one handle exchange at setup."""

    def __init__(self, store: ExpertStore, rank: int = 0, world: int = 1, device_of_rank=None):
        """device_of_rank: CUDA device of each rank (default: rank r on device r,
        one process per GPU; several ranks may share one device in tests)."""
        import torch.distributed as dist

        c = store.cfg
        E, L = c.experts, c.layers
        self.rank, self.world = rank, world
        self.per = -(-E // world)
        dev = store.device
        self.arena = torch.empty((L * self.per, c.slot_elems), dtype=torch.bfloat16, device=dev)
        mine = [e for e in range(E) if e % world == rank]
        for l in range(L):
            h = l % store.host_layers
            rows = torch.tensor([h * E + e for e in mine], dtype=torch.long)
            self.arena[l * self.per: l * self.per + len(mine)].copy_(store.pool.index_select(0, rows).to(dev))
        torch.cuda.synchronize(dev)
        L_ = _lib.lib()
        bases = [self.arena.data_ptr()]
        self._opened = []
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, _lib.ipc_export(self.arena.data_ptr()))
            bases = []
            for r in range(world):
                if r == rank:
                    bases.append(self.arena.data_ptr())
                    continue
                check(L_.vmm_peer_enable(r if device_of_rank is None else int(device_of_rank[r])))
                base, p = _lib.ipc_import(handles[r])
                self._opened.append(base)
                bases.append(p)
        self.table = np.zeros(L * E, dtype=np.uint64)
        for l in range(L):
            for e in range(E):
                self.table[l * E + e] = bases[e % world] + (l * self.per + e // world) * c.slot_bytes

    def close(self):
        L_ = _lib.lib()
        for p in self._opened:
            L_.vmm_ipc_close(p)
        self._opened = []


class MoEStack:
    """One-request-at-a-time VL-MoE layer stack with the offloaded expert cache."""

    def __init__(self, cfg: StackConfig, store: ExpertStore | None = None, seed: int = 0,
                 home: ShardedHome | None = None, mlp_model=None):
        """home=None: misses are served from the pinned host pool over PCIe;
        home=ShardedHome(...): from the sharded HBM home copies (D2D / NVLink).
        mlp_model: the reference's MLPModel (or this package's; JSON-compatible)
        for predictor="mlp" (predictor.py:521-550): its features are the
        decayed routing histogram of the stack's OWN routes over the retained
        tokens, the mean of those tokens' embeddings plus the layer drift, and
        the kept-visual embedding mean (build_features, predictor.py:86-112);
        the token embeddings are a side input of forward()."""
        if cfg.predictor == "oracle" and cfg.routing != "trace":
            raise ValidationError("the oracle predictor needs trace routing (future routes)")
        if not 1 <= cfg.l_pinned <= cfg.layers:
            # the prune reads the pinned prefix's routes (prefix_layers non-empty, compress.py:41-42)
            raise ValidationError("the stack needs 1 <= l_pinned <= layers")
        if cfg.predictor not in ("history", "gate", "oracle", "mlp", "none"):
            raise ValidationError(f"unknown predictor kind '{cfg.predictor}'")
        if cfg.predictor == "mlp" and mlp_model is None:
            raise ValidationError("mlp predictor requires a trained model")  # pipeline.py:185-186
        self.cfg = cfg
        self.store = store or ExpertStore(cfg, seed)
        self.device = self.store.device
        self.home = home
        self._L = _lib.lib()
        h = C.c_void_p()
        check(self._L.vmm_xfer_create(cfg.num_slabs, cfg.slot_bytes, cfg.layers, C.byref(h)))
        self._x = h
        if home is not None:
            check(self._L.vmm_xfer_set_sources(h, home.table.ctypes.data, len(home.table)))
        E, L = cfg.experts, cfg.layers
        self.slot_host = torch.zeros((L, E), dtype=torch.int32, pin_memory=True)
        self.slot_dev = torch.zeros((L, E), dtype=torch.int32, device=self.device)
        # per-expert fill sequence numbers the fused FFN waits for (copy/compute overlap)
        self.need_host = torch.zeros((L, E), dtype=torch.int32, pin_memory=True)
        self.need_dev = torch.zeros((L, E), dtype=torch.int32, device=self.device)
        self.counts_host = torch.zeros((L, E), dtype=torch.int32, pin_memory=True)
        # per-layer expert walk / copy order of the CTA-pair FFN (largest experts first)
        self.order_host = torch.zeros((L, E), dtype=torch.int32, pin_memory=True)
        self.order_dev = torch.zeros((L, E), dtype=torch.int32, device=self.device)
        self.y_host = torch.zeros((L + 1, E), dtype=torch.float64, pin_memory=True)
        self.pow = torch.tensor(pow_table(cfg.history_decay, L), dtype=torch.float64, device=self.device)
        self.layer_ids = torch.arange(L, dtype=torch.int32, device=self.device)
        self.step_counts = torch.zeros((L, E), dtype=torch.int32, device=self.device)
        self._bufs = {}
        self._pbufs = {}  # chunked-prefix outputs (x_ready)
        self._mlp = None
        if mlp_model is not None:
            from .predictor import MLPModel, drift_table

            m = mlp_model if isinstance(mlp_model, MLPModel) else MLPModel.from_reference(mlp_model)
            d_in, d_h, d_b, n_out = m.dims
            D = (d_in - E) // 2
            if n_out != E or d_in != E + 2 * D:
                raise ValidationError(f"MLP dims {m.dims} do not fit {E} experts")
            self._mlp = dict(w=m.to_device(self.device), D=D, dh=d_h, db=d_b,
                             drift=torch.from_numpy(drift_table(L, D)).to(self.device),
                             hist=torch.empty(E, dtype=torch.float64, device=self.device),
                             hv=torch.zeros(D, dtype=torch.float64, device=self.device), emb=None, ids=None)
        self.profile = None  # list -> (start_ev, end_ev, bytes, flops, is_prefix) per FFN launch

    def __del__(self):
        h = getattr(self, "_x", None)
        if h:
            self._L.vmm_xfer_destroy(h)
            self._x = None

    @property
    def copy_stream_handle(self) -> int:
        return self._L.vmm_xfer_stream(self._x)

    def _buffers(self, n_tok: int):
        c = self.cfg
        if self._bufs.get("n", 0) < n_tok:
            dev = self.device
            M = n_tok * c.k
            self._bufs = dict(
                n=n_tok,
                off=torch.empty(c.experts + 1, dtype=torch.int32, device=dev),
                src=torch.empty(M, dtype=torch.int32, device=dev),
                pos=torch.empty(M, dtype=torch.int32, device=dev),
                xp=torch.empty(M, c.hidden, dtype=torch.bfloat16, device=dev),
                h1=torch.empty(M, c.inter, dtype=torch.bfloat16, device=dev),
                y=torch.empty(M, c.hidden, dtype=torch.bfloat16, device=dev),
                out=torch.empty(n_tok, c.hidden, dtype=torch.bfloat16, device=dev),
                out2=torch.empty(n_tok, c.hidden, dtype=torch.bfloat16, device=dev),
                xn=torch.empty(n_tok, c.hidden, dtype=torch.bfloat16, device=dev),
                ids=torch.empty(n_tok, c.k, dtype=torch.int32, device=dev),
                gates=torch.empty(n_tok, c.k, dtype=torch.float32, device=dev),
                y_dev=torch.empty(c.experts, dtype=torch.float64, device=dev),
                scratch=torch.empty(c.experts, dtype=torch.int32, device=dev),
                # shared experts (S per layer, every token)
                shared_src=torch.empty(max(n_tok * c.shared_experts, 1), dtype=torch.int32, device=dev),
                shared_off=torch.empty(c.shared_experts + 1, dtype=torch.int32, device=dev),
                xs=torch.empty(max(n_tok * c.shared_experts, 1), c.hidden, dtype=torch.bfloat16, device=dev),
                h1s=torch.empty(max(n_tok * c.shared_experts, 1), c.inter, dtype=torch.bfloat16, device=dev),
                ys=torch.empty(max(n_tok * c.shared_experts, 1), c.hidden, dtype=torch.bfloat16, device=dev),
                ffn_done=torch.empty(M // 128 + c.experts + 1, dtype=torch.int32, device=dev),
                iota=torch.arange(n_tok, dtype=torch.int32, device=dev),  # row ids (trace routing), made once
            )
        return self._bufs

    def forward(self, x, saliency, modality, trace=None, record: bool = False, req_off=None,
                keep_session: bool = False, attn_qk=None, x_ready=None, embeddings=None) -> StackResult:
        """Prefill a batch of requests through the whole stack.

        x bf16 [T, H] (device), saliency f64 [T], modality u8 [T] (0 visual,
        1 text; all prefill).  `req_off` (host ints, R+1) splits the rows into
        R requests (default: one request); each request is compressed on its
        own (one prune CTA per request) and the layers then run on the union of
        the retained rows, so expert transfers are shared by the batch.
        `trace` (device routes i32 [L,T,k], gates f32 [L,T,k]) is required for
        routing="trace".  saliency=None with attn_qk=(q [R,Hh,Q,D], k [R,Hh,T/R,D])
        derives the saliency on the device from the vision encoder's attention
        (head-averaged CLS/text->token attention, saliency.attention_saliency).
        x_ready: optional [(row_end, cuda.Event)] -- rows [prev_end, row_end) of x
        are valid once the event fires (a host->device copy in flight on another
        stream): the pinned prefix then runs chunk by chunk as the rows land
        (rows are independent in the prefix, so the result is identical).
        embeddings: f64 [>= T, D] token embeddings (device), required by the
        MLP predictor (rows beyond T may hold decode tokens, see decode_step)."""
        c = self.cfg
        L, E, k, lp = c.layers, c.experts, c.k, c.l_pinned
        dev = self.device
        T = int(x.shape[0])
        if saliency is None:
            if attn_qk is None:
                raise ContractError("forward needs saliency or attn_qk")
            from .saliency import attention_saliency

            saliency = attention_saliency(*attn_qk)
            if int(saliency.shape[0]) != T:
                raise ContractError("attn_qk keys must cover every token row (R requests x T/R tokens)")
        stream = torch.cuda.current_stream()
        sp = stream.cuda_stream
        bufs = self._buffers(T)
        if c.routing == "trace" and trace is None:
            raise ContractError("routing='trace' needs the trace's device routes")
        check(self._L.vmm_xfer_reset_stats(self._x))

        if c.predictor == "mlp" and (embeddings is None or int(embeddings.shape[0]) < T):
            raise ContractError("the MLP predictor needs the tokens' embeddings (f64 [T, D])")
        cur, x_ctx, prefix, counts_parts, ret, n_r, ret_off, xr = self._prefix_and_prune(
            x, saliency, modality, trace, req_off, bufs, x_ready=x_ready)
        if self._mlp is not None and c.predictor == "mlp":
            mp = self._mlp
            mp["emb"], mp["ids"] = embeddings.contiguous(), ret
            kernels.row_mean(mp["emb"], ret, modality, out=mp["hv"])  # visual_summary over the kept visual rows

        # --- per-layer demand counts over the retained tokens
        # (vmm_demand_counts overwrites its rows; the executor zeroes each later layer's row itself)
        counts_ret = torch.empty((L, E), dtype=torch.int32, device=dev)
        if lp:
            kernels.demand_counts(prefix[:lp], self.layer_ids[:lp], ret, E, out=counts_ret[:lp])
        oracle_table = None
        if c.predictor == "oracle":
            rl = trace["routes"]
            kernels.demand_counts(rl, self.layer_ids, ret, E, out=counts_ret)
            dec = torch.tensor(decay_table(c.gamma, c.window), dtype=torch.float64, device=dev)
            oracle_table = kernels.oracle_targets(counts_ret, self.layer_ids, c.window, dec)  # row = context layer

        cfg = c.sim_config()
        prefetching = c.predictor != "none" and c.budget > 0
        eng = Engine(L, E, cfg, c.num_slabs, lp, c.shared_experts, prefetching, False,
                     c.compress_ms + (c.bootstrap_ms if prefetching else 0.0))
        scores = {}

        def predict(ctx: int, x_in):
            """device y for context layer ctx (x_in: retained hidden states entering layer ctx)."""
            if c.predictor == "history":
                yt = kernels.history(counts_ret, torch.tensor([ctx], dtype=torch.int32, device=dev), self.pow)[0]
            elif c.predictor == "gate":
                yt = kernels.gate_lookahead(x_in, self.store.router[ctx + 1], k, scratch=bufs["scratch"],
                                            out=bufs["y_dev"])
            elif c.predictor == "mlp":
                mp = self._mlp
                cx = torch.tensor([ctx], dtype=torch.int32, device=dev)
                hist = kernels.history(counts_ret, cx, self.pow)
                yt = kernels.mlp_predict(hist, mp["emb"], mp["drift"], mp["ids"], mp["hv"], cx, mp["w"])[0][0]
            else:
                yt = oracle_table[ctx]
            self.y_host[ctx].copy_(yt, non_blocking=True)
            return self.y_host[ctx]

        # boot emission at context lp-1 over the retained tokens
        if prefetching and lp > 0:
            x_boot = kernels.gather_rows(x_ctx, ret) if c.predictor == "gate" else None
            yb = predict(lp - 1, x_boot)
            stream.synchronize()
            scores[lp - 1] = yb.numpy().copy()
            eng.begin(scores[lp - 1])
        else:
            eng.begin(None)
        n_copies = self._issue(eng)
        cp = None
        if lp:  # the pinned layers' demand over all prefill rows: per-chunk counts summed on the host
            cp = np.zeros((lp, E), dtype=np.int64)
            for l0_, t_ in counts_parts:
                cp[l0_:l0_ + int(t_.shape[0])] += t_.cpu().numpy()
        for l in range(lp):
            eng.layer(l, np.flatnonzero(cp[l]).astype(np.int32), 0, -1, None)

        # --- cached layers on the retained tokens: the native layer loop
        cur, n_cp, routes_t = self._native_layers(
            eng, xr, n_r, lp, L, 0, -1, rows=ret if c.routing == "trace" else None, counts=counts_ret,
            oracle_table=oracle_table, trace=trace, record=record)
        n_copies += n_cp
        for l in range(lp, L - 1):
            if eng.emits(l, 0):
                scores[l] = self.y_host[l].numpy().copy()
        routes = [routes_t[i] for i in range(L - lp)] if record else []
        check(self._L.vmm_xfer_join(self._x, sp))  # the step ends when its last transfer has landed
        report = eng.finish(with_events=False)
        b, ms, cnt = C.c_double(), C.c_double(), C.c_longlong()
        check(self._L.vmm_xfer_stats(self._x, C.byref(b), C.byref(ms), C.byref(cnt)))
        self._sess = dict(eng=eng, step=0, trace=trace) if keep_session else None
        return StackResult(hidden=cur, retained=ret.cpu().numpy(), report=report, prefix_routes=prefix[:lp],
                           routes=routes, scores=scores, copies=n_copies, h2d_bytes=b.value,
                           retained_offsets=ret_off, h2d_ms=ms.value)

    def _prefix_and_prune(self, x, saliency, modality, trace, req_off, bufs, x_ready=None):
        """Pinned prefix on all T rows (resident experts, engine-less executor,
        no host sync) then per-request compression on the prefix routes.
        Returns (rows after the prefix, xn of layer lp-1, prefix routes,
        prefix counts as [(first layer, device counts [n, E])] parts to sum,
        retained ids, N_r, per-request retained offsets, retained rows).
        Between the prefix and the first cached layer only our kernels and
        copy-engine copies run (no torch elementwise kernels)."""
        c = self.cfg
        L, E, k, lp = c.layers, c.experts, c.k, c.l_pinned
        dev = self.device
        T = int(x.shape[0])
        # The last prefix layer's FFN only matters for the tokens the prune keeps: route it on
        # every token (its routes feed the prune), run its experts on the retained rows only
        # (row-independent GEMMs: the retained rows come out bit-identical).  Live routing
        # without shared experts; VMM_PREFIX_FULL_LAST=1 runs it on every token.
        skip_last = lp >= 1 and c.routing == "live" and c.shared_experts == 0 and \
            not os.environ.get("VMM_PREFIX_FULL_LAST")
        lpe = lp - 1 if skip_last else lp  # prefix layers run in full on all tokens
        # --- pinned prefix: all prefill tokens, resident experts, no cache decisions:
        # the native executor in engine-less mode (no host sync inside the prefix)
        prefix = torch.empty((max(lp, 1), T, k), dtype=torch.int32, device=dev)
        # the executor zeroes (live) or overwrites (trace) each layer's counts row itself
        counts_pre = torch.empty((max(lp, 1), E), dtype=torch.int32, device=dev)
        counts_parts = []
        x_ctx = None
        cur = x
        offs_req = [0, T] if req_off is None else [int(v) for v in req_off]
        if lpe and not x_ready and len(offs_req) > 2 and T >= 16384 and not os.environ.get("VMM_PREFIX_ONE_STREAM"):
            # two request-aligned halves on two streams: one half's memory-bound kernels
            # (combine, permute, route) overlap the other half's tensor-core FFN
            mid = min(offs_req[1:-1], key=lambda v: abs(2 * v - T))
            x_ready = [(mid, None), (T, None)]
        if lpe and x_ready:
            # chunk by chunk (as the rows land, or the two halves), alternating over two streams
            if self._pbufs.get("n", 0) < T:
                self._pbufs = dict(n=T, cur=torch.empty_like(x), xn=torch.empty_like(x))
            cur_full, xn_full = self._pbufs["cur"][:T], self._pbufs["xn"][:T]
            main = torch.cuda.current_stream()
            if not hasattr(self, "_pstreams"):
                self._pstreams = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
            bounds, r0 = [], 0
            for r1, ev in x_ready:
                bounds.append((r0, int(r1), ev))
                r0 = int(r1)
            if r0 != T:
                raise ContractError("x_ready chunks must cover every row")
            caps = [max([b - a for i, (a, b, _) in enumerate(bounds) if i % 2 == j] or [0]) for j in range(2)]
            two = caps[0] + caps[1] <= int(bufs["n"])
            if not two:
                caps = [max(b - a for a, b, _ in bounds), 0]
            base = [0, caps[0]]
            for sp_ in self._pstreams:
                sp_.wait_stream(main)
            for i, (r0, r1, ev) in enumerate(bounds):
                n = r1 - r0
                if n <= 0:
                    continue
                lane = i % 2 if two else 0
                side = self._pstreams[lane]
                with torch.cuda.stream(side):
                    if ev is not None:
                        side.wait_event(ev)
                    routes_c = torch.empty((lpe, n, k), dtype=torch.int32, device=dev)
                    counts_c = torch.empty((lpe, E), dtype=torch.int32, device=dev)
                    rows_c = bufs["iota"][r0:r1] if c.routing == "trace" else None
                    out_c, _, _ = self._native_layers(None, x[r0:r1], n, 0, lpe, 0, -1, rows=rows_c, counts=counts_c,
                                                      trace=trace, record_into=routes_c,
                                                      region=(base[lane], caps[lane], lane), batch_rows=T)
                    cur_full[r0:r1].copy_(out_c)
                    if c.predictor == "gate" and not skip_last:  # boot emission context (layer lp-1 input)
                        xn_full[r0:r1].copy_(bufs["xn"][base[lane]:base[lane] + n])
                    # this chunk's rows of every prefix layer's routes into the [L][T][k] table
                    kernels.copy_rows_2d(prefix[:lpe, r0:r1].view(lpe, n * k), routes_c.view(lpe, n * k))
                    counts_parts.append((0, counts_c))
            for sp_ in self._pstreams:
                main.wait_stream(sp_)
            cur, x_ctx = cur_full, xn_full
        elif lpe:
            rows_all = bufs["iota"][:T] if c.routing == "trace" else None
            cur, _, _ = self._native_layers(None, x, T, 0, lpe, 0, -1, rows=rows_all, counts=counts_pre, trace=trace,
                                            record_into=prefix[:lpe])
            counts_parts.append((0, counts_pre[:lpe]))
            x_ctx = bufs["xn"][:T]  # normalised input of layer lp-1: context of the boot emission (gate predictor)
        if x_ready and not lpe:  # no full prefix layer ran: the rows must have landed before layer lp-1
            main = torch.cuda.current_stream()
            for _, ev in x_ready:
                if ev is not None:
                    main.wait_event(ev)
        last = None
        if skip_last:  # layer lp-1: RMSNorm + router on every token (the prune needs its routes)
            l = lp - 1
            xn_l = kernels.rmsnorm(cur, out=bufs["xn"][:T])
            kernels.memset_(counts_pre[l])  # the router accumulates its pick counts
            ids_l, gates_l, _ = kernels.route_topk(xn_l, self.store.router[l], k, counts=counts_pre[l],
                                                   ids=prefix[l], gates=bufs["gates"][:T])
            counts_parts.append((l, counts_pre[l:l + 1]))
            x_ctx = xn_l  # normalised input of layer lp-1: context of the boot emission (gate predictor)
            last = (cur, xn_l, ids_l, gates_l)


        # --- prune (token compression) on the prefix routes, one CTA per request; budgets
        # floor(alpha n_vis) / floor(beta n_vis) on the device, then the per-request lists are
        # packed into one ascending list of global rows.  One small D2H (retained counts +
        # status) is the only host sync: the row count sizes every later launch.
        offs = [0, T] if req_off is None else [int(v) for v in req_off]
        R = len(offs) - 1
        offs_d = torch.tensor(offs, dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
        pr = kernels.prune(saliency, modality, prefix[:max(lp, 1)], offs_d, None, None, E, c.lam,
                           alpha=c.alpha, beta=c.beta)
        ret_all, ret_off_d = kernels.retained_pack(offs_d, pr["retained"], pr["n_retained"])
        ns = self._ns_host[:, :R] if getattr(self, "_ns_host", None) is not None and \
            self._ns_host.shape[1] >= R else None
        if ns is None:
            self._ns_host = torch.empty((2, max(R, 1)), dtype=torch.int32, pin_memory=True)
            ns = self._ns_host[:, :R]
        ns.copy_(pr["ns"], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        n_ret = ns[0].numpy().astype(np.int64)
        st = ns[1].numpy()
        if (st != 0).any():
            from .compress import raise_prune_status

            raise_prune_status(int(st[st != 0][0]))
        ret_off = np.concatenate([[0], np.cumsum(n_ret)]).astype(np.int64)
        n_r = int(ret_off[-1])
        ret = ret_all[:n_r]
        if last is None:
            xr = kernels.gather_rows(cur, ret, out=bufs["xp"][:n_r])  # scratch until permute of layer lp
            xr = xr.clone()
        else:  # layer lp-1's experts on the retained rows only
            cur_l, xn_l, ids_l, gates_l = last
            x_ret = kernels.gather_rows(cur_l, ret)
            xn_ret = kernels.gather_rows(xn_l, ret)
            ids_ret, gates_ret = kernels.gather_cols(ids_l, ret), kernels.gather_cols(gates_l, ret)
            M = n_r * k
            off, src, pos, xp = kernels.permute(ids_ret, xn_ret, E, bufs=(bufs["off"], bufs["src"][:M], bufs["pos"][:M]),
                                                out=bufs["xp"][:M])
            _, y = kernels.grouped_swiglu(xp, off, self.store.arena, self.store.pinned_slot_of[lp - 1], c.inter,
                                          h1=bufs["h1"][:M], y=bufs["y"][:M])
            xr = kernels.combine(y, pos.view(n_r, k), gates_ret, x_ret)
            cur = xr
        return cur, x_ctx, prefix, counts_parts, ret, n_r, ret_off, xr


    def _native_layers(self, eng, x, n_rows, l0, l1, phase, step, rows=None, counts=None, oracle_table=None,
                       trace=None, record=False, record_into=None, region=None, mlp_ids=None, batch_rows=0):
        """Run layers [l0, l1) through the native executor (csrc/stack.cpp).
        eng=None: pinned-prefix mode (no decisions / copies / host syncs).
        region=(row_base, cap, lane): run in rows [row_base, row_base+cap) of the
        scratch buffers with lane's own small buffers (two pinned-prefix chunks
        on two streams at once; enqueued on the current stream).
        batch_rows: the rows are a chunk of a batch of that many rows (the router's
        numerics follow the batch: chunked prefixes route like one launch)."""
        c = self.cfg
        L, E, k = c.layers, c.experts, c.k
        bufs = self._buffers(n_rows)
        st = self.store
        pred = {"none": 0, "history": 1, "gate": 2, "oracle": 3, "mlp": 4}[c.predictor]
        rb, cap, lane = (0, int(bufs["n"]), 0) if region is None else region
        if region is not None:
            if eng is not None or rb + cap > int(bufs["n"]) or n_rows > cap:
                raise ContractError("scratch region outside the buffers (pinned prefix only)")
            if lane and "off_b" not in bufs:
                bufs["off_b"] = torch.empty_like(bufs["off"])
                bufs["ffn_done_b"] = torch.empty_like(bufs["ffn_done"])
                bufs["shared_off_b"] = torch.empty_like(bufs["shared_off"])
        H, I, S = c.hidden, c.inter, c.shared_experts

        def at(name, row_bytes):  # pointer of row rb of a [rows, ...] scratch buffer
            return bufs[name].data_ptr() + rb * row_bytes
        b_off, b_done, b_soff = (("off_b", "ffn_done_b", "shared_off_b") if lane else ("off", "ffn_done", "shared_off"))
        d = _lib.StackDesc(
            layers=L, experts=E, k=k, hidden=c.hidden, inter=c.inter, l_pinned=c.l_pinned,
            n_pinned_slots=st.n_pinned_slots, n_slots=int(st.arena.shape[0]), slot_bytes=c.slot_bytes,
            host_layers=st.host_layers, cap_rows=cap, routing=int(c.routing == "trace"), predictor=pred,
            counts_preset=int(oracle_table is not None and c.routing == "trace"),
            arena=st.arena.data_ptr(), pool=st.pool.data_ptr() if self.home is None else None,
            router=st.router.data_ptr(),
            pinned_slot_of=st.pinned_slot_of.data_ptr() if st.pinned_slot_of is not None else None,
            layer_ids=self.layer_ids.data_ptr(), pow_table=self.pow.data_ptr(),
            oracle_table=oracle_table.data_ptr() if oracle_table is not None else None,
            trace_routes=trace["routes"].data_ptr() if trace is not None else None,
            trace_gates=trace["gates"].data_ptr() if trace is not None else None,
            trace_tokens=int(trace["routes"].shape[1]) if trace is not None else 0,
            xn=at("xn", H * 2), xp=at("xp", k * H * 2), h1=at("h1", k * I * 2), y=at("y", k * H * 2),
            out0=at("out", H * 2), out1=at("out2", H * 2), ids=at("ids", k * 4),
            gates=at("gates", k * 4), off=bufs[b_off].data_ptr(), src=at("src", k * 4),
            pos=at("pos", k * 4), counts=counts.data_ptr(), la_counts=bufs["scratch"].data_ptr(),
            y_dev=bufs["y_dev"].data_ptr(), slot_dev=self.slot_dev.data_ptr(),
            counts_host=self.counts_host.data_ptr(), y_host=self.y_host.data_ptr(),
            slot_host=self.slot_host.data_ptr(), shared=c.shared_experts,
            shared_slot_of=st.shared_slot_of.data_ptr() if st.shared_slot_of is not None else None,
            shared_src=at("shared_src", max(S, 1) * 4), shared_off=bufs[b_soff].data_ptr(),
            xs=at("xs", max(S, 1) * H * 2), h1s=at("h1s", max(S, 1) * I * 2), ys=at("ys", max(S, 1) * H * 2),
            need_host=self.need_host.data_ptr(), need_dev=self.need_dev.data_ptr(),
            ffn_done=bufs[b_done].data_ptr(), route_batch_rows=int(batch_rows),
            order_host=self.order_host.data_ptr(), order_dev=self.order_dev.data_ptr())
        mp = self._mlp
        if pred == 4 and eng is not None:
            ids_t = mp["ids"] if mlp_ids is None else mlp_ids
            d.mlp_emb, d.mlp_drift, d.mlp_hv = mp["emb"].data_ptr(), mp["drift"].data_ptr(), mp["hv"].data_ptr()
            d.mlp_ids, d.mlp_n_ids = ids_t.data_ptr(), int(ids_t.shape[0])
            d.mlp_dim, d.mlp_hidden, d.mlp_bottleneck = mp["D"], mp["dh"], mp["db"]
            w = mp["w"]
            d.mlp_w1, d.mlp_b1, d.mlp_w2 = w["w1"].data_ptr(), w["b1"].data_ptr(), w["w2"].data_ptr()
            d.mlp_b2, d.mlp_wo, d.mlp_bo = w["b2"].data_ptr(), w["wo"].data_ptr(), w["bo"].data_ptr()
            d.mlp_hist = mp["hist"].data_ptr()
        h = C.c_void_p()
        check(self._L.vmm_stack_create(C.byref(d), C.byref(h)))
        nl = l1 - l0
        out = _lib.StackOut()
        if record_into is not None:
            routes_t, record = record_into, True
        else:
            routes_t = torch.empty((nl, n_rows, k), dtype=torch.int32, device=self.device) if record else None
        out.routes = routes_t.data_ptr() if record else None
        evs = None
        n_dem = np.zeros(nl, dtype=np.int32)
        out.n_demand = n_dem.ctypes.data
        cmarks = None
        if self.profile is not None:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nl)]
            for e in evs:
                e.record()  # materialise the CUDA events
            arr = (C.c_void_p * (2 * nl))(*[e.cuda_event for e in evs])
            out.ffn_start = C.cast(arr, C.c_void_p)
            out.ffn_end = C.cast(C.byref(arr, nl * C.sizeof(C.c_void_p)), C.c_void_p)
            if eng is not None:
                cmarks = [torch.cuda.Event(enable_timing=True) for _ in range(3 * nl)]
                for e in cmarks:
                    e.record()
                carr = (C.c_void_p * (3 * nl))(*[e.cuda_event for e in cmarks])
                out.copy_marks = C.cast(carr, C.c_void_p)
        try:
            check(self._L.vmm_stack_layers(h, None if eng is None else eng._h, self._x, x.data_ptr(), n_rows, l0, l1,
                                           phase, step,
                                           rows.data_ptr() if rows is not None else None,
                                           torch.cuda.current_stream().cuda_stream, C.byref(out)))
        finally:
            self._L.vmm_stack_destroy(h)
        if self.profile is not None:
            M = n_rows * k
            for i in range(nl):
                ne = c.experts if eng is None else int(n_dem[i])  # pinned prefix: every expert resident
                nbytes = ne * c.slot_bytes + M * c.hidden * 2 * 2  # weights + Xp read + Y write (H1 on chip)
                self.profile.append((evs[i], evs[nl + i], nbytes, 6.0 * M * c.hidden * c.inter, eng is None))
        res = bufs["out"] if out.x_out == at("out", H * 2) else bufs["out2"]
        self.last_host_us = list(out.host_us)
        self.last_copy_marks = cmarks
        return res[rb:rb + n_rows], out.copies, routes_t

    # ------------------------------------------------------------------
    # decode phase (pipeline.py:723-740): one token per step, the prefill's
    # cache persists, emissions after the last pinned layer and every cached
    # layer < L-1 over the single token
    # ------------------------------------------------------------------
    def decode_step(self, x_tok, tok: int | None = None, record: bool = False) -> "DecodeResult":
        """x_tok bf16 [1, H]: the decode token's hidden state entering layer 0.
        With routing="trace", `tok` is the token's row in the session trace; with
        predictor="mlp", its row in forward()'s embeddings."""
        sess = getattr(self, "_sess", None)
        if sess is None:
            raise ContractError("decode_step needs forward(..., keep_session=True) first")
        c = self.cfg
        L, E = c.layers, c.experts
        dev = self.device
        eng, s = sess["eng"], sess["step"]
        trace = sess["trace"]
        if c.routing == "trace" and tok is None:
            raise ContractError("routing='trace' decode needs the token's trace row")
        mlp_ids = None
        if c.predictor == "mlp":  # decode emissions pool the decode token alone (pipeline.py:723-740)
            if tok is None or self._mlp["emb"] is None or tok >= int(self._mlp["emb"].shape[0]):
                raise ContractError("mlp decode needs the token's row in forward()'s embeddings")
            mlp_ids = torch.tensor([tok], dtype=torch.int32, device=dev)
        check(self._L.vmm_xfer_reset_stats(self._x))
        counts = self.step_counts
        rows, otab = None, None
        if c.routing == "trace":
            rows = torch.tensor([tok], dtype=torch.int32, device=dev)
            if c.predictor == "oracle":
                kernels.demand_counts(trace["routes"], self.layer_ids, rows, E, out=counts)
                dec = torch.tensor(decay_table(c.gamma, c.window), dtype=torch.float64, device=dev)
                otab = kernels.oracle_targets(counts, self.layer_ids, c.window, dec)
        cur, n_cp, routes_t = self._native_layers(eng, x_tok, 1, 0, L, 1, s, rows=rows, counts=counts,
                                                  oracle_table=otab, trace=trace, record=record, mlp_ids=mlp_ids)
        scores = {l: self.y_host[l].numpy().copy() for l in range(L) if eng.emits(l, 1)}
        eng.end_step()
        sess["step"] = s + 1
        sp = torch.cuda.current_stream().cuda_stream
        check(self._L.vmm_xfer_join(self._x, sp))
        b, ms, cnt = C.c_double(), C.c_double(), C.c_longlong()
        check(self._L.vmm_xfer_stats(self._x, C.byref(b), C.byref(ms), C.byref(cnt)))
        routes = [routes_t[i] for i in range(L)] if record else []
        return DecodeResult(hidden=cur.clone(), copies=n_cp, h2d_bytes=b.value, routes=routes, scores=scores)

    def end_session(self) -> SimReport:
        sess = getattr(self, "_sess", None)
        if sess is None:
            raise ContractError("no open session")
        self._sess = None
        return sess["eng"].finish(with_events=False)

    def _issue(self, eng: Engine) -> int:
        n = C.c_int()
        pool = self.store.pool.data_ptr() if self.home is None else None
        check(self._L.vmm_xfer_issue_engine(self._x, eng._h, pool, self.store.host_layers,
                                            self.cfg.experts, self.store.arena.data_ptr(),
                                            self.store.n_pinned_slots, self.cfg.slot_bytes, C.byref(n)))
        return n.value

    def sync(self):
        check(self._L.vmm_xfer_sync(self._x))
        torch.cuda.synchronize()
