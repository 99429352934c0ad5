"""Expert-parallel layer stack: token rows move, weights stay.

In the sharded-cache mode (`moe.ShardedHome`) a miss pulls a 9.44 MB expert
slot from its home GPU over NVLink; at C3 that is ~1.06 GB of weights per
layer.  Expert parallelism inverts it: every expert of every cached layer
stays resident on its owner rank (expert e -> rank e % G, the same placement
as the sharded home copies) and each rank ships the ~40 MB of token rows its
requests route to the owners, which run the grouped tcgen05 FFN and ship the
outputs back:

    route -> stable sort of the picks by owner rank (vmm_permute_plan, key e % G)
          -> vmm_ep_dispatch: rows + {local expert, pick} tags written straight
             into the owners' receive buffers (P2P stores through IPC-mapped
             peer allocations; NVLink/NVSwitch on a multi-GPU box)
          -> [barrier] owner: permute by local expert, grouped SwiGLU (tcgen05)
          -> vmm_ep_return: outputs stored back into the sources' return buffers
          -> [barrier] source: the ordinary combine (+ next-layer RMSNorm)

There is no expert cache in this mode (no transfers, no hit/miss decisions):
it is the multi-GPU alternative to the offloaded cache, not a drop-in for the
reference's engine.  The pinned prefix and the per-request compression are the
shared `MoEStack` path.  The per-layer count exchange (G x G ints) and the
phase barriers use torch.distributed; the row traffic never does.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib, kernels
from ._lib import check, ptr, stream_ptr
from .errors import ContractError
from .moe import ExpertStore, MoEStack, ShardedHome, StackConfig


def ep_layout(counts: np.ndarray, rank: int) -> tuple[np.ndarray, np.ndarray, int]:
    """counts[s][e] = picks of expert e on source rank s ([G][E]).  Owner d =
    e % G holds its local experts j = e // G in ascending order, each block
    ordered by source rank.  Returns (base[e]: first row of MY block of expert
    e in its owner's buffer; off_local[j] (E/G + 1): my receive buffer's
    expert offsets; n_recv)."""
    counts = np.asarray(counts, dtype=np.int64)
    G, E = counts.shape
    total = counts.sum(axis=0)
    owner_off = np.zeros(E, dtype=np.int64)
    for d in range(G):
        run = 0
        for e in range(d, E, G):  # local experts of owner d in ascending order
            owner_off[e] = run
            run += total[e]
    base = owner_off + counts[:rank, :].sum(axis=0)
    mine = list(range(rank, E, G))
    per = -(-E // G)
    off_local = np.zeros(per + 1, dtype=np.int64)
    for j, e in enumerate(mine):
        off_local[j + 1] = off_local[j] + total[e]
    off_local[len(mine) + 1:] = off_local[len(mine)]
    return base.astype(np.int32), off_local.astype(np.int32), int(off_local[-1])


class EPBuffers:
    """This rank's receive / return buffers plus device tables of every rank's
    (IPC-mapped) buffers.  cap_recv rows may arrive per layer (fails loudly if
    the routing is more skewed than the capacity)."""

    def __init__(self, rank: int, world: int, cap_recv: int, cap_back: int, H: int, device, group=None):
        import torch.distributed as dist

        self.rank, self.world, self.cap_recv, self.cap_back = rank, world, cap_recv, cap_back
        self.rows = torch.empty(cap_recv, H, dtype=torch.bfloat16, device=device)
        self.meta = torch.empty(cap_recv, 2, dtype=torch.int32, device=device)
        self.back = torch.empty(cap_back, H, dtype=torch.bfloat16, device=device)
        L_ = _lib.lib()
        mine = [self.rows.data_ptr(), self.meta.data_ptr(), self.back.data_ptr()]
        tabs = [[0] * world for _ in range(3)]
        self._opened = []
        if world == 1:
            for j in range(3):
                tabs[j][0] = mine[j]
        else:
            blobs = [_lib.ipc_export(p) for p in mine]
            allh = [None] * world
            dist.all_gather_object(allh, blobs, group=group)
            for r in range(world):
                for j in range(3):
                    if r == rank:
                        tabs[j][r] = mine[j]
                        continue
                    base, q = _lib.ipc_import(allh[r][j])
                    self._opened.append(base)
                    tabs[j][r] = q
        self.rows_tab, self.meta_tab, self.back_tab = (
            torch.tensor(t, dtype=torch.int64, device=device) for t in tabs)

    def close(self):
        L_ = _lib.lib()
        for q in self._opened:
            L_.vmm_ipc_close(q)
        self._opened = []


class EPStack(MoEStack):
    """MoE stack whose cached layers run expert-parallel over `world` ranks."""

    def __init__(self, cfg: StackConfig, store: ExpertStore | None = None, seed: int = 0, rank: int = 0,
                 world: int = 1, max_rows: int = 0, cap_factor: float = 2.0, group=None, device_of_rank=None):
        """max_rows: largest retained-row count per forward on this rank (sizes
        the receive buffer: cap_factor x the balanced share of all ranks' picks)."""
        if cfg.routing != "live":
            raise ContractError("EP mode routes live")
        super().__init__(cfg, store=store, seed=seed)
        self.rank, self.world, self.group = rank, world, group
        self.home = None
        self.owner = ShardedHome(self.store, rank, world, device_of_rank)  # expert (l, e) resident on rank e % world
        k = cfg.k
        self.max_rows = int(max_rows)
        cap_recv = max(64, int(cap_factor * self.max_rows * k))  # ~ max_rows*k/world from each of world ranks
        self.buf = EPBuffers(rank, world, cap_recv, max(64, self.max_rows * k), cfg.hidden, self.device, group)
        E, L = cfg.experts, cfg.layers
        per = self.owner.per
        # local expert j of layer l lives in the owner arena at row l*per + j
        self.local_slots = torch.arange(L * per, dtype=torch.int32, device=self.device).reshape(L, per)
        self.local_E = per

    def _barrier(self):
        torch.cuda.current_stream().synchronize()
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier(group=self.group)

    def forward(self, x, saliency, modality, req_off=None, attn_qk=None):
        c = self.cfg
        L, E, k, lp, H, I = c.layers, c.experts, c.k, c.l_pinned, c.hidden, c.inter
        G, rank = self.world, self.rank
        dev = self.device
        if saliency is None:
            from .saliency import attention_saliency

            saliency = attention_saliency(*attn_qk)
        T = int(x.shape[0])
        bufs = self._buffers(max(T, -(-self.buf.cap_recv // k)))  # xp/h1/y also hold the received rows
        cur, _, prefix, _, ret, n_r, ret_off, xr = self._prefix_and_prune(x, saliency, modality, None, req_off, bufs)
        if n_r > self.max_rows:
            raise ContractError(f"{n_r} retained rows exceed the EP buffers ({self.max_rows})")
        Lb = _lib.lib()
        sp = stream_ptr()
        cur = xr
        M = n_r * k
        plan = (torch.empty(E + 1, dtype=torch.int32, device=dev), torch.empty(max(M, 1), dtype=torch.int32,
                device=dev), torch.empty(max(M, 1), dtype=torch.int32, device=dev))
        ident = torch.arange(max(M, 1), dtype=torch.int32, device=dev)  # combine reads the return buffer in pick order
        routes = []
        for l in range(lp, L):
            xn = kernels.rmsnorm(cur, out=bufs["xn"][:n_r])
            ids, gates, _ = kernels.route_topk(xn, self.store.router[l], k, ids=bufs["ids"][:n_r],
                                               gates=bufs["gates"][:n_r])
            routes.append(ids.clone())
            off_me, _, pos_me = kernels.permute_plan(ids, E, bufs=plan)  # my picks by expert (no row copy)
            # (source, expert) count exchange -> every pick's final row in its owner's FFN input
            my_counts = torch.diff(off_me[: E + 1]).to(torch.int64)
            if G > 1:
                import torch.distributed as dist

                mc = my_counts.cpu() if dist.get_backend(self.group) == "gloo" else my_counts
                allc = [torch.empty_like(mc) for _ in range(G)]
                dist.all_gather(allc, mc, group=self.group)
                counts = np.stack([t.cpu().numpy() for t in allc])
            else:
                counts = my_counts.cpu().numpy()[None, :]
            base, off_local, n_recv = ep_layout(counts, rank)
            if n_recv > self.buf.cap_recv:
                raise ContractError(f"EP receive buffer overflow ({n_recv} > {self.buf.cap_recv} rows)")
            base_d = torch.from_numpy(base).to(dev)
            off_local_d = torch.from_numpy(off_local).to(dev)
            kernels._n(1)
            check(Lb.vmm_ep_dispatch(ptr(xn), H, ptr(ids), k, ptr(pos_me), ptr(off_me), ptr(base_d),
                                     ptr(self.buf.rows_tab), ptr(self.buf.meta_tab), G, rank, M, sp))
            self._barrier()  # every source's rows have landed, already grouped by my experts
            y_loc = bufs["y"][:max(n_recv, 1)]
            if n_recv:
                _, y_loc = kernels.grouped_swiglu(self.buf.rows[:n_recv], off_local_d, self.owner.arena,
                                                  self.local_slots[l], I, h1=bufs["h1"][:n_recv],
                                                  y=bufs["y"][:n_recv])
                self.last_ffn = (self.buf.rows[:n_recv], off_local_d, l, n_recv)  # bench roofline replay
            kernels._n(1)
            check(Lb.vmm_ep_return(ptr(y_loc), H, ptr(self.buf.meta), ptr(self.buf.back_tab), n_recv, sp))
            self._barrier()  # every owner has returned my rows
            out = bufs["out"] if cur.data_ptr() != bufs["out"].data_ptr() else bufs["out2"]
            cur = kernels.combine(self.buf.back[:M], ident[:M].reshape(n_r, k), gates, cur, out=out[:n_r])
        return cur, ret.cpu().numpy(), routes

    def close(self):
        self.buf.close()
        self.owner.close()
