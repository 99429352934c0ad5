"""Torch-facing wrappers of the device entry points of libvismmoe.

Each function takes device tensors, launches on the current (or given) CUDA
stream and returns device tensors; nothing here copies to the host unless the
name says so.  Every call goes through the C-ABI (`_lib`), which refuses to
run without an sm_100 device.
"""
from __future__ import annotations

import math

import torch

from . import _lib
from ._lib import check, ptr, stream_ptr

_i32 = torch.int32

# number of libvismmoe kernels launched through these wrappers (bench evidence)
LAUNCHES = [0]


def _n(k: int) -> None:
    LAUNCHES[0] += k


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def memset_(t, byte_value: int = 0, stream=None):
    """Fill a contiguous device tensor's bytes with a stream-ordered memset (no kernel)."""
    if not t.is_contiguous():
        raise ValueError("memset_ needs a contiguous tensor")
    check(_lib.lib().vmm_memset_async(ptr(t), int(byte_value), t.numel() * t.element_size(), stream_ptr(stream)))
    return t


def copy_rows_2d(dst, src, stream=None):
    """dst[i, :n] = src[i, :n] for 2-D views whose rows are contiguous (any row pitch): one
    strided copy-engine copy (cudaMemcpy2DAsync), no kernel."""
    h, w = (int(v) for v in src.shape[:2])
    if tuple(dst.shape[:2]) != (h, w) or dst.dtype != src.dtype or dst.stride(1) != 1 or src.stride(1) != 1:
        raise ValueError("copy_rows_2d needs equal shapes and contiguous rows")
    es = src.element_size()
    check(_lib.lib().vmm_copy2d_async(ptr(dst), dst.stride(0) * es, ptr(src), src.stride(0) * es, w * es, h,
                                      stream_ptr(stream)))
    return dst


# ---------------------------------------------------------------------------
# prune
# ---------------------------------------------------------------------------
def prune(saliency, modality, prefix_routes, req_off, k_core, k_keep, experts: int, lam: float, stream=None,
          alpha: float = 0.0, beta: float = 0.0):
    """Batched compression.  Shapes: saliency f64 [T], modality u8 [T],
    prefix_routes i32 [P, T, k], req_off i32 [R+1], k_core/k_keep i32 [R]
    (or both None: budgets floor(alpha*n_visual), floor(beta*n_visual) per
    request on the device).  Returns dict of device tensors (include/vismmoe.h
    vmm_prune)."""
    L = _lib.lib()
    T = int(saliency.shape[0])
    P, _, k = (int(x) for x in prefix_routes.shape)
    R = int(req_off.shape[0]) - 1
    dev = saliency.device
    out = dict(
        s_norm=torch.empty(T, dtype=torch.float64, device=dev),
        delta=torch.empty(T, dtype=torch.float64, device=dev),
        score=torch.empty(T, dtype=torch.float64, device=dev),
        flags=torch.empty(T, dtype=torch.uint8, device=dev),
        retained=torch.empty(max(T, 1), dtype=_i32, device=dev),
        # n_retained and status side by side: one D2H reads both
        ns=memset_(torch.empty((2, R), dtype=_i32, device=dev), 0xFF, stream),  # -1
        target=memset_(torch.empty(R, 4, dtype=torch.int64, device=dev), 0, stream),
    )
    out["n_retained"], out["status"] = out["ns"][0], out["ns"][1]
    _n(1)
    check(L.vmm_prune(ptr(saliency), ptr(modality), ptr(prefix_routes), ptr(req_off),
                      None if k_core is None else ptr(k_core), None if k_keep is None else ptr(k_keep),
                      float(alpha), float(beta), R, T, P, k, experts, float(lam), ptr(out["s_norm"]),
                      ptr(out["delta"]), ptr(out["score"]), ptr(out["flags"]), ptr(out["retained"]),
                      ptr(out["n_retained"]), ptr(out["target"]), ptr(out["status"]), stream_ptr(stream)))
    return out


def retained_pack(req_off, retained, n_retained, stream=None, out=None, out_off=None):
    """Per-request retained lists -> (global ascending row ids [T cap], offsets [R+1])."""
    R = int(req_off.shape[0]) - 1
    dev = retained.device
    out = torch.empty(int(retained.shape[0]), dtype=_i32, device=dev) if out is None else out
    out_off = torch.empty(R + 1, dtype=_i32, device=dev) if out_off is None else out_off
    _n(1)
    check(_lib.lib().vmm_retained_pack(ptr(req_off), ptr(retained), ptr(n_retained), R, ptr(out), ptr(out_off),
                                       stream_ptr(stream)))
    return out, out_off


def gather_rows(src, idx, stream=None, out=None):
    n = int(idx.shape[0])
    H = int(src.shape[1])
    out = torch.empty(n, H, dtype=src.dtype, device=src.device) if out is None else out
    _n(1)
    check(_lib.lib().vmm_gather_rows(ptr(src), ptr(idx), n, H, ptr(out), stream_ptr(stream)))
    return out


def row_mean(emb, ids, modality=None, stream=None, out=None):
    """Column means of emb[ids] (numpy axis-0 order), skipping rows whose modality != 0."""
    D = int(emb.shape[1])
    out = torch.empty(D, dtype=torch.float64, device=emb.device) if out is None else out
    _n(1)
    check(_lib.lib().vmm_row_mean(ptr(emb), D, ptr(ids), int(ids.shape[0]),
                                  None if modality is None else ptr(modality), ptr(out), stream_ptr(stream)))
    return out


def gather_cols(src, idx, stream=None, out=None):
    """Rows of an i32 or f32 [N, width] table by index (vmm_gather_i32/f32)."""
    n, width = int(idx.shape[0]), int(src.shape[1])
    out = torch.empty(n, width, dtype=src.dtype, device=src.device) if out is None else out
    fn = {torch.int32: _lib.lib().vmm_gather_i32, torch.float32: _lib.lib().vmm_gather_f32}[src.dtype]
    _n(1)
    check(fn(ptr(src), ptr(idx), n, width, ptr(out), stream_ptr(stream)))
    return out


# ---------------------------------------------------------------------------
# router / predictors
# ---------------------------------------------------------------------------
def route_topk(x, w_gate, k: int, counts=None, want_logits=False, stream=None, ids=None, gates=None,
               batch_rows=None):
    """x bf16 [N, H], w_gate bf16 [E, H] -> (ids i32 [N,k], gates f32 [N,k], logits|None).
    batch_rows: the rows are a chunk of a batch of that many rows -- the result is
    bit-identical to routing the whole batch in one call (vmm_route_topk_ex)."""
    N, H = (int(s) for s in x.shape)
    E = int(w_gate.shape[0])
    ids = torch.empty(N, k, dtype=_i32, device=x.device) if ids is None else ids
    gates = torch.empty(N, k, dtype=torch.float32, device=x.device) if gates is None else gates
    logits = torch.empty(N, E, dtype=torch.float32, device=x.device) if want_logits else None
    _n(1)
    check(_lib.lib().vmm_route_topk_ex(ptr(x), ptr(w_gate), N, H, E, k, ptr(ids), ptr(gates), ptr(logits),
                                       ptr(counts), max(N, batch_rows or 0), stream_ptr(stream)))
    return ids, gates, logits


def route_lookahead(x, router, layer: int, k: int, counts, la_counts, stream=None, ids=None, gates=None,
                    batch_rows=None):
    """Fused router (layer) + gate lookahead (layer+1) on the same rows; router bf16 [L, E, H].
    batch_rows: as for route_topk."""
    N, H = (int(s) for s in x.shape)
    L_, E = int(router.shape[0]), int(router.shape[1])
    ids = torch.empty(N, k, dtype=_i32, device=x.device) if ids is None else ids
    gates = torch.empty(N, k, dtype=torch.float32, device=x.device) if gates is None else gates
    _n(1)
    check(_lib.lib().vmm_route_lookahead_ex(ptr(x), ptr(router), layer, L_, N, H, E, k, ptr(ids), ptr(gates),
                                            ptr(counts), ptr(la_counts), max(N, batch_rows or 0),
                                            stream_ptr(stream)))
    return ids, gates


def normalize_counts(counts, denom: float, stream=None, out=None):
    E = int(counts.shape[0])
    out = torch.empty(E, dtype=torch.float64, device=counts.device) if out is None else out
    _n(1)
    check(_lib.lib().vmm_normalize_counts(ptr(counts), E, float(denom), ptr(out), stream_ptr(stream)))
    return out


def demand_counts(routes, layers, ids, experts: int, stream=None, out=None):
    """routes i32 [L, T, k]; layers i32 [n]; ids i32 [m] -> u32-as-i32 counts [n, E]."""
    L_, T, k = (int(s) for s in routes.shape)
    n = int(layers.shape[0])
    out = torch.empty(n, experts, dtype=_i32, device=routes.device) if out is None else out
    _n(1)
    check(_lib.lib().vmm_demand_counts(ptr(routes), L_, T, k, experts, ptr(layers), n, ptr(ids), int(ids.shape[0]),
                                       ptr(out), stream_ptr(stream)))
    return out


def oracle_targets(counts_all, ctx, window: int, decay, stream=None):
    L_, E = (int(s) for s in counts_all.shape)
    y = torch.empty(int(ctx.shape[0]), E, dtype=torch.float64, device=counts_all.device)
    _n(1)
    check(_lib.lib().vmm_oracle_targets(ptr(counts_all), L_, E, ptr(ctx), int(ctx.shape[0]), window, ptr(decay),
                                        ptr(y), stream_ptr(stream)))
    return y


def history(counts_all, ctx, pow_table, stream=None):
    L_, E = (int(s) for s in counts_all.shape)
    y = torch.empty(int(ctx.shape[0]), E, dtype=torch.float64, device=counts_all.device)
    _n(1)
    check(_lib.lib().vmm_history(ptr(counts_all), L_, E, ptr(ctx), int(ctx.shape[0]), ptr(pow_table), ptr(y),
                                 stream_ptr(stream)))
    return y


def mlp_predict(hist, emb, drift, ids, h_v, ctx, model: dict, want_features=False, stream=None):
    n_ctx, E = (int(s) for s in hist.shape)
    D = int(emb.shape[1])
    dh = int(model["w1"].shape[0])
    db = int(model["w2"].shape[0])
    y = torch.empty(n_ctx, E, dtype=torch.float64, device=hist.device)
    feat = torch.empty(n_ctx, E + 2 * D, dtype=torch.float64, device=hist.device) if want_features else None
    _n(1)
    check(_lib.lib().vmm_mlp_predict(ptr(hist), ptr(emb), D, ptr(drift), ptr(ids), int(ids.shape[0]), ptr(h_v),
                                     ptr(ctx), n_ctx, E, ptr(model["w1"]), ptr(model["b1"]), dh, ptr(model["w2"]),
                                     ptr(model["b2"]), db, ptr(model["wo"]), ptr(model["bo"]), ptr(feat), ptr(y),
                                     stream_ptr(stream)))
    return y, feat


def gate_lookahead(x, w_next, k: int, stream=None, scratch=None, out=None):
    N, H = (int(s) for s in x.shape)
    E = int(w_next.shape[0])
    scratch = torch.empty(E, dtype=_i32, device=x.device) if scratch is None else scratch
    out = torch.empty(E, dtype=torch.float64, device=x.device) if out is None else out
    _n(2)
    check(_lib.lib().vmm_gate_lookahead(ptr(x), ptr(w_next), N, H, E, k, ptr(scratch), ptr(out),
                                        stream_ptr(stream)))
    return out


# ---------------------------------------------------------------------------
# permutation / expert FFN / combine
# ---------------------------------------------------------------------------
def permute_plan(ids, experts: int, stream=None, bufs=None):
    N, k = (int(s) for s in ids.shape)
    if bufs is None:
        bufs = (torch.empty(experts + 1, dtype=_i32, device=ids.device),
                torch.empty(max(N * k, 1), dtype=_i32, device=ids.device),
                torch.empty(max(N * k, 1), dtype=_i32, device=ids.device))
    offsets, src_row, pos = bufs
    _n(1)
    check(_lib.lib().vmm_permute_plan(ptr(ids), N, k, experts, ptr(offsets), ptr(src_row), ptr(pos),
                                      stream_ptr(stream)))
    return offsets, src_row, pos


def permute(ids, x, experts: int, stream=None, bufs=None, out=None):
    """Fused plan + row copy: (offsets, src_row, pos, xp) with xp[p] = x[src_row[p]]."""
    N, k = (int(s) for s in ids.shape)
    H = int(x.shape[1])
    if bufs is None:
        bufs = (torch.empty(experts + 1, dtype=_i32, device=ids.device),
                torch.empty(max(N * k, 1), dtype=_i32, device=ids.device),
                torch.empty(max(N * k, 1), dtype=_i32, device=ids.device))
    offsets, src_row, pos = bufs
    out = torch.empty(N * k, H, dtype=x.dtype, device=x.device) if out is None else out
    _n(3)
    check(_lib.lib().vmm_permute(ptr(ids), N, k, experts, ptr(x), H, ptr(offsets), ptr(src_row), ptr(pos),
                                 ptr(out), stream_ptr(stream)))
    return offsets, src_row, pos, out


def permute_rows(x, src_row, n_rows: int, stream=None, out=None):
    H = int(x.shape[1])
    out = torch.empty(n_rows, H, dtype=x.dtype, device=x.device) if out is None else out
    _n(1)
    check(_lib.lib().vmm_permute_rows(ptr(x), ptr(src_row), n_rows, H, ptr(out), stream_ptr(stream)))
    return out


class keep_h1:
    """Context: the fused FFN keeps its H1 scratch (by default the CTA-pair path
    drops consumed H1 rows from L2 without a write-back, so H1 is undefined
    after the call -- vmm_ffn_keep_h1)."""

    def __enter__(self):
        check(_lib.lib().vmm_ffn_keep_h1(1))
        return self

    def __exit__(self, *exc):
        check(_lib.lib().vmm_ffn_keep_h1(0))


def grouped_swiglu(xp, offsets, arena, slot_of, inter: int, stream=None, h1=None, y=None, simt: bool = False,
                   fused: bool = True, need=None, ready=None, ready_base: int = 0, x_rows=None, src_row=None,
                   order=None):
    """Grouped SwiGLU over expert-contiguous rows of xp.

    Default: the fused persistent tcgen05 kernel (GEMM1+GEMM2 in one launch);
    fused=False: two tcgen05 launches; simt=True: CUDA-core cross-check.
    need/ready: optional per-expert fill sequence numbers / device flags
    (vmm_grouped_swiglu_fused's copy overlap).  x_rows/src_row: gather the
    GEMM1 rows from the token rows (TMA gather4) -- xp may then be None and
    only its row count matters (pass an int).  order: optional i32 [E] device
    permutation, the fused CTA-pair kernel's expert walk order.
    arena: bf16 [n_slots, 3*I*H] -- per slot W13 ([2I,H], interleaved) then W2 ([H,I])."""
    if src_row is not None:
        M, H = int(xp), int(x_rows.shape[1])
        dev, xp = x_rows.device, None
    else:
        M, H = (int(s) for s in xp.shape)
        dev = xp.device
    E = int(offsets.shape[0]) - 1
    n_slots, stride = (int(s) for s in arena.shape[:2])
    if stride != 3 * inter * H:
        raise ValueError("arena slot must hold W13 and W2 (3*I*H elements)")
    w2_base = arena.data_ptr() + 2 * inter * H * 2
    h1 = torch.empty(M, inter, dtype=torch.bfloat16, device=dev) if h1 is None else h1
    y = torch.empty(M, H, dtype=torch.bfloat16, device=dev) if y is None else y
    L = _lib.lib()
    if simt:
        _n(2)
        check(L.vmm_grouped_swiglu_simt(ptr(xp), ptr(offsets), E, M, H, inter, ptr(arena), w2_base, stride,
                                        ptr(slot_of), ptr(h1), ptr(y), stream_ptr(stream)))
    elif fused:
        _n(1)
        done = torch.empty(M // 128 + E + 1, dtype=torch.int32, device=dev)
        check(L.vmm_grouped_swiglu_fused_ex(ptr(xp), ptr(offsets), E, M, H, inter, ptr(arena), w2_base, stride,
                                            n_slots, ptr(slot_of), ptr(need), ready, ready_base, ptr(done),
                                            ptr(x_rows), ptr(src_row), 0 if x_rows is None else int(x_rows.shape[0]),
                                            ptr(h1), ptr(y), ptr(order), stream_ptr(stream)))
    else:
        _n(1 if M <= 16 else 2)
        check(L.vmm_grouped_swiglu(ptr(xp), ptr(offsets), E, M, H, inter, ptr(arena), w2_base, stride, n_slots,
                                   ptr(slot_of), ptr(h1), ptr(y), stream_ptr(stream)))
    return h1, y


def pack_expert(w_gate, w_up, w_down):
    """One arena/host-pool slot: [interleaved W13 (2I*H) | W2 (H*I)] bf16, flat."""
    return torch.cat([interleave_w13(w_gate, w_up).reshape(-1), w_down.reshape(-1)])


def shared_plan(N: int, S: int, src, offsets, stream=None):
    _n(1)
    check(_lib.lib().vmm_shared_plan(N, S, ptr(src), ptr(offsets), stream_ptr(stream)))
    return src[: N * S], offsets


def combine_shared(y, pos, gates, resid, ys, S: int, stream=None, out=None):
    N, k = (int(s) for s in gates.shape)
    H = int(y.shape[1])
    out = torch.empty(N, H, dtype=torch.bfloat16, device=y.device) if out is None else out
    _n(1)
    check(_lib.lib().vmm_combine_shared(ptr(y), ptr(pos), ptr(gates), ptr(resid), N, k, H, ptr(ys), S, ptr(out),
                                        stream_ptr(stream)))
    return out


def rmsnorm(x, weight=None, eps: float = 1e-6, stream=None, out=None):
    n, H = (int(s) for s in x.shape)
    out = torch.empty_like(x) if out is None else out
    _n(1)
    check(_lib.lib().vmm_rmsnorm(ptr(x), ptr(weight), n, H, float(eps), ptr(out), stream_ptr(stream)))
    return out


def decode_glue(y, pos_prev, gates_prev, resid, tr_l, tg_l, rows, experts: int, out=None, xn=None, stream=None):
    """One-launch decode glue (vmm_decode_glue): returns (out, xn, ids, gates,
    offsets, src_row, pos, xp).  y=None: resid is the layer input (no combine)."""
    n, H = (int(s) for s in resid.shape)
    k = int(tr_l.shape[1])
    dev = resid.device
    out = torch.empty_like(resid) if out is None else out
    xn = torch.empty_like(resid) if xn is None else xn
    ids = torch.empty(n, k, dtype=_i32, device=dev)
    gates = torch.empty(n, k, dtype=torch.float32, device=dev)
    offsets = torch.empty(experts + 1, dtype=_i32, device=dev)
    src = torch.empty(n * k, dtype=_i32, device=dev)
    pos = torch.empty(n * k, dtype=_i32, device=dev)
    xp = torch.empty(n * k, H, dtype=resid.dtype, device=dev)
    _n(1)
    check(_lib.lib().vmm_decode_glue(ptr(y), ptr(pos_prev), ptr(gates_prev), ptr(resid), n, k, H, ptr(out), ptr(xn),
                                     ptr(tr_l), ptr(tg_l), ptr(rows), experts, ptr(ids), ptr(gates), ptr(offsets),
                                     ptr(src), ptr(pos), ptr(xp), stream_ptr(stream)))
    return out, xn, ids, gates, offsets, src, pos, xp


def combine(y, pos, gates, resid, stream=None, out=None):
    N, k = (int(s) for s in gates.shape)
    H = int(y.shape[1])
    out = torch.empty(N, H, dtype=torch.bfloat16, device=y.device) if out is None else out
    _n(1)
    check(_lib.lib().vmm_combine(ptr(y), ptr(pos), ptr(gates), ptr(resid), N, k, H, ptr(out), stream_ptr(stream)))
    return out


def interleave_w13(w_gate, w_up):
    """[I,H] gate and up projections -> the arena's [2I,H] layout (64-row blocks
    of gate rows followed by the matching 64 up rows)."""
    I, H = (int(s) for s in w_gate.shape)
    if I % 64:
        raise ValueError("inter size must be a multiple of 64")
    g = w_gate.reshape(I // 64, 64, H)
    u = w_up.reshape(I // 64, 64, H)
    return torch.stack([g, u], dim=1).reshape(2 * I, H).contiguous()


def ceil_div(a, b):
    return -(-a // b)


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("math", "torch")]
