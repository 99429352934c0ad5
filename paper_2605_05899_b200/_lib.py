"""ctypes binding of libvismmoe.so (the C-ABI declared in include/vismmoe.h).

The library is built in-tree by `paper_2605_05899_b200.build` for sm_100a.
There is deliberately no fallback: if the library is missing, or no sm_100
device is present when a device entry point is used, this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DeviceError, raise_status

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VMM_LIB") or os.path.join(HERE, "libvismmoe.so")  # VMM_LIB: dev override

P = C.c_void_p
I32 = C.c_int
I64 = C.c_longlong
F64 = C.c_double
SZ = C.c_size_t
PI32 = C.POINTER(C.c_int32)
PF64 = C.POINTER(C.c_double)


class EngineConfig(C.Structure):
    _fields_ = [
        ("layers", I32), ("experts", I32), ("num_slabs", I32), ("victim_fifo", I32),
        ("speculative_grace", I32), ("budget", I32), ("window", I32), ("l_pinned", I32),
        ("shared", I32), ("prefetching", I32), ("reactive", I32), ("event_log", I32),
        ("transfer_ms", F64), ("gpu_ms", F64), ("boot_ms", F64), ("decay", PF64),
    ]


class EngineEvent(C.Structure):
    _fields_ = [("t", F64), ("kind", C.c_int32), ("layer", C.c_int32), ("expert", C.c_int32), ("slab", C.c_int32)]


class EngineReport(C.Structure):
    _fields_ = [
        ("makespan", F64), ("total_compute", F64), ("total_transfer", F64), ("exposed_transfer", F64),
        ("prefill_ms", F64), ("hits", I64), ("misses", I64), ("stalls", I64), ("rejected_loads", I64),
        ("on_demand_transfers", I64), ("inflight_waits", I64), ("evictions", I64), ("decode_steps", I32),
    ]


class StackDesc(C.Structure):
    _fields_ = [
        ("layers", I32), ("experts", I32), ("k", I32), ("hidden", I32), ("inter", I32), ("l_pinned", I32),
        ("n_pinned_slots", I64), ("n_slots", I64), ("slot_bytes", SZ), ("host_layers", I32), ("cap_rows", I32),
        ("routing", I32), ("predictor", I32), ("counts_preset", I32),
        ("arena", P), ("pool", P), ("router", P), ("pinned_slot_of", P), ("layer_ids", P), ("pow_table", P),
        ("oracle_table", P), ("trace_routes", P), ("trace_gates", P), ("trace_tokens", I32),
        ("xn", P), ("xp", P), ("h1", P), ("y", P), ("out0", P), ("out1", P),
        ("ids", P), ("gates", P), ("off", P), ("src", P), ("pos", P),
        ("counts", P), ("la_counts", P), ("y_dev", P), ("slot_dev", P),
        ("counts_host", P), ("y_host", P), ("slot_host", P),
        ("shared", I32), ("shared_slot_of", P), ("shared_src", P), ("shared_off", P),
        ("xs", P), ("h1s", P), ("ys", P),
        ("need_host", P), ("need_dev", P), ("ffn_done", P),
        ("mlp_emb", P), ("mlp_drift", P), ("mlp_hv", P), ("mlp_ids", P),
        ("mlp_dim", I32), ("mlp_n_ids", I32), ("mlp_hidden", I32), ("mlp_bottleneck", I32),
        ("mlp_w1", P), ("mlp_b1", P), ("mlp_w2", P), ("mlp_b2", P), ("mlp_wo", P), ("mlp_bo", P),
        ("mlp_hist", P), ("route_batch_rows", I32), ("order_host", P), ("order_dev", P),
    ]


class StackOut(C.Structure):
    _fields_ = [("x_out", P), ("copies", I32), ("routes", P), ("ffn_start", P), ("ffn_end", P), ("n_demand", P),
                ("host_us", F64 * 4), ("copy_marks", P)]


_SIGS = {
    "vmm_last_error": (C.c_char_p, []),
    "vmm_abi_version": (I32, []),
    "vmm_launch_count": (I64, []),
    "vmm_device_check": (I32, [I32]),
    "vmm_prune": (I32, [P, P, P, P, P, P, F64, F64, I32, I32, I32, I32, I32, F64, P, P, P, P, P, P, P, P, P]),
    "vmm_retained_pack": (I32, [P, P, P, I32, P, P, P]),
    "vmm_gather_rows": (I32, [P, P, I32, I32, P, P]),
    "vmm_route_topk": (I32, [P, P, I32, I32, I32, I32, P, P, P, P, P]),
    "vmm_route_lookahead": (I32, [P, P, I32, I32, I32, I32, I32, I32, P, P, P, P, P]),
    "vmm_ffn_keep_h1": (I32, [I32]),
    "vmm_grouped_swiglu_decode": (I32, [P, P, I32, I32, I32, I32, P, P, I64, P, P, P, I32, P, P, P]),
    "vmm_route_topk_ex": (I32, [P, P, I32, I32, I32, I32, P, P, P, P, I32, P]),
    "vmm_route_lookahead_ex": (I32, [P, P, I32, I32, I32, I32, I32, I32, P, P, P, P, I32, P]),
    "vmm_normalize_counts": (I32, [P, I32, F64, P, P]),
    "vmm_demand_counts": (I32, [P, I32, I32, I32, I32, P, I32, P, I32, P, P]),
    "vmm_oracle_targets": (I32, [P, I32, I32, P, I32, I32, P, P, P]),
    "vmm_history": (I32, [P, I32, I32, P, I32, P, P, P]),
    "vmm_mlp_predict": (I32, [P, P, I32, P, P, I32, P, P, I32, I32, P, P, I32, P, P, I32, P, P, P, P, P]),
    "vmm_row_mean": (I32, [P, I32, P, I32, P, P, P]),
    "vmm_gate_lookahead": (I32, [P, P, I32, I32, I32, I32, P, P, P]),
    "vmm_permute_plan": (I32, [P, I32, I32, I32, P, P, P, P]),
    "vmm_permute_rows": (I32, [P, P, I32, I32, P, P]),
    "vmm_attn_saliency": (I32, [P, P, I32, I32, I32, I32, I32, C.c_float, P, P, P]),
    "vmm_attn_map_saliency": (I32, [P, I32, I32, I32, P, P]),
    "vmm_routing_diagnostics": (I32, [P, I32, I32, I32, I32, I32, P, P]),
    "vmm_ep_dispatch": (I32, [P, I32, P, I32, P, P, P, P, P, I32, I32, I32, P]),
    "vmm_ep_return": (I32, [P, I32, P, P, I32, P]),
    "vmm_permute": (I32, [P, I32, I32, I32, P, I32, P, P, P, P, P]),
    "vmm_combine": (I32, [P, P, P, P, I32, I32, I32, P, P]),
    "vmm_rmsnorm": (I32, [P, P, I32, I32, C.c_float, P, P]),
    "vmm_decode_glue": (I32, [P, P, P, P, I32, I32, I32, P, P, P, P, P, I32, P, P, P, P, P, P, P]),
    "vmm_grouped_swiglu": (I32, [P, P, I32, I32, I32, I32, P, P, I64, I64, P, P, P, P]),
    "vmm_grouped_swiglu_fused": (I32, [P, P, I32, I32, I32, I32, P, P, I64, I64, P, P, P, I32, P, P, P, I32, P, P, P]),
    "vmm_grouped_swiglu_fused_ex": (I32, [P, P, I32, I32, I32, I32, P, P, I64, I64, P, P, P, I32, P, P, P, I32, P, P, P,
                                          P]),
    "vmm_grouped_swiglu_simt": (I32, [P, P, I32, I32, I32, I32, P, P, I64, P, P, P, P]),
    "vmm_engine_create": (I32, [C.POINTER(EngineConfig), C.POINTER(P)]),
    "vmm_engine_destroy": (None, [P]),
    "vmm_engine_begin": (I32, [P, P]),
    "vmm_engine_layer": (I32, [P, I32, P, I32, I32, I32, P]),
    "vmm_engine_end_step": (I32, [P]),
    "vmm_engine_emit": (I32, [P, I32, P]),
    "vmm_engine_slots": (I32, [P, I32, P, I32, P]),
    "vmm_engine_finish": (I32, [P, C.POINTER(EngineReport)]),
    "vmm_engine_emits": (I32, [P, I32, I32]),
    "vmm_engine_events": (I32, [P, P, I32]),
    "vmm_engine_pending_events": (I32, [P]),
    "vmm_engine_copies": (I32, [P, P, I32]),
    "vmm_engine_decode_ms": (I32, [P, P, I32]),
    "vmm_engine_layer_stats": (I32, [P, P, I32]),
    "vmm_engine_slab_of": (I32, [P, I32, I32]),
    "vmm_engine_slab": (I32, [P, I32, PI32, PI32, PI32, PI32, PF64, PF64]),
    "vmm_cache_create": (I32, [I32, I32, C.POINTER(P)]),
    "vmm_cache_destroy": (None, [P]),
    "vmm_cache_lookup": (I32, [P, I32, I32, PF64]),
    "vmm_cache_request": (I32, [P, I32, I32, F64, I32, PI32, PI32, PI32, PI32]),
    "vmm_cache_set_ready": (I32, [P, I32, I32, F64]),
    "vmm_cache_complete": (I32, [P, I32, I32, F64]),
    "vmm_cache_cancel": (I32, [P, I32, I32]),
    "vmm_cache_executed": (I32, [P, I32, I32]),
    "vmm_cache_reclassify": (I32, [P, P, I32, I32, P, P, I32]),
    "vmm_cache_select_victim": (I32, [P]),
    "vmm_cache_info": (I32, [P, C.POINTER(I64), PI32, PI32]),
    "vmm_cache_slab": (I32, [P, I32, PI32, PI32, PI32, PI32, PF64, PF64, PI32, PI32, PI32]),
    "vmm_cache_slabs": (I32, [P, P, P, I32]),
    "vmm_cache_find": (I32, [P, I32, I32]),
    "vmm_xfer_create": (I32, [I32, SZ, I32, C.POINTER(P)]),
    "vmm_xfer_destroy": (None, [P]),
    "vmm_xfer_copy": (I32, [P, I32, P, P, SZ, I32]),
    "vmm_xfer_fence": (I32, [P, P, I32, P]),
    "vmm_xfer_ready": (P, [P]),
    "vmm_xfer_need": (I32, [P, P, I32, P]),
    "vmm_xfer_layer_done": (I32, [P, I32, P]),
    "vmm_xfer_sync": (I32, [P]),
    "vmm_xfer_join": (I32, [P, P]),
    "vmm_xfer_stats": (I32, [P, PF64, PF64, C.POINTER(I64)]),
    "vmm_xfer_reset_stats": (I32, [P]),
    "vmm_xfer_stream": (P, [P]),
    "vmm_xfer_issue_engine": (I32, [P, P, P, I32, I32, P, I64, SZ, PI32]),
    "vmm_xfer_issue_engine_ordered": (I32, [P, P, P, I32, I32, P, I64, SZ, I32, P, P, PI32]),
    "vmm_combine_shared": (I32, [P, P, P, P, I32, I32, I32, P, I32, P, P]),
    "vmm_shared_plan": (I32, [I32, I32, P, P, P]),
    "vmm_combine_norm": (I32, [P, P, P, P, I32, I32, I32, P, I32, C.c_float, P, P, P]),
    "vmm_xfer_set_sources": (I32, [P, P, I64]),
    "vmm_host_register": (I32, [P, SZ]),
    "vmm_host_unregister": (I32, [P]),
    "vmm_ipc_get": (I32, [P, P]),
    "vmm_ipc_open": (I32, [P, C.POINTER(P)]),
    "vmm_ipc_offset": (I32, [P, C.POINTER(I64)]),
    "vmm_ipc_close": (I32, [P]),
    "vmm_copy_async": (I32, [P, P, SZ, P]),
    "vmm_memset_async": (I32, [P, I32, SZ, P]),
    "vmm_copy2d_async": (I32, [P, SZ, P, SZ, SZ, SZ, P]),
    "vmm_peer_enable": (I32, [I32]),
    "vmm_gather_i32": (I32, [P, P, I32, I32, P, P]),
    "vmm_gather_f32": (I32, [P, P, I32, I32, P, P]),
    "vmm_stack_create": (I32, [C.POINTER(StackDesc), C.POINTER(P)]),
    "vmm_stack_destroy": (None, [P]),
    "vmm_stack_layers": (I32, [P, P, P, P, I32, I32, I32, I32, I32, P, P, C.POINTER(StackOut)]),
}

_lock = threading.Lock()
_lib = None
_device_ok = None


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def load():
    """Load the shared library (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2605_05899_b200.build` "
                    "(there is no CPU fallback)"
                )
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int) -> None:
    if status:
        msg = load().vmm_last_error().decode(errors="replace")
        raise_status(status, msg)


def lib():
    """Library handle for device entry points: requires an sm_100 GPU."""
    global _device_ok
    L = load()
    if _device_ok is None:
        import torch

        if not torch.cuda.is_available():
            _device_ok = False
        else:
            _device_ok = L.vmm_device_check(torch.cuda.current_device()) == 0
    if not _device_ok:
        raise DeviceError("the VisMMOE hot path needs an sm_100 (B200) device; no CPU fallback exists")
    return L


def ptr(t) -> int | None:
    """data_ptr of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ipc_export(dptr: int) -> bytes:
    """64-byte IPC handle + 8-byte offset of a device pointer inside its allocation."""
    L = lib()
    h = (C.c_char * 64)()
    check(L.vmm_ipc_get(dptr, h))
    off = C.c_longlong()
    check(L.vmm_ipc_offset(dptr, C.byref(off)))
    return bytes(h) + int(off.value).to_bytes(8, "little")


def ipc_import(blob: bytes) -> tuple[int, int]:
    """Map a peer's exported pointer: (mapped base to close later, pointer)."""
    L = lib()
    q = C.c_void_p()
    buf = (C.c_char * 64).from_buffer_copy(blob[:64])
    check(L.vmm_ipc_open(buf, C.byref(q)))
    return q.value, q.value + int.from_bytes(blob[64:72], "little")

