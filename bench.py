#!/usr/bin/env python3
"""Benchmark: prefill tokens/s through the VL-MoE layer stack on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3_qwen3vl]
    python bench.py --impl reference ...     # the reference CPU path (oracle port)

One step = one batch of R requests per GPU (default R=256; BASELINE.json
configs[4], the batch sweep of the configs[2] shape: Qwen3-VL-30B-A3B, each
request 2304 visual + 64 text tokens, 48 MoE layers, 128 experts top-8,
expert intermediate 768, 8 pinned layers, 826-slab expert cache) through the
whole stack: live router -> prune (per request) -> lookahead predictor ->
expert cache with real H2D expert transfers (shared by the batch) -> permute
-> grouped SwiGLU (tcgen05) -> combine.  `--requests 1` is the single-request
configs[2] line.  Synthetic bf16 hidden states and random-init weights of
that shape.

Multi-GPU (torchrun): requests are data-parallel, one engine + cache per GPU,
no data-path collective ("scaling": "weak"); time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="c3_qwen3vl")
    p.add_argument("--routing", default="live", choices=["live", "trace"])
    p.add_argument("--predictor", default=None)
    p.add_argument("--requests", type=int, default=256,
                   help="requests per GPU per step (BASELINE configs[4] batch sweep; 1 = one request per step)")
    p.add_argument("--source", default="host", choices=["host", "sharded", "ep"],
                   help="miss source: pinned host pool over PCIe, or HBM home copies sharded over the GPUs (NVLink)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--out", default=None)
    return p.parse_args()


# ---------------------------------------------------------------------------
def _host_info():
    """os.cpu_count(), the lscpu model name and the BLAS thread setting."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "model": model,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


def _cpu_restatement(w, T1, n_r):
    """The builder's torch-CPU fp32 restatement of router + expert FFN + combine
    (oracle/moe_ref.py) on one post-prefix layer of one request (n_r retained
    rows), all host threads -- labelled "restatement, not ref".
    Extrapolated to the stack: l_pinned layers on all T1 tokens plus the rest on
    n_r rows, at the measured per-row cost."""
    import torch

    from oracle import moe_ref

    nth = os.cpu_count() or 1
    torch.set_num_threads(nth)
    g = torch.Generator().manual_seed(0)
    H, I, E, k = w.hidden, w.inter, w.experts, w.k
    x = torch.randn(n_r, H, generator=g).to(torch.bfloat16)
    wg_r = (torch.randn(E, H, generator=g) / H ** 0.5).to(torch.bfloat16)
    # one weight set shared by every expert (the FLOPs, not the bytes, are the restatement's cost)
    w_gate = (torch.randn(I, H, generator=g) / H ** 0.5).to(torch.bfloat16)
    w_up = (torch.randn(I, H, generator=g) / H ** 0.5).to(torch.bfloat16)
    w_down = (torch.randn(H, I, generator=g) / I ** 0.5).to(torch.bfloat16)
    t0 = time.perf_counter()
    xn = (x.float() * torch.rsqrt(x.float().pow(2).mean(1, keepdim=True) + 1e-6)).to(torch.bfloat16)
    ids, gates, _ = moe_ref.route(xn, wg_r, k)
    off, src, pos = moe_ref.permute(ids, E)
    xr = xn[src]
    y = torch.empty(n_r * k, H, dtype=torch.bfloat16)
    for e in range(E):
        a, b = int(off[e]), int(off[e + 1])
        if b > a:
            _, y[a:b] = moe_ref.expert_ffn(xr[a:b], w_gate, w_up, w_down)
    moe_ref.combine(y, pos, gates, x)
    layer_s = time.perf_counter() - t0
    per_row = layer_s / n_r
    stack_s = per_row * (w.l_pinned * T1 + (w.layers - w.l_pinned) * n_r)
    return {"label": "restatement, not ref", "value": T1 / stack_s, "unit": "tokens/s", "threads": nth,
            "layer_ms": layer_s * 1e3, "sample": f"one post-prefix {w.name} layer on {n_r} rows "
            "(oracle/moe_ref.py: fp64 router, fp32 SwiGLU per expert, combine), extrapolated to the stack"}


# reference arm: the UNMODIFIED reference (moesim from baseline/_ref) on the host
# cores -- build_plan (compress) + simulate, its own public API and stock path
# (pipeline.py:191,768; compress.py:142).  The oracle port is timed beside it
# as a labelled secondary figure.
# ---------------------------------------------------------------------------
def load_moesim():
    """The reference package from its offline install (baseline/_ref); None if absent."""
    try:
        import moesim  # noqa: F401
        return sys.modules["moesim"]
    except ImportError:
        pass
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "moesim")):
        sys.path.insert(0, p)
        try:
            import moesim  # noqa: F401
            return sys.modules["moesim"]
        except ImportError:
            sys.path.remove(p)
    return None


_REF = {}


def _ref_setup(kind, w, seed=0):
    """Build one request's inputs for the reference path (in the parent, before fork)."""
    gen = {k: v for k, v in w.trace_config(seed=seed).__dict__.items()}
    if kind == "reference":
        m = load_moesim()
        tr = m.generate_trace(m.TraceGenConfig(**gen))
        cfg = m.SimConfig(**{k: v for k, v in ref_sim_dict(w).items() if k not in ("predictor", "l_pinned")},
                          l_pinned=w.l_pinned, predictor=m.PredictorSpec(**ref_sim_dict(w)["predictor"]))
        ccfg = m.CompressionConfig(alpha=w.alpha, beta=w.beta, lam=w.lam, prefix_layers=tuple(w.prefix_layers))
        _REF.update(kind=kind, m=m, trace=tr, cfg=cfg, ccfg=ccfg)
    else:
        from paper_2605_05899_b200.trace import TraceGenConfig, generate_trace

        _REF.update(kind=kind, trace=generate_trace(TraceGenConfig(**gen)), sim=ref_sim_dict(w),
                    comp=dict(alpha=w.alpha, beta=w.beta, lam=w.lam, prefix=list(w.prefix_layers)))


def _ref_request(_=None):
    """One request through the reference path; returns seconds."""
    t0 = time.perf_counter()
    if _REF["kind"] == "reference":
        m = _REF["m"]
        plan = m.build_plan(_REF["trace"], _REF["cfg"], _REF["ccfg"])
        m.simulate(_REF["trace"], plan, _REF["cfg"])
    else:
        from oracle import harness

        harness.simulate(_REF["trace"], _REF["sim"], _REF["comp"], False)
    return time.perf_counter() - t0


def ref_sim_dict(w):
    """Reference SimConfig for one request of workload w (the oracle predictor:
    the reference's default kind; it has no router, so no gate predictor)."""
    return dict(bandwidth_mb_per_ms=1.0, expert_size_mb=0.17, gpu_ms_per_expert=0.002, num_slabs=w.num_slabs,
                victim_policy="priority", speculative_grace=w.grace, l_pinned=w.l_pinned, shared_experts=0,
                compress_latency_ms=0.0, predictor_bootstrap_ms=0.0,
                predictor=dict(kind="oracle", budget=w.budget, window=w.window, gamma=w.gamma,
                               history_decay=w.history_decay))


def _ref_pool_rate(kind, w, cores, warmup, steps):
    """tokens/s of `cores` processes, one request each per step (fork after setup)."""
    import multiprocessing as mp

    _ref_setup(kind, w)
    pool = mp.get_context("fork").Pool(cores)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        pool.map(_ref_request, range(cores))
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    pool.close()
    pool.join()
    step = float(np.mean(times))
    return cores * w.n_tokens / step, step


def run_reference(a, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    kind = "reference" if load_moesim() is not None else "port"
    val, step = _ref_pool_rate(kind, w, cores, a.warmup, a.steps)
    port = None
    if kind == "reference":  # the builder's port beside it, labelled (not the arm's value)
        pv, ps = _ref_pool_rate("port", w, cores, 1, max(1, min(a.steps, 3)))
        port = {"label": "oracle port (oracle/harness.py), not the reference", "value": pv, "unit": "tokens/s",
                "ms_per_step": ps * 1e3}
    what = ("moesim.build_plan (compress) + moesim.simulate, unmodified reference from baseline/_ref"
            if kind == "reference" else "oracle port of moesim (baseline/_ref absent)")
    line = {
        "impl": "reference", "metric": "prefill tokens/s per VL-MoE layer stack", "value": val, "unit": "tokens/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference trace generator, seed 0)",
        "config": {"workload": w.name, "requests_per_step": cores, "path": what,
                   "routing": "trace (the reference has no router)",
                   "predictor": "oracle B=%d W=%d (the reference has no gate predictor)" % (w.budget, w.window),
                   "vs_ours": "decision path only: the reference moves no expert bytes and computes no expert "
                              "FLOPs; our arm routes live and predicts with the gate-reuse lookahead"},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": kind,
                         "sample": f"{cores} {w.name} requests per step, one per process ({what})",
                         "port": port},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class ClockSampler:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self, dev_index=0):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or f[0] != str(dev_index):
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


class _EPResult:
    """EP mode has no cache: no transfers, no decisions."""

    def __init__(self, hidden):
        self.hidden, self.h2d_bytes, self.h2d_ms, self.copies = hidden, 0.0, 0.0, 0
        self.report = type("R", (), dict(hit_rate=None, hits=0, misses=0, evictions=0))()


def measure_h2d_peak(torch, dev):
    """Best of 3 pinned 1 GiB host->device copies on this rank."""
    n = 1 << 30
    src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(n, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, n / (a.elapsed_time(b) * 1e-3) / 1e9)
    del src, dst
    return best


def measure_peer_peak(torch, dev, rank, world, device_of_rank=None, reps=10):
    """Best of `reps` 1 GiB copy-engine pulls from the next rank's HBM into this
    rank's (IPC-mapped peer pointer, peer access enabled: NVLink/NVSwitch on a
    multi-GPU box; a local D2D copy when the ranks share one device or world=1).
    Run on every rank at once, so the figure is the per-GPU rate under all-to-all load."""
    import torch.distributed as dist

    from paper_2605_05899_b200 import _lib as vlib

    L = vlib.lib()
    n = 1 << 30
    src = torch.empty(n, dtype=torch.uint8, device=dev).fill_(rank & 0xFF)
    dst = torch.empty(n, dtype=torch.uint8, device=dev)
    opened, ptr = None, src.data_ptr()
    if world > 1:
        handles = [None] * world
        dist.all_gather_object(handles, vlib.ipc_export(src.data_ptr()))
        peer = (rank + 1) % world
        vlib.check(L.vmm_peer_enable(peer if device_of_rank is None else int(device_of_rank[peer])))
        opened, ptr = vlib.ipc_import(handles[peer])
        dist.barrier()
    torch.cuda.synchronize(dev)
    s = torch.cuda.current_stream(dev)
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        vlib.check(L.vmm_copy_async(dst.data_ptr(), ptr, n, s.cuda_stream))
        b.record(s)
        b.synchronize()
        best = max(best, n / (a.elapsed_time(b) * 1e-3) / 1e9)
    ok = world == 1 or int(dst[0].item()) == ((rank + 1) % world) & 0xFF
    if opened is not None:
        vlib.check(L.vmm_ipc_close(opened))
    if world > 1:
        dist.barrier()
    del src, dst
    torch.cuda.synchronize(dev)
    return best if ok else None


def ffn_kernel_name(M: int, E: int, H: int, I: int) -> str:
    """The grouped-SwiGLU kernel libvismmoe launches for M picks (csrc/ffn_sm100.cu dispatch)."""
    wide = H % 256 == 0 and (2 * I) % 256 == 0
    if M <= 16:
        return "skinny_ffn_kernel (decode-sized, CUDA cores)"
    if wide and M >= 256 * E:
        return "ffn_pair_kernel (tcgen05 cta_group::2, 256x256 tiles, GEMM1+SwiGLU+GEMM2 in one launch)"
    return f"ffn_fused_kernel<{256 if wide else 128}> (tcgen05, 128x{256 if wide else 128} tiles, one launch)"


def step_roofline(w, T, n_r, report, ms, tc_tflops, hbm_gbs, link_gbs, skip_last, slot_bytes):
    """SURVEY 8(d) stack roofline: sum over layers of max(FLOP / tensor peak,
    HBM bytes / HBM peak, miss bytes / link peak) against the measured step.
    Per layer: FLOP = router 2*N_route*H*E + FFN 6*N_ffn*k*H*I; HBM bytes = the
    demanded experts' weights + one read of the layer input + one write of its
    output + the router weights (the minimum any implementation moves); miss
    bytes = the layer's transfers (report.per_layer) x the expert slot."""
    H, I, E, k, L, lp = w.hidden, w.inter, w.experts, w.k, w.layers, w.l_pinned
    stats = {s.layer: s for s in report.per_layer if s.phase == "prefill"}
    floor_s, parts = 0.0, {"tensor": 0.0, "hbm": 0.0, "link": 0.0}
    for l in range(L):
        n_route = T if l < lp else n_r
        n_ffn = n_route if (l < lp - 1 or (l == lp - 1 and not skip_last)) else n_r
        st = stats.get(l)
        ne = E if l < lp or st is None else int(st.hits + st.transfers)
        miss = 0 if l < lp or st is None else int(st.transfers)
        fl = 2.0 * n_route * H * E + 6.0 * n_ffn * k * H * I
        by = ne * slot_bytes + E * H * 2 + n_route * H * 2 + n_ffn * H * 2
        t = {"tensor": fl / (tc_tflops * 1e12), "hbm": by / (hbm_gbs * 1e9),
             "link": miss * slot_bytes / (link_gbs * 1e9) if link_gbs else 0.0}
        b = max(t, key=t.get)
        parts[b] += t[b]
        floor_s += t[b]
    return {"step_frac": floor_s * 1e3 / ms, "floor_ms": floor_s * 1e3,
            "floor_by_bound_ms": {k_: v * 1e3 for k_, v in parts.items()},
            "peaks": {"tensor_tflops": tc_tflops, "hbm_gbs": hbm_gbs, "link_gbs": link_gbs},
            "definition": "sum_layer max(FLOP/tensor, bytes/HBM, miss bytes/link) / ms_per_step; "
                          "sustained peaks (MEASURED_PEAKS.json) and the link peak measured in this run"}


def relaunch(a) -> int:
    """--gpus N without a torchrun environment: re-exec under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = parse()
    from paper_2605_05899_b200.configs import WORKLOADS

    w = WORKLOADS[a.workload]
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(a)
    if a.impl == "reference":
        return run_reference(a, w)

    import torch
    import torch.distributed as dist

    from paper_2605_05899_b200 import dist as vdist

    rank, world, local = vdist.env_rank_world()
    # VMM_SHARE_GPU=1 (test only): every rank on device 0 with gloo collectives, to exercise the
    # multi-rank paths on a one-GPU box (NCCL refuses two ranks on one GPU)
    share = bool(os.environ.get("VMM_SHARE_GPU"))
    local = 0 if share else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    vdist.init("gloo" if share else "nccl", dev)

    from paper_2605_05899_b200 import kernels
    from paper_2605_05899_b200.moe import MoEStack, StackConfig
    from paper_2605_05899_b200.trace import generate_trace

    predictor = a.predictor or ("gate" if a.routing == "live" else "oracle")
    from paper_2605_05899_b200.moe import ExpertStore, ShardedHome

    # link peaks, measured on every rank at once before the stack exists:
    # pinned H2D (the host pool's link) and a peer-HBM pull (NVLink; local D2D at world 1)
    vdist.barrier()
    h2d_rank_peak = measure_h2d_peak(torch, dev)
    h2d_peak_job = sum(vdist.sum_over_ranks([h2d_rank_peak], dev))
    p2p_peak = measure_peer_peak(torch, dev, rank, world, [0] * world if share else None)
    if p2p_peak is None:
        raise SystemExit(f"rank {rank}: the peer copy returned the wrong bytes")
    p2p_peak_min = -vdist.max_over_ranks(-p2p_peak, dev)  # the slowest rank's link
    # pinned host pool: layer l is served from pool layer l % 8 (every byte moved is a real PCIe
    # transfer); the same synthetic model at every N (9.7 GB pinned per rank)
    kw = dict(routing=a.routing, predictor=predictor, host_layers=8)
    # Calibrated logical clock (hard part 2: decide on a logical clock, execute on
    # real streams): one transfer = the expert slot at the link rate measured above; one
    # expert's compute = the roofline time of the average expert at this batch (retained
    # rows x k / E picks), at the sustained peaks.  Decisions stay exactly replayable: the
    # values are in the JSON line and in cfg.sim_config().
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(pk_path)) if os.path.exists(pk_path) else {}
    hbm_sus = float(peaks.get("hbm_gbs", 6650.0))
    tc_sus = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0)))
    rows_per_req = math.floor(w.beta * w.n_visual) + w.n_text
    picks_per_expert = a.requests * rows_per_req * w.k / w.experts
    kw["gpu_ms"] = max(w.expert_bytes / (hbm_sus * 1e9),
                       6.0 * picks_per_expert * w.hidden * w.inter / (tc_sus * 1e12)) * 1e3
    kw["transfer_ms"] = w.expert_bytes / (h2d_rank_peak * 1e9) * 1e3
    if a.source == "sharded":  # one slot pulled at the measured peer (or D2D) rate
        kw["transfer_ms"] = w.expert_bytes / (p2p_peak_min * 1e9) * 1e3
    if a.source == "ep":
        kw.update(predictor="none", budget=0)
        predictor = "none (expert-parallel: no cache)"
    cfg = StackConfig.from_workload(w, **kw)
    R = a.requests
    # one model for the whole job: every rank builds the same weights (the pinned prefix and router are
    # replicated; sharded/EP modes keep each expert's home copy on rank e % world)
    store = ExpertStore(cfg, seed=1000)
    home = ShardedHome(store, rank, world, device_of_rank=[0] * world if share else None) \
        if a.source == "sharded" else None
    if a.source == "ep":
        from paper_2605_05899_b200.ep import EPStack

        stack = EPStack(cfg, store=store, rank=rank, world=world, max_rows=R * (w.n_visual // 2 + w.n_text) + 64,
                        device_of_rank=[0] * world if share else None)
    else:
        stack = MoEStack(cfg, store=store, home=home)
    tr = generate_trace(w.trace_config(seed=rank * R))
    T1 = tr.num_tokens
    T = T1 * R
    g = torch.Generator(device=dev).manual_seed(rank)
    x = torch.randn((T, w.hidden), generator=g, device=dev).to(torch.bfloat16)
    # requests beyond the first: same shape, saliency drawn like the generator's Gamma(2, 1)
    rng = np.random.default_rng(1000 + rank)
    sal_np = np.concatenate([tr.saliency] + [rng.gamma(2.0, 1.0, size=T1) for _ in range(R - 1)])
    mod_np = np.concatenate([tr.device_modality()] * R)
    sal = torch.from_numpy(sal_np).to(dev)
    mod = torch.from_numpy(mod_np).to(dev)
    req_off = [r * T1 for r in range(R + 1)]
    dtr = None
    if a.routing == "trace":
        if R != 1:
            raise SystemExit("--routing trace supports --requests 1")
        dtr = dict(routes=torch.from_numpy(tr.route_experts.astype(np.int32)).to(dev),
                   gates=torch.from_numpy(tr.route_gates.astype(np.float32)).to(dev))
    # host copies for the end-to-end leg
    x_h = x.cpu().pin_memory()
    sal_h = sal.cpu().pin_memory()
    mod_h = mod.cpu().pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2 (126 MB)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    out_h = [None]

    # e2e: the batch's hidden states cross PCIe in request-aligned chunks on a side
    # stream, and the pinned prefix starts on each chunk as it lands (x_ready)
    side = torch.cuda.Stream(device=dev)
    n_chunks = 8 if (R >= 8 and a.source != "ep") else 1
    bounds = [req_off[(R * (c + 1)) // n_chunks] for c in range(n_chunks)]
    x_dev = torch.empty_like(x)  # device landing buffers (allocation is not a transfer)
    x_dev2 = torch.empty_like(x) if a.source != "ep" else None

    def step(e2e=False, read_back=True):
        x_ready = None
        if e2e:
            sd = sal_h.to(dev, non_blocking=True)
            md = mod_h.to(dev, non_blocking=True)
            side.wait_stream(torch.cuda.current_stream())
            x_ready, r0 = [], 0
            with torch.cuda.stream(side):
                for r1 in bounds:
                    x_dev[r0:r1].copy_(x_h[r0:r1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(side)
                    x_ready.append((r1, ev))
                    r0 = r1
            xd = x_dev
        else:
            xd, sd, md = x, sal, mod
        if a.source == "ep":
            if x_ready:
                torch.cuda.current_stream().wait_event(x_ready[-1][1])
            h, ret, _ = stack.forward(xd, sd, md, req_off=req_off)
            res = _EPResult(h)
        else:
            if x_ready and n_chunks == 1:  # one chunk: simply order the step after its copy
                torch.cuda.current_stream().wait_event(x_ready[-1][1])
                x_ready = None
            res = stack.forward(xd, sd, md, trace=dtr, req_off=req_off, x_ready=x_ready)
        if e2e and read_back:
            n = int(res.hidden.shape[0])
            if out_h[0] is None or out_h[0].shape[0] < n:  # pinned result buffer, allocated once
                out_h[0] = torch.empty((max(n, T), w.hidden), dtype=res.hidden.dtype, pin_memory=True)
            out = out_h[0][:n]
            out.copy_(res.hidden, non_blocking=True)
            return res, out
        return res, None

    def timed(n, e2e=False, prof=False):
        times, results = [], []
        for _ in range(n):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if prof:
                stack.profile = []
            e0.record()
            res, out = step(e2e)
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            results.append((res, list(stack.profile) if prof else None, out))
            stack.profile = None
        return times, results

    def timed_e2e_streamed(n):
        """End to end as a serving loop runs it, one timed region over the n steps: every
        step's inputs cross PCIe (pinned host -> HBM) and its result is read back (HBM ->
        pinned host).  The link is idle during a step's pinned prefix once that step's own
        inputs have landed, so step i+1's inputs are copied then, into the other half of a
        double-buffered landing area (the first step's inputs are copied inside the region in
        request-aligned chunks the prefix starts on as they land); step i's result is staged
        on the device and read back on its own stream beside step i+1's prefix.  Returns ms
        per step."""
        if a.source == "ep":  # the EP stack has no chunked-input path: the serial figure stands
            return float(np.mean(e2e_times))
        d2h = torch.cuda.Stream(device=dev)
        n0 = int(res0_rows[0])
        stage = [torch.empty((n0, w.hidden), dtype=torch.bfloat16, device=dev) for _ in range(2)]
        outs = [torch.empty((n0, w.hidden), dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
        xb = [x_dev, x_dev2]
        sb = [torch.empty_like(sal) for _ in range(2)]
        mb = [torch.empty_like(mod) for _ in range(2)]
        ev_d2h = [None, None]

        def enqueue_inputs(b):  # on the side stream, behind whatever it already holds
            evs, r0 = [], 0
            with torch.cuda.stream(side):
                sb[b].copy_(sal_h, non_blocking=True)
                mb[b].copy_(mod_h, non_blocking=True)
                for r1 in bounds:
                    xb[b][r0:r1].copy_(x_h[r0:r1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(side)
                    evs.append((r1, ev))
                    r0 = r1
            return evs

        barrier()
        main = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        side.wait_stream(main)
        pending = enqueue_inputs(0)
        for i in range(n):
            b = i & 1
            evs = pending
            if i + 1 < n:
                side.wait_stream(main)  # buffer b^1 was last read by step i-1's prefix (already queued)
                pending = enqueue_inputs(b ^ 1)
            if i == 0 and n_chunks > 1:
                res = stack.forward(xb[b], sb[b], mb[b], trace=dtr, req_off=req_off, x_ready=evs)
            else:
                main.wait_event(evs[-1][1])
                res = stack.forward(xb[b], sb[b], mb[b], trace=dtr, req_off=req_off)
            nr = int(res.hidden.shape[0])
            if nr > n0:
                raise SystemExit("retained rows grew between steps")
            if ev_d2h[b] is not None:
                main.wait_event(ev_d2h[b])  # staging buffer b's previous read-back is done
            stage[b][:nr].copy_(res.hidden)
            ev = torch.cuda.Event()
            ev.record(main)
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                outs[b][:nr].copy_(stage[b][:nr], non_blocking=True)
            ev_d2h[b] = torch.cuda.Event()
            ev_d2h[b].record(d2h)
        main.wait_stream(d2h)
        main.wait_stream(side)
        e1.record(main)
        e1.synchronize()
        return e0.elapsed_time(e1) / n

    # warm-up
    timed(a.warmup)
    barrier()
    from paper_2605_05899_b200 import _lib as vlib

    launches0 = vlib.load().vmm_launch_count()
    with ClockSampler(os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")
                      if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "/tmp/clocks.csv") as clk:
        times, results = timed(a.steps, prof=True)
    launches = (vlib.load().vmm_launch_count() - launches0) // max(a.steps, 1)
    timed(1, e2e=True)  # warm the e2e path (pinned result buffer) outside the timed steps
    e2e_times, e2e_results = timed(a.steps, e2e=True)  # serial: each step's read-back inside its own step
    res0_rows = [int(results[-1][0].hidden.shape[0])]
    timed_e2e_streamed(1)  # warm the streamed path's buffers
    ms_e2e_streamed = timed_e2e_streamed(a.steps)

    def max_over_ranks(v):
        return vdist.max_over_ranks(v, dev)

    ms = max_over_ranks(float(np.mean(times)))
    ms_e2e_serial = max_over_ranks(float(np.mean(e2e_times)))
    ms_e2e = max_over_ranks(float(ms_e2e_streamed))
    value = world * T / (ms * 1e-3)
    e2e_value = world * T / (ms_e2e * 1e-3)

    # roofline: the fused grouped SwiGLU (dominant kernel).  Inside the step its
    # duration includes the per-expert waits on the copy stream (it starts while
    # the layer's misses still stream in), so the kernel's own rate is measured
    # by replaying the LAST layer's FFN launch on its real inputs (permuted rows,
    # expert offsets, slot table) with every expert resident, L2 flushed before
    # each replay, CUDA events on the launching stream.
    prof = [p for _, pl, _ in results for p in pl if not p[4]]  # cached layers (not the pinned prefix)
    live_ms = float(np.mean([p[0].elapsed_time(p[1]) for p in prof])) if prof else None
    bufs = stack._bufs
    if a.source == "ep":  # the owner-side FFN of the last layer: the rows this rank received
        xp_r, off, last_l, M = stack.last_ffn
        arena_r, slot_row = stack.owner.arena, stack.local_slots[last_l]
    else:
        n_r = int(results[-1][0].hidden.shape[0])
        M = n_r * w.k
        off = bufs["off"]
        xp_r, arena_r, slot_row = bufs["xp"][:M], stack.store.arena, stack.slot_dev[w.layers - 1]
    ne = int((off[1:] - off[:-1] > 0).sum().item())
    durs = []
    for _ in range(5):
        flush.zero_()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        kernels.grouped_swiglu(xp_r, off, arena_r, slot_row, w.inter, h1=bufs["h1"][:M], y=bufs["y"][:M])
        f1.record()
        f1.synchronize()
        durs.append(f0.elapsed_time(f1))
    # algorithmic bytes: weights of the demanded experts + permuted rows (read) + Y (write); H1 never
    # has to leave the chip (the CTA-pair kernel drops consumed H1 rows from L2 without write-back)
    nbytes = [ne * cfg.slot_bytes + M * w.hidden * 2 * 2]
    nflops = [6.0 * M * w.hidden * w.inter]
    durs = [float(np.mean(durs))]
    peaks = {}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        peaks = json.load(open(pk_path))
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    tc_peak = float(peaks.get("bf16_tflops", 1590.0))
    t_mem = sum(nbytes) / (hbm_peak * 1e9)
    t_tc = sum(nflops) / (tc_peak * 1e12)
    t_act = sum(durs) * 1e-3
    if t_tc > t_mem:
        bound, ach, peak, unit = "tensor", sum(nflops) / t_act / 1e12, tc_peak, "TFLOP/s"
        peak_src = "of measured (MEASURED_PEAKS.json bf16_tflops)" if "bf16_tflops" in peaks else \
            "of fallback (B200_PROFILING.md: 1.59 PFLOP/s burst)"
    else:
        bound, ach, peak, unit = "hbm", sum(nbytes) / t_act / 1e9, hbm_peak, "GB/s"
        peak_src = "of measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else \
            "of fallback (B200_PROFILING.md: 6.65 TB/s)"
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath)).get(f"{w.name}/R{a.requests}")
        if tj:
            traffic = tj["dram_bytes_per_launch"]
            traffic_src = f"from profiles/ncu_traffic.json ({tj.get('source', 'ncu --set full capture')}), " \
                          "not measured in this run"
    res0 = results[-1][0]
    h2d_peak = h2d_peak_job if a.source == "host" else (p2p_peak_min * world if a.source == "sharded" else None)
    h2d_bytes = res0.h2d_bytes
    rep = res0.report
    # whole-job counters (mode DP: one sum-reduction of the per-rank counters)
    hits, misses, evictions, copies = rep.hits, rep.misses, rep.evictions, res0.copies
    retained = int(res0.hidden.shape[0])
    if world > 1:
        hits, misses, evictions, copies, h2d_bytes, retained = (v for v in vdist.sum_over_ranks(
            [hits, misses, evictions, copies, h2d_bytes, retained], dev))
    hit_rate = hits / (hits + misses) if (hits or misses) and rep.hit_rate is not None else rep.hit_rate
    h2d_gbs = h2d_bytes / (ms * 1e-3) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            def single_thread(kind, budget_s):
                _ref_setup(kind, w)
                t0, n = time.perf_counter(), 0
                while time.perf_counter() - t0 < budget_s or n == 0:
                    _ref_request()
                    n += 1
                return T1 * n / (time.perf_counter() - t0), n

            kind = "reference" if load_moesim() is not None else "port"
            v, n_req = single_thread(kind, 10.0)
            cpu = {"value": v, "unit": "tokens/s", "cores": 1, "kind": kind,
                   "sample": f"{n_req} x one {w.name} request, single thread: " +
                             ("moesim.build_plan + moesim.simulate (unmodified reference, oracle predictor)"
                              if kind == "reference" else "oracle port (compress + simulate, oracle predictor)")}
            if kind == "reference":
                pv, pn = single_thread("port", 3.0)
                cpu["port"] = {"label": "oracle port (oracle/harness.py), not the reference", "value": pv,
                               "unit": "tokens/s", "cores": 1, "sample": f"{pn} requests"}
            cpu["host"] = _host_info()
            try:
                cpu["restatement"] = _cpu_restatement(w, T1, max(1, int(res0.hidden.shape[0]) // R))
            except Exception as exc:  # noqa: BLE001
                cpu["restatement"] = {"label": "restatement, not ref", "value": None, "sample": f"failed: {exc}"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "tokens/s", "cores": 1, "kind": "port", "sample": f"failed: {exc}"}

    step_rl = None
    if a.source != "ep":
        skip_last = a.routing == "live" and w.shared_experts == 0 and not os.environ.get("VMM_PREFIX_FULL_LAST")
        link = h2d_rank_peak if a.source == "host" else p2p_peak_min
        step_rl = step_roofline(w, T, int(res0.hidden.shape[0]), rep, ms, tc_sus, hbm_sus, link, skip_last,
                                cfg.slot_bytes)
    if rank == 0:
        line = {
            "metric": "prefill tokens/s per VL-MoE layer stack", "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, N(0,1) hidden states, reference trace generator saliency)",
            "config": {"workload": w.name, "tokens": T, "layers": w.layers, "hidden": w.hidden, "experts": w.experts,
                       "top_k": w.k, "moe_inter": w.inter, "l_pinned": w.l_pinned, "num_slabs": w.num_slabs,
                       "routing": a.routing, "predictor": f"{predictor} B={w.budget} W={w.window}",
                       "miss_source": a.source, "host_pool": store.host_pool_kind,
                       "parallelism": f"dp{world} (requests)", "requests_per_gpu_step": R,
                       "l2": "flushed (256 MB write) between the timed device-resident steps; the streamed e2e "
                             "loop runs without a flush on "
                             + ("inputs larger than L2" if T * w.hidden * 2 > (126 << 20) else "inputs smaller than L2")
                             + f" (hidden states {T * w.hidden * 2 / 1e9:.3f} GB per step)"},
            "hit_rate": hit_rate, "hits": int(hits), "misses": int(misses), "evictions": int(evictions),
            "retained_tokens": int(retained),
            "h2d": {"gbs": h2d_gbs, "bytes_per_step": h2d_bytes, "copies_per_step": int(copies),
                    "window_ms": res0.h2d_ms,
                    "window_gbs": h2d_bytes / (res0.h2d_ms * 1e-3) / 1e9 if res0.h2d_ms else None,
                    "peak_gbs": h2d_peak, "frac": h2d_gbs / h2d_peak if h2d_peak else None,
                    "link": "PCIe (pinned host pool)" if a.source == "host" else
                            ("none: expert-parallel, token rows over peer memory" if a.source == "ep" else
                             ("NVLink P2P + local D2D (sharded HBM home copies)" if world > 1 else
                              "local D2D (HBM home)")),
                    "peak_source": ("pinned 1 GiB H2D, measured in this run on all ranks at once (job sum)"
                                    if a.source == "host" else
                                    "1 GiB peer-HBM pull (IPC, copy engine), best of 10, all ranks at once "
                                    "(min over ranks x world)" if world > 1 else "1 GiB local D2D copy, best of 10")},
            "links": {"h2d_gbs_per_rank": h2d_rank_peak, "h2d_gbs_job": h2d_peak_job,
                      "peer_gbs_per_rank_min": p2p_peak_min,
                      "peer_kind": ("NVLink P2P (IPC-mapped peer HBM)" if world > 1 and not share else
                                    "same-device IPC copy (ranks share one GPU)" if world > 1 else "local D2D")},
            "roofline": {"bound": bound,
                         "kernel": ffn_kernel_name(M, w.experts, w.hidden, w.inter),
                         "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                         "traffic": traffic, "traffic_source": traffic_src, "launch_ms": float(np.mean(durs)),
                         "timing": "last layer's FFN replayed on its real inputs, experts resident, L2 flushed",
                         "live_launch_ms_incl_copy_waits": live_ms,
                         "bytes_per_launch": float(np.mean(nbytes)), "flops_per_launch": float(np.mean(nflops)),
                         "hbm_frac": (sum(nbytes) / t_act / 1e9) / hbm_peak,
                         "tensor_frac": (sum(nflops) / t_act / 1e12) / tc_peak,
                         # the replay runs right after the long timed steps, in the power-capped regime the
                         # in-step FFN runs in: its fraction of the SUSTAINED tensor peak beside the burst one
                         "tensor_frac_of_sustained": (sum(nflops) / t_act / 1e12) / tc_sus,
                         "peak_source": peak_src,
                         "step": step_rl},
            "clocks": clk.summary(local),
            "gpu_launches": int(launches),
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": int(T * w.hidden * 2 + T * 9),
                    "d2h_bytes_per_step": int(res0.hidden.numel() * 2), "ms_per_step": ms_e2e,
                    "mode": "streamed: one timed region over the steps, every step's inputs H2D and result D2H "
                            "inside it; step i+1's inputs cross PCIe during step i's prefix (link idle), step i's "
                            "read-back runs beside step i+1's prefix",
                    "serial": {"value": world * T / (ms_e2e_serial * 1e-3), "ms_per_step": ms_e2e_serial,
                               "mode": "each step's H2D and D2H inside its own timed step"}},
            "cpu_baseline": cpu,
            "config_clock": {"transfer_ms": cfg.transfer_ms, "gpu_ms": cfg.gpu_ms,
                             "basis": "transfer = expert slot / measured link peak; gpu = roofline time of the "
                                      "average expert's picks at sustained peaks"},
        }
        print(json.dumps(line), flush=True)
        if a.out:
            with open(a.out, "w") as f:
                json.dump(line, f, indent=1)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
