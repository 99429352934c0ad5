"""Data-parallel plumbing for multi-GPU runs (one process per GPU).

Requests are independent units (the reference builds a fresh engine and cache
per simulate call, pkg/src/moesim/pipeline.py:397), so the multi-GPU mode is
request data parallelism with no data-path collective: each rank owns an
engine, a slab cache, a copy stream and its share of the requests.  The only
collectives are bookkeeping: a barrier around timed regions, a max over ranks
of the step time, and a gather of per-rank counters.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str = "nccl", device=None) -> tuple[int, int]:
    rank, world, _ = env_rank_world()
    if world > 1 and not dist.is_initialized():
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, **kw)
    return rank, world


def shard_requests(n_requests: int, rank: int, world: int) -> list[int]:
    """Request r -> rank r mod world (SURVEY §8(e) DP placement)."""
    return [r for r in range(n_requests) if r % world == rank]


def _coll_device(device):
    """gloo collectives run on CPU tensors"""
    return torch.device("cpu") if dist.get_backend() == "gloo" else device


def max_over_ranks(value: float, device=None) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values, device=None) -> list[float]:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def barrier():
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
