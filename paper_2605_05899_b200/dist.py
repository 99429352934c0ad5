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


class SharedHostPool:
    """The node's expert pool in POSIX shared memory, page-locked in every rank
    (SURVEY 8(e) mode DP: "each GPU runs its own policy and slab cache, against
    one portable pinned pool").  Local rank 0 creates and sizes the segment
    (posix_fallocate, so a full /dev/shm fails here rather than at a page
    fault), every local rank maps it MAP_SHARED and registers it with
    cudaHostRegisterPortable (vmm_host_register) for its own context, and the
    name is unlinked once all ranks hold a mapping: one copy of the experts per
    node, and nothing left behind if a rank dies.  `filler` is True on the one
    rank that must write the weights; the others wait in `ready()`.
    `create()` returns None when the segment cannot be made on any rank (the
    caller then pins a pool per rank); all ranks agree on the outcome."""

    def __init__(self, mm, nbytes, addr, filler):
        self.mm, self.nbytes, self.addr, self.filler = mm, nbytes, addr, filler
        self._registered = False

    @staticmethod
    def create(nbytes: int, tag: str, device=None):
        import ctypes as C
        import mmap

        from . import _lib

        rank, world, _ = env_rank_world()
        if world == 1 or not dist.is_initialized():
            return None
        # ranks spawned without torchrun (tests) carry no LOCAL_RANK: one node, local = global rank
        local = int(os.environ["LOCAL_RANK"]) if "LOCAL_RANK" in os.environ else rank
        path = f"/dev/shm/vmm_pool_{tag}"
        ok, fd = 1, -1
        if local == 0:
            try:
                try:
                    os.unlink(path)  # a stale segment of an earlier job with the same tag
                except FileNotFoundError:
                    pass
                fd = os.open(path, os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
                os.posix_fallocate(fd, 0, nbytes)
            except OSError:
                ok = 0
        ok = int(-max_over_ranks(-ok, device))  # min over ranks: every rank takes the same branch
        if not ok:
            if fd >= 0:
                os.close(fd)
                os.unlink(path)
            return None
        barrier()
        if local != 0:
            fd = os.open(path, os.O_RDWR)
        try:
            mm = mmap.mmap(fd, nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        finally:
            os.close(fd)
        addr = C.addressof(C.c_char.from_buffer(mm))
        _lib.check(_lib.lib().vmm_host_register(addr, nbytes))
        barrier()  # every rank holds a mapping: the name can go
        if local == 0:
            os.unlink(path)
        pool = SharedHostPool(mm, nbytes, addr, filler=local == 0)
        pool._registered = True
        return pool

    def ready(self):
        """Fence after the filler wrote the weights."""
        barrier()

    def close(self):
        if self._registered:
            try:
                from . import _lib

                _lib.lib().vmm_host_unregister(self.addr)
            except Exception:  # noqa: BLE001  (interpreter teardown: the context may be gone)
                pass
            self._registered = False
