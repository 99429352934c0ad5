"""Expert-parallel token exchange on the device.

world=1 in-process, and world=2 as two processes sharing this one GPU (IPC-
mapped peer buffers, gloo for the G x G count exchange and the phase
barriers): every rank's hidden states equal a layer-by-layer run of its own
requests on resident experts, bit for bit (each output row depends only on its
own input row and the expert weights, whichever rank computes it)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cfg():
    from paper_2605_05899_b200.moe import StackConfig

    return StackConfig(layers=8, hidden=256, experts=8, k=2, inter=512, l_pinned=2, num_slabs=24, alpha=0.05,
                       beta=0.25, predictor="none", budget=0, window=3, routing="live")


def _requests(cfg, seeds):
    from paper_2605_05899_b200.trace import TraceGenConfig, generate_trace

    trs = [generate_trace(TraceGenConfig(n_visual=576, n_text=64, layers=cfg.layers, experts=cfg.experts, k=cfg.k,
                                         seed=s)) for s in seeds]
    g = torch.Generator(device="cuda").manual_seed(int(seeds[0]))
    x = torch.randn((sum(t.num_tokens for t in trs), cfg.hidden), generator=g, device="cuda").to(torch.bfloat16)
    sal = torch.from_numpy(np.concatenate([t.saliency for t in trs])).cuda()
    mod = torch.from_numpy(np.concatenate([t.device_modality() for t in trs])).cuda()
    offs = np.cumsum([0] + [t.num_tokens for t in trs]).tolist()
    return x, sal, mod, offs


def _resident_reference(cfg, store, x, retained):
    from paper_2605_05899_b200 import kernels
    from paper_2605_05899_b200.moe import moe_layer_forward

    E = cfg.experts
    arena = torch.stack([store.pool[(l % store.host_layers) * E + e] for l in range(cfg.layers)
                         for e in range(E)]).cuda()
    cur = x
    for l in range(cfg.layers):
        if l == cfg.l_pinned:
            cur = kernels.gather_rows(cur, torch.from_numpy(retained.astype(np.int32)).cuda())
        xn = kernels.rmsnorm(cur)
        ids, gates, _ = kernels.route_topk(xn, store.router[l], cfg.k)
        cur = moe_layer_forward(cur, ids, gates, arena, torch.arange(l * E, (l + 1) * E, dtype=torch.int32,
                                                                      device="cuda"), cfg.inter, E, xn=xn)
    return cur


def test_ep_world1_matches_resident_run():
    from paper_2605_05899_b200.ep import EPStack
    from paper_2605_05899_b200.moe import ExpertStore

    cfg = _cfg()
    store = ExpertStore(cfg, seed=5)
    x, sal, mod, offs = _requests(cfg, [1, 2, 3])
    ep = EPStack(cfg, store=store, max_rows=4096)
    h, ret, _ = ep.forward(x, sal, mod, req_off=offs)
    torch.cuda.synchronize()
    ref = _resident_reference(cfg, store, x, ret)
    assert torch.equal(h, ref)
    ep.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2605_05899_b200.ep import EPStack
        from paper_2605_05899_b200.moe import ExpertStore

        cfg = _cfg()
        store = ExpertStore(cfg, seed=5)  # same model on every rank
        x, sal, mod, offs = _requests(cfg, [10 + 3 * rank, 11 + 3 * rank, 12 + 3 * rank])
        ep = EPStack(cfg, store=store, rank=rank, world=world, max_rows=4096, device_of_rank=[0] * world)
        h, ret, _ = ep.forward(x, sal, mod, req_off=offs)
        torch.cuda.synchronize()
        ref = _resident_reference(cfg, store, x, ret)
        ok = bool(torch.equal(h, ref))
        dist.barrier()
        ep.close()
        dist.destroy_process_group()
        q.put((rank, ok, int(h.shape[0])))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, f"error: {exc!r}", 0))


def test_ep_world2_two_processes_one_gpu():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert [o[1] for o in outs] == [True, True], outs
    assert all(o[2] > 0 for o in outs)


def _sharded_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2605_05899_b200.moe import ExpertStore, MoEStack, ShardedHome, StackConfig

        cfg = StackConfig(**{**_cfg().__dict__, "predictor": "history", "budget": 4})
        store = ExpertStore(cfg, seed=5)
        home = ShardedHome(store, rank, world, device_of_rank=[0] * world)
        stack = MoEStack(cfg, store=store, home=home)
        x, sal, mod, offs = _requests(cfg, [30 + rank, 40 + rank])
        res = stack.forward(x, sal, mod, req_off=offs)
        torch.cuda.synchronize()
        ref = _resident_reference(cfg, store, x, res.retained)
        ok = bool(torch.equal(res.hidden, ref)) and res.copies > 0
        dist.barrier()
        home.close()
        dist.destroy_process_group()
        q.put((rank, ok, res.copies))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, f"error: {exc!r}", 0))


def test_sharded_cache_world2_peer_pulls_bit_identical():
    """Sharded expert cache with 2 ranks on one GPU: misses are copy-engine
    pulls from the peer rank's IPC-mapped home copies; the cached run still
    equals the all-resident run bit for bit."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert [o[1] for o in outs] == [True, True], outs


def _pool_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2605_05899_b200.moe import ExpertStore

        cfg = _cfg()
        store = ExpertStore(cfg, seed=11)
        # every rank reads the segment the filler (local rank 0) wrote, through its own page-locked mapping:
        # a copy-engine H2D of the whole pool and a host-side checksum
        dev_copy = torch.empty(store.pool.shape, dtype=store.pool.dtype, device="cuda")
        dev_copy.copy_(store.pool, non_blocking=True)
        torch.cuda.synchronize()
        ck = float(dev_copy.float().abs().sum().item())
        same = bool(torch.equal(dev_copy.cpu(), store.pool))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, store.host_pool_kind, ck, same, float(store.router.float().abs().sum().item())))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, f"error: {exc!r}", 0.0, False, 0.0))


def test_dp_ranks_share_one_page_locked_host_pool():
    """SURVEY 8(e) mode DP: the ranks of a node share ONE expert pool (a /dev/shm
    segment page-locked in every rank); every rank's copy engine reads the
    weights the filler wrote, identical to a single-process store of the same
    seed (same generator stream: the router weights after the pool agree too)."""
    import torch.multiprocessing as mp

    from paper_2605_05899_b200.moe import ExpertStore

    ref = ExpertStore(_cfg(), seed=11)
    ref_ck = float(ref.pool.float().abs().sum().item())
    ref_router = float(ref.router.float().abs().sum().item())
    assert ref.host_pool_kind == "pinned per rank"  # alone: no process group, own pinned pool
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pool_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for rank, kind, ck, same, router_ck in outs:
        assert kind.startswith("shared"), outs
        assert same and ck == ref_ck and router_ck == ref_router, outs
