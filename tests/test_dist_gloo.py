"""World-size-2 data-parallel path on CPU (gloo): request sharding, per-rank
native engines, max-over-ranks timing and counter reduction.  Each rank's
decision stream must equal the single-process stream for the same requests."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_05899_b200 import dist as vdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _requests(n):
    """Synthetic per-request demand lists (L=6 layers, E=8 experts, 1 pinned layer)."""
    out = []
    for r in range(n):
        rng = np.random.default_rng(100 + r)
        out.append([np.sort(rng.choice(8, size=int(rng.integers(1, 6)), replace=False)).astype(np.int32)
                    for _ in range(6)])
    return out


def _run_request(demand):
    from paper_2605_05899_b200.pipeline import Engine, PredictorSpec, SimConfig

    cfg = SimConfig(bandwidth_mb_per_ms=1.0, expert_size_mb=2.0, gpu_ms_per_expert=1.0, l_pinned=1, num_slabs=10,
                    predictor=PredictorSpec(kind="none", budget=0), compress_latency_ms=0.0,
                    predictor_bootstrap_ms=0.0)
    eng = Engine(6, 8, cfg, 10, 1, 0, False, False, 0.0)
    eng.begin(None)
    for layer, dem in enumerate(demand):
        eng.layer(layer, dem, 0, -1, None)
    r = eng.finish(with_events=False)
    return [r.makespan, r.hits, r.misses, r.evictions, r.stalls]


def _worker(rank, world, port, n_req, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    vdist.init("gloo")
    reqs = _requests(n_req)
    mine = vdist.shard_requests(n_req, rank, world)
    results = {r: _run_request(reqs[r]) for r in mine}
    t = vdist.max_over_ranks(float(rank + 1) * 1.5)
    tot = vdist.sum_over_ranks([sum(v[1] for v in results.values()), sum(v[2] for v in results.values())])
    vdist.barrier()
    q.put((rank, results, t, tot))
    import torch.distributed as dist

    dist.destroy_process_group()


def test_data_parallel_world2_gloo():
    n_req, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_req, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    reqs = _requests(n_req)
    single = {r: _run_request(reqs[r]) for r in range(n_req)}
    seen = {}
    for rank, results, t, tot in outs:
        assert t == 3.0  # max over ranks of (rank+1)*1.5
        assert set(results) == set(vdist.shard_requests(n_req, rank, world))
        seen.update(results)
        assert tot == [float(sum(v[1] for v in single.values())), float(sum(v[2] for v in single.values()))]
    assert seen == single


def _ep_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist

    from paper_2605_05899_b200.ep import ep_layout

    vdist.init("gloo")
    E = 10  # not a multiple of the world size on purpose
    rng = np.random.default_rng(rank)
    mine = torch.from_numpy(rng.integers(0, 50, size=E).astype(np.int64))
    allc = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine)
    counts = np.stack([a.numpy() for a in allc])
    q.put((rank, counts, ep_layout(counts, rank)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ep_count_exchange_and_layout_gloo(world):
    """EP host plan: after the (source, expert) count exchange, every source's
    block of every expert lands at a disjoint range of the owner's buffer, the
    blocks are expert-major then source-ordered, and tile the buffer exactly."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = {r: (c, lay) for r, c, lay in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    counts = outs[0][0]
    G, E = counts.shape
    for r in range(world):
        assert np.array_equal(outs[r][0], counts)
    for d in range(world):
        _, off_local, n_recv = outs[d][1]
        assert n_recv == int(counts[:, d::G].sum())
        expect = 0
        for j, e in enumerate(range(d, E, G)):
            assert off_local[j] == expect
            for s in range(world):
                base, _, _ = outs[s][1]
                assert base[e] == expect  # source s's block of expert e starts here
                expect += int(counts[s, e])
        assert expect == n_recv == off_local[-1]
