"""End-to-end layer stack on the device.

* trace routing: the stack's cache decisions equal simulate() on the same trace
  (which is itself pinned to the reference) -- hits, misses, evictions, stalls,
  makespan, per-layer rows;
* live routing: the routes the run produced, replayed through the oracle
  restatement of the reference engine, give the same report (history and
  gate-lookahead predictors; the latter with the recorded scores);
* data path: hidden states after the cached run are bit-identical to a run
  with every expert resident (wrong slab / copy race would show up here) and
  close to a torch fp32 restatement of the stack.
"""
import numpy as np
import pytest
import torch

from oracle import harness, moe_ref
from paper_2605_05899_b200 import CompressionConfig, build_plan, simulate
from paper_2605_05899_b200.configs import WORKLOADS
from paper_2605_05899_b200.moe import ExpertStore, MoEStack, StackConfig
from paper_2605_05899_b200.trace import RoutingTrace, TraceGenConfig, generate_trace

pytestmark = pytest.mark.gpu

_F = ("makespan", "total_compute", "total_transfer", "exposed_transfer", "hits", "misses", "stalls",
      "on_demand_transfers", "inflight_waits", "evictions", "prefill_ms")


def tiny_cfg(**kw):
    base = dict(layers=8, hidden=256, experts=8, k=2, inter=512, l_pinned=2, num_slabs=24, alpha=0.05, beta=0.25,
                predictor="history", budget=4, window=3, host_layers=8, transfer_ms=0.3, gpu_ms=0.02)
    base.update(kw)
    return StackConfig(**base)


def request(trace, H, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    T = trace.num_tokens
    x = torch.randn((T, H), generator=g, device="cuda").to(torch.bfloat16)
    sal = torch.from_numpy(trace.saliency).cuda()
    mod = torch.from_numpy(trace.device_modality()).cuda()
    dtr = dict(routes=torch.from_numpy(trace.route_experts.astype(np.int32)).cuda(),
               gates=torch.from_numpy(trace.route_gates.astype(np.float32)).cuda())
    return x, sal, mod, dtr


def small_trace(cfg, seed=0):
    return generate_trace(TraceGenConfig(n_visual=576, n_text=64, layers=cfg.layers, experts=cfg.experts, k=cfg.k,
                                         cluster_support=4, visual_noise=0.3, seed=seed))


@pytest.mark.parametrize("pred", ["oracle", "history"])
def test_trace_routing_decisions_equal_simulate(pred):
    cfg = tiny_cfg(routing="trace", predictor=pred)
    tr = small_trace(cfg)
    stack = MoEStack(cfg)
    x, sal, mod, dtr = request(tr, cfg.hidden)
    res = stack.forward(x, sal, mod, trace=dtr)
    sim = cfg.sim_config()
    plan = build_plan(tr, sim, CompressionConfig(cfg.alpha, cfg.beta, cfg.lam, tuple(range(cfg.l_pinned))))
    assert res.retained.tolist() == plan.retained_ids(tr)
    rep = simulate(tr, plan, sim).to_dict()
    got = res.report.to_dict()
    for key in _F:
        assert got[key] == rep[key], key
    assert got["per_layer"] == rep["per_layer"]
    # every decided transfer was issued as exactly one copy
    sim.event_log = True
    issues = [e for e in simulate(tr, plan, sim).events if e[1] == "issue"]
    assert res.copies == len(issues) > 0
    assert res.h2d_bytes == len(issues) * cfg.slot_bytes


def _trace_from_run(cfg, tr_in, res):
    """RoutingTrace whose routes are the ones the live run produced."""
    T = tr_in.num_tokens
    re = np.zeros((cfg.layers, T, cfg.k), dtype=np.int64)
    re[:] = np.arange(cfg.k)
    re[: cfg.l_pinned] = res.prefix_routes.cpu().numpy()
    for i, l in enumerate(range(cfg.l_pinned, cfg.layers)):
        re[l, res.retained] = res.routes[i].cpu().numpy()
    return RoutingTrace(cfg.layers, cfg.experts, cfg.k, re, np.full(re.shape, 1.0 / cfg.k), tr_in.saliency,
                        tr_in.modality, tr_in.embedding)


def _sim_dict(cfg):
    s = cfg.sim_config()
    return dict(bandwidth_mb_per_ms=s.bandwidth_mb_per_ms, expert_size_mb=s.expert_size_mb,
                gpu_ms_per_expert=s.gpu_ms_per_expert, num_slabs=s.num_slabs, victim_policy=s.victim_policy,
                speculative_grace=s.speculative_grace, l_pinned=s.l_pinned, shared_experts=0,
                compress_latency_ms=s.compress_latency_ms, predictor_bootstrap_ms=s.predictor_bootstrap_ms,
                predictor=dict(kind=s.predictor.kind, budget=s.predictor.budget, window=s.predictor.window,
                               gamma=s.predictor.gamma, history_decay=s.predictor.history_decay))


@pytest.mark.parametrize("pred", ["history", "gate"])
def test_live_routing_decisions_replay_through_oracle(pred):
    cfg = tiny_cfg(routing="live", predictor=pred)
    tr = small_trace(cfg, seed=3)
    stack = MoEStack(cfg)
    x, sal, mod, _ = request(tr, cfg.hidden, seed=1)
    res = stack.forward(x, sal, mod, record=True)
    tr_live = _trace_from_run(cfg, tr, res)
    comp = dict(alpha=cfg.alpha, beta=cfg.beta, lam=cfg.lam, prefix=list(range(cfg.l_pinned)))
    y_over = (lambda ctx, ids: res.scores[ctx]) if pred == "gate" else None
    sd = _sim_dict(cfg)
    if pred == "gate":
        sd["predictor"]["kind"] = "history"  # placeholder kind; scores come from y_override
    exp = harness.simulate(tr_live, sd, comp, False, y_override=y_over)
    assert exp["hits"] + exp["misses"] > 0
    got = res.report.to_dict()
    for key in _F:
        assert got[key] == exp[key], key
    assert got["per_layer"] == exp["per_layer"]


def test_cached_run_bit_identical_to_all_resident_run():
    cfg = tiny_cfg(routing="live", predictor="history", num_slabs=24)
    store = ExpertStore(cfg, seed=7)
    tr = small_trace(cfg, seed=5)
    x, sal, mod, _ = request(tr, cfg.hidden, seed=2)
    res = MoEStack(cfg, store=store).forward(x, sal, mod, record=True)
    torch.cuda.synchronize()
    # every expert resident: pinned prefix covering all layers, no cache traffic
    full = StackConfig(**{**cfg.__dict__, "l_pinned": cfg.layers, "num_slabs": 1})
    # the prune must still see the same prefix: run the resident reference by hand
    E = cfg.experts
    arena = torch.stack([store.pool[(l % store.host_layers) * E + e] for l in range(cfg.layers) for e in range(E)]).cuda()
    from paper_2605_05899_b200.moe import moe_layer_forward
    from paper_2605_05899_b200 import kernels
    cur = x
    for l in range(cfg.l_pinned):
        xn = kernels.rmsnorm(cur)
        ids, gates, _ = kernels.route_topk(xn, store.router[l], cfg.k)
        cur = moe_layer_forward(cur, ids, gates, arena, torch.arange(l * E, (l + 1) * E, dtype=torch.int32,
                                                                      device="cuda"), cfg.inter, E, xn=xn)
    ret = torch.from_numpy(res.retained.astype(np.int32)).cuda()
    cur = kernels.gather_rows(cur, ret)
    x_in = []
    for l in range(cfg.l_pinned, cfg.layers):
        xn = kernels.rmsnorm(cur)
        x_in.append((cur, xn))
        ids, gates, _ = kernels.route_topk(xn, store.router[l], cfg.k)
        cur = moe_layer_forward(cur, ids, gates, arena, torch.arange(l * E, (l + 1) * E, dtype=torch.int32,
                                                                      device="cuda"), cfg.inter, E, xn=xn)
    torch.cuda.synchronize()
    assert res.copies > 0
    assert torch.equal(res.hidden, cur)
    # and close to a torch fp32 restatement of the last layer
    l = cfg.layers - 1
    xr, xl = (t.cpu() for t in x_in[-1])
    # rmsnorm restated in fp32 (bf16 rounded like the device) vs the device rows
    xnf = (xr.float() * torch.rsqrt(xr.float().pow(2).mean(1, keepdim=True) + 1e-6)).to(torch.bfloat16)
    torch.testing.assert_close(xnf.float(), xl.float(), rtol=1e-2, atol=1e-2)
    ids, gates, _ = moe_ref.route(xl, store.router[l].cpu(), cfg.k)
    acc = xr.float().clone()
    for t in range(0, xl.shape[0], 97):
        for j in range(cfg.k):
            e = int(ids[t, j])
            wg, wu, wd = store.expert(l, e)
            _, y = moe_ref.expert_ffn(xl[t:t + 1], wg, wu, wd)
            acc[t] += gates[t, j] * y[0].float()
    rows = list(range(0, xl.shape[0], 97))
    torch.testing.assert_close(res.hidden.cpu()[rows].float(), acc[rows], rtol=3e-2, atol=3e-2)


@pytest.mark.parametrize("n_req", [3, 44])
def test_batched_requests_share_transfers_and_replay_exactly(n_req):
    """R requests in one pass: each request is compressed on its own (prune CTA
    per request, identical to the oracle's per-request compress) and the
    layers run on the union of retained rows; the batch's decisions replay
    exactly through the oracle engine on the merged routes.  44 requests give
    > 8192 retained rows: the executor's early-decision split path."""
    from oracle import compress_ref
    cfg = tiny_cfg(routing="live", predictor="gate")
    trs = [small_trace(cfg, seed=s) for s in range(11, 11 + n_req)]
    stack = MoEStack(cfg)
    xs, sals, mods = [], [], []
    for i, tr in enumerate(trs):
        x, sal, mod, _ = request(tr, cfg.hidden, seed=20 + i)
        xs.append(x), sals.append(sal), mods.append(mod)
    offs = np.cumsum([0] + [t.num_tokens for t in trs]).tolist()
    res = stack.forward(torch.cat(xs), torch.cat(sals), torch.cat(mods), record=True, req_off=offs)
    T = offs[-1]
    re = np.zeros((cfg.layers, T, cfg.k), dtype=np.int64)
    re[:] = np.arange(cfg.k)
    re[: cfg.l_pinned] = res.prefix_routes.cpu().numpy()
    for i, l in enumerate(range(cfg.l_pinned, cfg.layers)):
        re[l, res.retained] = res.routes[i].cpu().numpy()
    # per-request compression of the live prefix routes == the batch's retained rows
    exp_ret = []
    for r, tr in enumerate(trs):
        o = compress_ref.compress(tr.saliency, tr.modality, [], re[:, offs[r]:offs[r + 1]], cfg.experts,
                                  cfg.alpha, cfg.beta, cfg.lam, list(range(cfg.l_pinned)))
        exp_ret.append(o["retained"] + offs[r])
    exp_ret = np.concatenate(exp_ret)
    assert res.retained.tolist() == exp_ret.tolist()
    assert res.retained_offsets[-1] == len(exp_ret)
    merged = RoutingTrace(cfg.layers, cfg.experts, cfg.k, re, np.full(re.shape, 1.0 / cfg.k),
                          np.concatenate([t.saliency for t in trs]), np.concatenate([t.modality for t in trs]),
                          np.concatenate([t.embedding for t in trs]))
    sd = _sim_dict(cfg)
    sd["predictor"]["kind"] = "history"
    comp = dict(alpha=cfg.alpha, beta=cfg.beta, lam=cfg.lam, prefix=list(range(cfg.l_pinned)))
    exp = harness.simulate(merged, sd, comp, False, y_override=lambda ctx, ids: res.scores[ctx], retained=exp_ret)
    got = res.report.to_dict()
    for key in _F:
        assert got[key] == exp[key], key
    assert got["per_layer"] == exp["per_layer"]


@pytest.mark.parametrize("pred", ["gate", "history"])
def test_decode_steps_replay_exactly(pred):
    """Prefill then D decode tokens with the cache persisting (pipeline.py:723-740);
    the whole session's decisions replay exactly through the oracle engine."""
    cfg = tiny_cfg(routing="live", predictor=pred, num_slabs=20)
    tr = small_trace(cfg, seed=21)
    stack = MoEStack(cfg)
    x, sal, mod, _ = request(tr, cfg.hidden, seed=4)
    res = stack.forward(x, sal, mod, record=True, keep_session=True)
    D = 3
    g = torch.Generator(device="cuda").manual_seed(9)
    steps = [stack.decode_step(torch.randn((1, cfg.hidden), generator=g, device="cuda").to(torch.bfloat16),
                               record=True) for _ in range(D)]
    rep = stack.end_session()
    T = tr.num_tokens
    re = np.zeros((cfg.layers, T + D, cfg.k), dtype=np.int64)
    re[:] = np.arange(cfg.k)
    re[: cfg.l_pinned, :T] = res.prefix_routes.cpu().numpy()
    for i, l in enumerate(range(cfg.l_pinned, cfg.layers)):
        re[l, res.retained] = res.routes[i].cpu().numpy()
    for s, st in enumerate(steps):
        for l in range(cfg.layers):
            re[l, T + s] = st.routes[l].cpu().numpy()[0]
    merged = RoutingTrace(cfg.layers, cfg.experts, cfg.k, re, np.full(re.shape, 1.0 / cfg.k),
                          np.r_[tr.saliency, np.ones(D)], np.r_[tr.modality, np.ones(D, np.uint8)],
                          np.r_[tr.embedding, np.zeros((D, tr.embed_dim))], phase_marks=list(range(T, T + D)))
    sd = _sim_dict(cfg)
    sd["decode_steps"] = D
    comp = dict(alpha=cfg.alpha, beta=cfg.beta, lam=cfg.lam, prefix=list(range(cfg.l_pinned)))
    y_over = None
    if pred == "gate":
        sd["predictor"]["kind"] = "history"

        def y_over(ctx, ids):
            ids = list(ids)
            if len(ids) == 1 and ids[0] >= T:
                return steps[ids[0] - T].scores[ctx]
            return res.scores[ctx]
    exp = harness.simulate(merged, sd, comp, False, y_override=y_over)
    got = rep.to_dict()
    for key in _F + ("decode_ms_per_step",):
        assert got[key] == exp[key], key
    assert got["per_layer"] == exp["per_layer"]
    assert sum(st.copies for st in steps) >= 0


def test_shared_experts_decisions_and_data_path():
    """C4-style layer with 2 always-resident shared experts: decisions equal
    simulate() with shared_experts=2 (pipeline.py:406,640-641) and the hidden
    states equal a hand-run of the same kernels with every expert resident."""
    from paper_2605_05899_b200 import kernels
    cfg = tiny_cfg(layers=6, experts=16, k=4, inter=512, l_pinned=2, num_slabs=40, routing="trace",
                   predictor="history", shared_experts=2)
    tr = generate_trace(TraceGenConfig(n_visual=300, n_text=20, layers=6, experts=16, k=4, cluster_support=6,
                                       visual_noise=0.3, seed=8, shared_experts=2))
    stack = MoEStack(cfg)
    x, sal, mod, dtr = request(tr, cfg.hidden, seed=6)
    res = stack.forward(x, sal, mod, trace=dtr)
    sim = cfg.sim_config()
    plan = build_plan(tr, sim, CompressionConfig(cfg.alpha, cfg.beta, cfg.lam, tuple(range(cfg.l_pinned))))
    rep = simulate(tr, plan, sim).to_dict()
    got = res.report.to_dict()
    for key in _F:
        assert got[key] == rep[key], key
    # hand-run with every routed expert resident
    st = stack.store
    E, S = cfg.experts, cfg.shared_experts
    full = torch.cat([st.pool[(l % st.host_layers) * E:(l % st.host_layers + 1) * E] for l in range(cfg.layers)])
    arena = torch.cat([full.cuda(), st.arena[st.shared_slot_of[0, 0]:]])  # routed slots 0..L*E-1, then shared
    shared0 = cfg.layers * E
    routes = dtr["routes"]
    gts = dtr["gates"]
    cur = x
    rows = torch.arange(tr.num_tokens, dtype=torch.int32, device="cuda")
    ret = torch.from_numpy(res.retained.astype(np.int32)).cuda()
    for l in range(cfg.layers):
        if l == cfg.l_pinned:
            cur = kernels.gather_rows(cur, ret)
            rows = ret
        N = int(cur.shape[0])
        xn = kernels.rmsnorm(cur)
        ids = routes[l].index_select(0, rows.long()).contiguous()
        gates = gts[l].index_select(0, rows.long()).contiguous()
        off, src, pos = kernels.permute_plan(ids, E)
        xp = kernels.permute_rows(xn, src, N * cfg.k)
        _, y = kernels.grouped_swiglu(xp, off, arena, torch.arange(l * E, (l + 1) * E, dtype=torch.int32,
                                                                   device="cuda"), cfg.inter)
        ssrc = torch.arange(N, dtype=torch.int32, device="cuda").repeat(S)
        soff = torch.tensor([s * N for s in range(S + 1)], dtype=torch.int32, device="cuda")
        xs = kernels.permute_rows(xn, ssrc, N * S)
        _, ys = kernels.grouped_swiglu(xs, soff, arena, torch.arange(shared0 + l * S, shared0 + (l + 1) * S,
                                                                     dtype=torch.int32, device="cuda"), cfg.inter)
        cur = kernels.combine_shared(y, pos, gates, cur, ys, S)
    torch.cuda.synchronize()
    assert torch.equal(res.hidden, cur)


def test_sharded_home_mode_bit_identical_to_host_pool_mode():
    """Misses served from the HBM home copies (sharded mode, world=1 -> local
    D2D pulls) give the same decisions and bit-identical hidden states as the
    pinned-host-pool mode."""
    from paper_2605_05899_b200.moe import ShardedHome
    cfg = tiny_cfg(routing="live", predictor="gate")
    store = ExpertStore(cfg, seed=3)
    tr = small_trace(cfg, seed=31)
    x, sal, mod, _ = request(tr, cfg.hidden, seed=5)
    a = MoEStack(cfg, store=store).forward(x, sal, mod)
    torch.cuda.synchronize()
    ha = a.hidden.clone()
    home = ShardedHome(store, 0, 1)
    b = MoEStack(cfg, store=store, home=home).forward(x, sal, mod)
    torch.cuda.synchronize()
    assert b.copies == a.copies > 0
    assert b.report.to_dict() == a.report.to_dict()
    assert torch.equal(b.hidden, ha)


def test_batched_split_path_bit_identical_to_all_resident_layers():
    """> 8192 retained rows: early decisions split each layer's combine/norm/route
    into two launches; the hidden states still equal a layer-by-layer run on
    resident experts bit for bit."""
    cfg = tiny_cfg(routing="live", predictor="history", num_slabs=24)
    store = ExpertStore(cfg, seed=9)
    trs = [small_trace(cfg, seed=s) for s in range(40, 84)]
    xs, sals, mods = [], [], []
    for i, tr in enumerate(trs):
        x, sal, mod, _ = request(tr, cfg.hidden, seed=100 + i)
        xs.append(x), sals.append(sal), mods.append(mod)
    offs = np.cumsum([0] + [t.num_tokens for t in trs]).tolist()
    x = torch.cat(xs)
    res = MoEStack(cfg, store=store).forward(x, torch.cat(sals), torch.cat(mods), req_off=offs)
    torch.cuda.synchronize()
    assert len(res.retained) >= 8192
    from paper_2605_05899_b200 import kernels
    from paper_2605_05899_b200.moe import moe_layer_forward
    E = cfg.experts
    arena = torch.stack([store.pool[(l % store.host_layers) * E + e] for l in range(cfg.layers) for e in range(E)]).cuda()
    cur = x
    for l in range(cfg.layers):
        if l == cfg.l_pinned:
            cur = kernels.gather_rows(cur, torch.from_numpy(res.retained.astype(np.int32)).cuda())
        xn = kernels.rmsnorm(cur)
        ids, gates, _ = kernels.route_topk(xn, store.router[l], cfg.k)
        cur = moe_layer_forward(cur, ids, gates, arena, torch.arange(l * E, (l + 1) * E, dtype=torch.int32,
                                                                      device="cuda"), cfg.inter, E, xn=xn)
    torch.cuda.synchronize()
    assert torch.equal(res.hidden, cur)


def test_chunked_prefix_as_rows_land_is_bit_identical():
    """forward(x_ready=...): the pinned prefix runs chunk by chunk as the rows
    arrive from a side-stream H2D; outputs and decisions equal the one-shot run."""
    cfg = tiny_cfg(routing="live", predictor="gate")
    store = ExpertStore(cfg, seed=3)
    trs = [small_trace(cfg, seed=s) for s in range(60, 66)]
    xs, sals, mods = [], [], []
    for i, tr in enumerate(trs):
        x, sal, mod, _ = request(tr, cfg.hidden, seed=200 + i)
        xs.append(x), sals.append(sal), mods.append(mod)
    offs = np.cumsum([0] + [t.num_tokens for t in trs]).tolist()
    x = torch.cat(xs)
    sal, mod = torch.cat(sals), torch.cat(mods)
    a = MoEStack(cfg, store=store).forward(x, sal, mod, req_off=offs)
    ha, reta, repa = a.hidden.clone(), a.retained.copy(), a.report.to_dict()
    x_h = x.cpu().pin_memory()
    x_dev = torch.empty_like(x)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    ready, r0 = [], 0
    with torch.cuda.stream(side):
        for r1 in (offs[2], offs[4], offs[6]):
            x_dev[r0:r1].copy_(x_h[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            ready.append((r1, ev))
            r0 = r1
    b = MoEStack(cfg, store=store).forward(x_dev, sal, mod, req_off=offs, x_ready=ready)
    torch.cuda.synchronize()
    assert np.array_equal(reta, b.retained)
    assert torch.equal(ha, b.hidden)
    assert b.report.to_dict() == repa


@pytest.mark.parametrize("routing,pred", [("live", "history"), ("trace", "oracle"), ("trace", "history")])
def test_decode_step_hidden_matches_resident_layers(routing, pred):
    """Decode tokens through the cached executor (skinny FFN, one-launch decode glue
    on trace routing) give bit-identically the hidden state of the same layers run
    on resident experts with the plain kernels (rmsnorm, route/trace ids, permute,
    grouped SwiGLU, combine)."""
    from paper_2605_05899_b200 import kernels
    from paper_2605_05899_b200.moe import moe_layer_forward

    cfg = tiny_cfg(routing=routing, predictor=pred, num_slabs=20)
    D = 2
    tr = generate_trace(TraceGenConfig(n_visual=576, n_text=64, layers=cfg.layers, experts=cfg.experts, k=cfg.k,
                                       cluster_support=4, visual_noise=0.3, seed=31, decode_steps=D))
    T = tr.num_tokens - D
    stack = MoEStack(cfg)
    x, sal, mod, dtr = request(tr, cfg.hidden, seed=4)
    stack.forward(x[:T], sal[:T], mod[:T], trace=dtr if routing == "trace" else None, keep_session=True)
    store, E = stack.store, cfg.experts
    arena = torch.stack([store.pool[(l % store.host_layers) * E + e] for l in range(cfg.layers)
                         for e in range(E)]).cuda()
    g = torch.Generator(device="cuda").manual_seed(9)
    for s in range(D):
        xt = torch.randn((1, cfg.hidden), generator=g, device="cuda").to(torch.bfloat16)
        r = stack.decode_step(xt, tok=T + s if routing == "trace" else None)
        cur = xt
        for l in range(cfg.layers):
            xn = kernels.rmsnorm(cur)
            if routing == "trace":
                ids = dtr["routes"][l, T + s].view(1, -1).contiguous()
                gates = dtr["gates"][l, T + s].view(1, -1).contiguous()
            else:
                ids, gates, _ = kernels.route_topk(xn, store.router[l], cfg.k)
            cur = moe_layer_forward(cur, ids, gates, arena, torch.arange(l * E, (l + 1) * E, dtype=torch.int32,
                                                                          device="cuda"), cfg.inter, E, xn=xn)
        torch.cuda.synchronize()
        assert torch.equal(r.hidden, cur), (routing, pred, s)
    stack.end_session()


@pytest.mark.parametrize("routing", ["trace", "live"])
def test_mlp_predictor_in_the_stack(routing):
    """predictor="mlp" (predictor.py:521-550) inside MoEStack: every emission's scores
    equal the MLP predictor evaluated on the routes the run used (rtol 1e-12: the
    reference's BLAS order is not bit-reproducible), and the whole
    decision stream replays exactly through the oracle engine with those scores."""
    from paper_2605_05899_b200 import CompressionConfig, MLPPredictor, compress
    from paper_2605_05899_b200.predictor import MLPModel

    cfg = tiny_cfg(routing=routing, predictor="mlp")
    tr = small_trace(cfg, seed=41)
    D = tr.embed_dim
    rng = np.random.default_rng(3)
    d_in, E = cfg.experts + 2 * D, cfg.experts

    def uni(r, c):
        return rng.uniform(-1 / np.sqrt(c), 1 / np.sqrt(c), size=(r, c))
    model = MLPModel(uni(32, d_in), np.zeros(32), uni(16, 32), np.zeros(16), uni(E, 16), np.zeros(E))
    stack = MoEStack(cfg, mlp_model=model)
    x, sal, mod, dtr = request(tr, cfg.hidden, seed=7)
    emb = torch.from_numpy(np.ascontiguousarray(tr.embedding)).cuda()
    res = stack.forward(x, sal, mod, trace=dtr if routing == "trace" else None, record=True, embeddings=emb)
    tr_run = tr if routing == "trace" else _trace_from_run(cfg, tr, res)
    plan = compress(tr_run, CompressionConfig(cfg.alpha, cfg.beta, cfg.lam, tuple(range(cfg.l_pinned))))
    ret = plan.retained_ids(tr_run)
    assert res.retained.tolist() == ret
    pred = MLPPredictor(model, tr_run, plan, cfg.history_decay)
    assert len(res.scores) >= cfg.layers - cfg.l_pinned
    for ctx, y in res.scores.items():
        np.testing.assert_allclose(y, pred.priorities(ctx, ret), rtol=1e-12, atol=0)
    sd = _sim_dict(cfg)
    sd["predictor"]["kind"] = "history"  # placeholder kind; scores come from y_override
    comp = dict(alpha=cfg.alpha, beta=cfg.beta, lam=cfg.lam, prefix=list(range(cfg.l_pinned)))
    exp = harness.simulate(tr_run, sd, comp, False, y_override=lambda ctx, ids: res.scores[ctx])
    got = res.report.to_dict()
    for key in _F:
        assert got[key] == exp[key], key
    assert got["per_layer"] == exp["per_layer"]
