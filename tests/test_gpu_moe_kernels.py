"""Router, permutation, grouped SwiGLU (tcgen05) and combine vs the torch oracle.

Tolerances (stated): routed ids exact on exact-arithmetic inputs;
gates |d| <= 1e-6; FFN bf16 outputs assert_close(rtol=2e-2, atol=2e-2) plus
relative Frobenius error <= 5e-3 against the fp32 restatement.
"""
import numpy as np
import pytest
import torch

from oracle import moe_ref
from paper_2605_05899_b200 import kernels

pytestmark = pytest.mark.gpu


def test_router_exact_ids_on_integer_inputs_with_ties():
    g = torch.Generator().manual_seed(1)
    for N, H, E, k in ((2368, 2048, 128, 8), (333, 256, 8, 2), (100, 2560, 4, 2), (64, 2048, 64, 6)):
        x = torch.randint(-4, 5, (N, H), generator=g).to(torch.bfloat16)
        w = torch.randint(-1, 2, (E, H), generator=g).to(torch.bfloat16)
        counts = torch.zeros(E, dtype=torch.int32, device="cuda")
        ids, gates, logits = kernels.route_topk(x.cuda(), w.cuda(), k, counts=counts, want_logits=True)
        rid, rg, rl = moe_ref.route(x, w, k)
        assert torch.equal(logits.cpu().double(), rl)
        assert torch.equal(ids.cpu(), rid)
        assert (gates.cpu() - rg).abs().max().item() <= 1e-6
        assert torch.equal(counts.cpu().long(), torch.bincount(rid.reshape(-1).long(), minlength=E))


def test_router_realistic_inputs_margin_aware():
    g = torch.Generator().manual_seed(2)
    x = torch.randn(1216, 2048, generator=g).to(torch.bfloat16)
    w = (torch.randn(128, 2048, generator=g) / 45).to(torch.bfloat16)
    ids, gates, _ = kernels.route_topk(x.cuda(), w.cuda(), 8)
    rid, rg, rl = moe_ref.route(x, w, 8)
    srt = torch.sort(rl, dim=1, descending=True).values
    safe = (srt[:, 7] - srt[:, 8]) > 1e-3  # margin-safe tokens must agree exactly
    assert torch.equal(ids.cpu()[safe], rid[safe])
    assert safe.float().mean() > 0.9
    torch.testing.assert_close(gates.cpu()[safe], rg[safe], rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("N,k,E", [(1216, 8, 128), (1000, 8, 128), (155648, 8, 128), (30000, 6, 64), (5000, 2, 4),
                                   (3000, 8, 256), (4097, 1, 16)])
def test_permute_plan_is_stable_counting_sort(N, k, E):
    """Single-CTA (<= 8192 picks) and multi-CTA (count / scan / scatter) paths."""
    g = torch.Generator().manual_seed(3 + N)
    # skewed, distinct ids per token (some experts empty at small E... all ids drawn from a biased order)
    logits = torch.randn(N, E, generator=g) + torch.linspace(2, -2, E)
    ids = torch.topk(logits, k, dim=1).indices.int()
    off, src, pos = kernels.permute_plan(ids.cuda(), E)
    roff, rsrc, rpos = moe_ref.permute(ids, E)
    assert torch.equal(off.cpu().long(), roff)
    assert torch.equal(src.cpu().long()[: N * k], rsrc)
    assert torch.equal(pos.cpu().long()[: N * k].reshape(N, k), rpos)
    # fused plan + row copy
    H = 2560 if E == 4 else 256
    x = torch.randn(N, H, device="cuda").to(torch.bfloat16)
    off2, src2, pos2, xp2 = kernels.permute(ids.cuda(), x, E)
    assert torch.equal(off2, off) and torch.equal(src2, src) and torch.equal(pos2, pos)
    assert torch.equal(xp2, x[rsrc.cuda()])


def _expert_setup(N, H, I, E, k, n_slots, seed):
    g = torch.Generator().manual_seed(seed)
    x = (torch.randn(N, H, generator=g)).to(torch.bfloat16)
    wg = (torch.randn(n_slots, I, H, generator=g) / H ** 0.5).to(torch.bfloat16)
    wu = (torch.randn(n_slots, I, H, generator=g) / H ** 0.5).to(torch.bfloat16)
    wd = (torch.randn(n_slots, H, I, generator=g) / I ** 0.5).to(torch.bfloat16)
    arena = torch.stack([kernels.pack_expert(wg[s], wu[s], wd[s]) for s in range(n_slots)])
    # skewed routing: some experts empty, some with > 128 rows
    logits = torch.randn(N, E, generator=g) + torch.linspace(3, -3, E)
    ids = torch.topk(logits, k, dim=1).indices.int()
    slot_of = torch.randperm(n_slots, generator=g)[:E].int()
    return x, wg, wu, wd, arena, ids, slot_of


@pytest.mark.parametrize("simt", [False, True])
@pytest.mark.parametrize("shape", [(1216, 2048, 768, 128, 8), (300, 256, 512, 8, 2), (640, 2048, 1408, 64, 6)])
def test_grouped_swiglu_matches_fp32_restatement(shape, simt):
    N, H, I, E, k = shape
    n_slots = E + 3
    x, wg, wu, wd, arena, ids, slot_of = _expert_setup(N, H, I, E, k, n_slots, seed=N + E)
    off, src, pos = kernels.permute_plan(ids.cuda(), E)
    M = N * k
    xp = kernels.permute_rows(x.cuda(), src, M)
    h1, y = kernels.grouped_swiglu(xp, off, arena.cuda(), slot_of.cuda(), I, simt=simt)
    torch.cuda.synchronize()
    roff, rsrc, rpos = moe_ref.permute(ids, E)
    xr = x[rsrc]
    assert torch.equal(xp.cpu(), xr)
    h_exp = torch.empty(M, I, dtype=torch.bfloat16)
    y_exp = torch.empty(M, H, dtype=torch.bfloat16)
    for e in range(E):
        a, b = int(roff[e]), int(roff[e + 1])
        if b > a:
            s = int(slot_of[e])
            h_exp[a:b], y_exp[a:b] = moe_ref.expert_ffn(xr[a:b], wg[s], wu[s], wd[s])
    torch.testing.assert_close(h1.cpu().float(), h_exp.float(), rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(y.cpu().float(), y_exp.float(), rtol=2e-2, atol=2e-2)
    rel = (y.cpu().float() - y_exp.float()).norm() / y_exp.float().norm()
    assert rel.item() <= 5e-3
    # combine back to token order with residual
    gates = torch.softmax(torch.randn(N, k), dim=1)
    out = kernels.combine(y, pos, gates.cuda(), x.cuda())
    ref = moe_ref.combine(y.cpu(), rpos, gates, x)
    torch.testing.assert_close(out.cpu().float(), ref.float(), rtol=2e-2, atol=2e-2)


def test_fused_route_and_lookahead_exact_on_integer_inputs():
    g = torch.Generator().manual_seed(9)
    L, N, H, E, k = 4, 1216, 2048, 128, 8
    x = torch.randint(-4, 5, (N, H), generator=g).to(torch.bfloat16)
    router = torch.randint(-1, 2, (L, E, H), generator=g).to(torch.bfloat16)
    for layer in (0, 2):
        counts = torch.zeros(E, dtype=torch.int32, device="cuda")
        la = torch.zeros(E, dtype=torch.int32, device="cuda")
        ids, gates = kernels.route_lookahead(x.cuda(), router.cuda(), layer, k, counts, la)
        rid, rg, _ = moe_ref.route(x, router[layer], k)
        assert torch.equal(ids.cpu(), rid)
        assert (gates.cpu() - rg).abs().max().item() <= 1e-6
        nid, _, _ = moe_ref.route(x, router[layer + 1], k)
        assert torch.equal(la.cpu().long(), torch.bincount(nid.reshape(-1).long(), minlength=E))
        assert torch.equal(counts.cpu().long(), torch.bincount(rid.reshape(-1).long(), minlength=E))


@pytest.mark.parametrize("N,E,k", [(130, 128, 8), (1216, 128, 8), (2368, 64, 6), (4000, 128, 8), (700, 16, 2)])
def test_split_k_router_exact_on_integer_inputs(N, E, k):
    """Few row tiles: the cluster split-K router (partials over K summed across the
    cluster in rank order).  Integer inputs keep every partial sum exact, so logits,
    ids, gates and both count vectors must equal the restatement exactly."""
    g = torch.Generator().manual_seed(N + E)
    L, H = 3, 2048
    x = torch.randint(-4, 5, (N, H), generator=g).to(torch.bfloat16)
    router = torch.randint(-1, 2, (L, E, H), generator=g).to(torch.bfloat16)
    counts = torch.zeros(E, dtype=torch.int32, device="cuda")
    ids, gates, logits = kernels.route_topk(x.cuda(), router[0].cuda(), k, counts=counts, want_logits=True)
    rid, rg, rl = moe_ref.route(x, router[0], k)
    assert torch.equal(logits.cpu().double(), rl)
    assert torch.equal(ids.cpu(), rid)
    assert (gates.cpu() - rg).abs().max().item() <= 1e-6
    assert torch.equal(counts.cpu().long(), torch.bincount(rid.reshape(-1).long(), minlength=E))
    if E % 16 == 0:
        c2 = torch.zeros(E, dtype=torch.int32, device="cuda")
        la = torch.zeros(E, dtype=torch.int32, device="cuda")
        ids2, gates2 = kernels.route_lookahead(x.cuda(), router.cuda(), 1, k, c2, la)
        rid1, rg1, _ = moe_ref.route(x, router[1], k)
        nid, _, _ = moe_ref.route(x, router[2], k)
        assert torch.equal(ids2.cpu(), rid1)
        assert (gates2.cpu() - rg1).abs().max().item() <= 1e-6
        assert torch.equal(la.cpu().long(), torch.bincount(nid.reshape(-1).long(), minlength=E))
        assert torch.equal(c2.cpu().long(), torch.bincount(rid1.reshape(-1).long(), minlength=E))


@pytest.mark.parametrize("N,chunks", [(9728, (1216,)), (18944, (9472,)), (2432, (1216,)), (40, (12,)),
                                      (75776 * 2, (75776,))])
def test_router_chunks_bit_identical_to_one_launch(N, chunks):
    """Batch invariance of the chunked router (vmm_route_topk_ex): the executor
    routes a layer's first chunk early (decisions) and the two-stream prefix
    routes request-aligned halves; with the batch's row count as the split hint
    each chunk's ids/gates/counts equal one launch over the whole batch, bit for
    bit, on N(0,1) inputs (real-valued logits, so a different K-split order would
    show in the gates).  Chunk sizes are the R=8 headline layer (1216 of 9728),
    the R=8 prefix halves, R=2, a chunk below the decode-sized kernel's 16 rows
    and the R=64 prefix halves."""
    g = torch.Generator(device="cuda").manual_seed(N)
    L, H, E, k = 3, 2048, 128, 8
    x = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
    router = (torch.randn(L, E, H, device="cuda", generator=g) / 45).to(torch.bfloat16)
    bounds = [0, *chunks, N]
    c_one = torch.zeros(E, dtype=torch.int32, device="cuda")
    ids1, g1, _ = kernels.route_topk(x, router[0], k, counts=c_one)
    ids2 = torch.empty_like(ids1)
    g2 = torch.empty_like(g1)
    c_ch = torch.zeros(E, dtype=torch.int32, device="cuda")
    for a, b in zip(bounds[:-1], bounds[1:]):
        kernels.route_topk(x[a:b], router[0], k, counts=c_ch, ids=ids2[a:b], gates=g2[a:b], batch_rows=N)
    assert torch.equal(ids1, ids2) and torch.equal(g1, g2) and torch.equal(c_one, c_ch)
    c1, la1 = (torch.zeros(E, dtype=torch.int32, device="cuda") for _ in range(2))
    ids3, g3 = kernels.route_lookahead(x, router, 0, k, c1, la1)
    assert torch.equal(ids3, ids1) and torch.equal(g3, g1)  # the fused lookahead's router columns too
    c2, la2 = (torch.zeros(E, dtype=torch.int32, device="cuda") for _ in range(2))
    ids4, g4 = torch.empty_like(ids1), torch.empty_like(g1)
    for a, b in zip(bounds[:-1], bounds[1:]):
        kernels.route_lookahead(x[a:b], router, 0, k, c2, la2, ids=ids4[a:b], gates=g4[a:b], batch_rows=N)
    assert torch.equal(ids4, ids1) and torch.equal(g4, g1) and torch.equal(la1, la2) and torch.equal(c1, c2)


@pytest.mark.parametrize("N", [1, 5, 32])
def test_skinny_router_decode_sizes_exact(N):
    g = torch.Generator().manual_seed(N)
    L, H, E, k = 3, 2048, 128, 8
    x = torch.randint(-4, 5, (N, H), generator=g).to(torch.bfloat16)
    router = torch.randint(-1, 2, (L, E, H), generator=g).to(torch.bfloat16)
    counts = torch.zeros(E, dtype=torch.int32, device="cuda")
    ids, gates, logits = kernels.route_topk(x.cuda(), router[1].cuda(), k, counts=counts, want_logits=True)
    rid, rg, rl = moe_ref.route(x, router[1], k)
    assert torch.equal(logits.cpu().double(), rl)
    assert torch.equal(ids.cpu(), rid)
    assert (gates.cpu() - rg).abs().max().item() <= 1e-6
    c2 = torch.zeros(E, dtype=torch.int32, device="cuda")
    la = torch.zeros(E, dtype=torch.int32, device="cuda")
    ids2, _ = kernels.route_lookahead(x.cuda(), router.cuda(), 1, k, c2, la)
    assert torch.equal(ids2.cpu(), rid)
    nid, _, _ = moe_ref.route(x, router[2], k)
    assert torch.equal(la.cpu().long(), torch.bincount(nid.reshape(-1).long(), minlength=E))


@pytest.mark.parametrize("shape", [(1, 2048, 768, 128, 8), (2, 2048, 768, 128, 8), (2, 1024, 512, 16, 8),
                                   (2, 2048, 1408, 64, 6), (1, 2560, 10240, 4, 2)])
def test_decode_sized_swiglu_matches_fp32_restatement(shape):
    """M_total <= 16 rows takes the weight-streaming CUDA-core path."""
    _check_swiglu(shape)


@pytest.mark.parametrize("shape", [(1, 2048, 768, 128, 8), (2, 2048, 768, 128, 8), (2, 1024, 512, 16, 8),
                                   (1, 2048, 1408, 64, 6)])
def test_decode_sized_tensor_core_swiglu_matches_fp32_restatement(shape, monkeypatch):
    """Opt-in swap-AB tcgen05 decode FFN (TMA weight ring, per-expert H1 counters)."""
    monkeypatch.setenv("VMM_DECODE_TC", "1")
    _check_swiglu(shape)


def _check_swiglu(shape):
    N, H, I, E, k = shape
    n_slots = E + 3
    x, wg, wu, wd, arena, ids, slot_of = _expert_setup(N, H, I, E, k, n_slots, seed=N + E + 7)
    off, src, pos = kernels.permute_plan(ids.cuda(), E)
    M = N * k
    xp = kernels.permute_rows(x.cuda(), src, M)
    h1, y = kernels.grouped_swiglu(xp, off, arena.cuda(), slot_of.cuda(), I)
    roff, rsrc, rpos = moe_ref.permute(ids, E)
    xr = x[rsrc]
    y_exp = torch.empty(M, H, dtype=torch.bfloat16)
    for e in range(E):
        a, b = int(roff[e]), int(roff[e + 1])
        if b > a:
            s = int(slot_of[e])
            _, y_exp[a:b] = moe_ref.expert_ffn(xr[a:b], wg[s], wu[s], wd[s])
    torch.testing.assert_close(y.cpu().float(), y_exp.float(), rtol=2e-2, atol=2e-2)
    rel = (y.cpu().float() - y_exp.float()).norm() / y_exp.float().norm()
    assert rel.item() <= 5e-3


def test_fused_combine_norm_bit_identical_to_combine_then_rmsnorm():
    g = torch.Generator().manual_seed(4)
    N, k, H, S = 300, 6, 2048, 2
    y = torch.randn(N * k, H, generator=g).to(torch.bfloat16).cuda()
    ys = torch.randn(N * S, H, generator=g).to(torch.bfloat16).cuda()
    pos = torch.randperm(N * k, generator=g).int().reshape(N, k).cuda()
    gates = torch.softmax(torch.randn(N, k, generator=g), 1).cuda()
    resid = torch.randn(N, H, generator=g).to(torch.bfloat16).cuda()
    for shared in (0, S):
        ref = kernels.combine_shared(y, pos, gates, resid, ys, shared) if shared else kernels.combine(y, pos, gates, resid)
        refn = kernels.rmsnorm(ref)
        out = torch.empty_like(resid)
        xn = torch.empty_like(resid)
        from paper_2605_05899_b200 import _lib
        _lib.check(_lib.lib().vmm_combine_norm(y.data_ptr(), pos.data_ptr(), gates.data_ptr(), resid.data_ptr(), N, k,
                                               H, ys.data_ptr() if shared else None, shared, 1e-6, out.data_ptr(),
                                               xn.data_ptr(), torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        assert torch.equal(xn, refn)


@pytest.mark.parametrize("N,k,E", [(1, 8, 128), (2, 8, 128), (4, 6, 64), (1, 2, 4), (16, 2, 8), (200, 8, 128)])
def test_permute_plan_small_batches(N, k, E):
    g = torch.Generator().manual_seed(N * 100 + k)
    ids = torch.stack([torch.randperm(E, generator=g)[:k] for _ in range(N)]).int()
    off, src, pos = kernels.permute_plan(ids.cuda(), E)
    roff, rsrc, rpos = moe_ref.permute(ids, E)
    assert torch.equal(off.cpu().long(), roff)
    assert torch.equal(src.cpu().long()[: N * k], rsrc)
    assert torch.equal(pos.cpu().long()[: N * k].reshape(N, k), rpos)
    # the fused plan + row copy writes every permuted row (also for <= 32 picks)
    x = torch.randn(N, 64, device="cuda").to(torch.bfloat16)
    _, src2, _, xp = kernels.permute(ids.cuda(), x, E)
    assert torch.equal(xp, x[src2[: N * k].long()])


@pytest.mark.parametrize("shape", [(1216, 2048, 768, 128, 8), (300, 256, 512, 8, 2), (640, 2048, 1408, 64, 6),
                                   (9728, 2048, 768, 128, 8), (3, 2048, 768, 128, 8), (40000, 2048, 768, 128, 8),
                                   (9000, 2048, 1408, 64, 6), (2000, 256, 512, 256, 8), (70000, 256, 512, 256, 8)])
def test_fused_ffn_bit_identical_to_two_launches(shape):
    """The one-launch persistent FFN (GEMM2 tiles gated on H1 block counters;
    CTA-pair 256x256 tiles once experts average >= 256 rows) computes every
    tile exactly like the two-launch path."""
    N, H, I, E, k = shape
    n_slots = E + 3
    x, wg, wu, wd, arena, ids, slot_of = _expert_setup(N, H, I, E, k, n_slots, seed=N + 2 * E)
    off, src, pos = kernels.permute_plan(ids.cuda(), E)
    xp = kernels.permute_rows(x.cuda(), src, N * k)
    arena, slot_of = arena.cuda(), slot_of.cuda()
    h1a, ya = kernels.grouped_swiglu(xp, off, arena, slot_of, I, fused=False)
    with kernels.keep_h1():  # H1 is scratch: kept here so the GEMM1 tiles are compared too
        h1b, yb = kernels.grouped_swiglu(xp, off, arena, slot_of, I, fused=True)
        # A rows gathered from the token rows by TMA gather4 (no permuted copy)
        h1c, yc = kernels.grouped_swiglu(N * k, off, arena, slot_of, I, x_rows=x.cuda(), src_row=src)
    # the product path: consumed H1 rows dropped from L2 without write-back (CTA-pair tiles)
    _, yd = kernels.grouped_swiglu(xp, off, arena, slot_of, I, fused=True)
    # any expert walk order (the executor's largest-first order on the CTA-pair path)
    perm = torch.randperm(E, generator=torch.Generator().manual_seed(N)).int().cuda()
    _, ye = kernels.grouped_swiglu(xp, off, arena, slot_of, I, fused=True, order=perm)
    torch.cuda.synchronize()
    assert torch.equal(ya, ye)
    assert torch.equal(h1a, h1b)
    assert torch.equal(ya, yb)
    assert torch.equal(h1a, h1c)
    assert torch.equal(ya, yc)
    assert torch.equal(ya, yd)


@pytest.mark.parametrize("N", [1, 2, 1216, 5000])
def test_fused_ffn_waits_for_copy_stream_fills(N):
    """Copy overlap: the FFN is launched BEFORE its experts' weights are copied
    in; each expert's tiles wait on the copy stream's ready flag.  The result
    must equal the all-resident computation bit for bit (N=1, 2: the persistent
    decode kernel; N=1216: single-CTA 128x256 tiles; N=5000: CTA-pair 256x256)."""
    import ctypes as C

    from paper_2605_05899_b200 import _lib

    H, I, E, k = 2048, 768, 128, 8
    x, wg, wu, wd, arena, ids, slot_of = _expert_setup(N, H, I, E, k, E, seed=77)
    slot_of = torch.arange(E, dtype=torch.int32)  # expert e -> slab e
    pool = arena.pin_memory()
    L = _lib.lib()
    xf = C.c_void_p()
    _lib.check(L.vmm_xfer_create(E, arena.shape[1] * 2, 1, C.byref(xf)))
    try:
        ready = L.vmm_xfer_ready(xf)
        assert ready
        off, src, pos = kernels.permute_plan(ids.cuda(), E)
        xp = kernels.permute_rows(x.cuda(), src, N * k)
        dev_arena = torch.zeros_like(arena, device="cuda")
        torch.cuda.synchronize()
        need = torch.arange(1, E + 1, dtype=torch.int32, device="cuda")  # fill e is the (e+1)-th copy
        ready_t = torch.empty(0)  # placeholder; pass the raw pointer below
        h1 = torch.empty(N * k, I, dtype=torch.bfloat16, device="cuda")
        y = torch.empty(N * k, H, dtype=torch.bfloat16, device="cuda")
        done = torch.empty(N * k // 128 + E + 1, dtype=torch.int32, device="cuda")
        w2 = dev_arena.data_ptr() + 2 * I * H * 2
        _lib.check(L.vmm_ffn_keep_h1(int(N <= 1216)))  # N=5000 (CTA pairs) runs the product's H1 discard
        _lib.check(L.vmm_grouped_swiglu_fused(xp.data_ptr(), off.data_ptr(), E, N * k, H, I, dev_arena.data_ptr(),
                                              w2, 3 * I * H, E, slot_of.cuda().data_ptr(), need.data_ptr(), ready, 0,
                                              done.data_ptr(), None, None, 0, h1.data_ptr(), y.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream))
        del ready_t
        nbytes = arena.shape[1] * 2
        for e in range(E):  # the copies are issued only now, while the FFN kernel already runs
            _lib.check(L.vmm_xfer_copy(xf, e, pool[e].data_ptr(), dev_arena[e].data_ptr(), nbytes, 0))
        torch.cuda.synchronize()
        _lib.check(L.vmm_xfer_sync(xf))
        h1r, yr = kernels.grouped_swiglu(xp, off, dev_arena, slot_of.cuda(), I, fused=False)
        torch.cuda.synchronize()
        assert torch.equal(dev_arena.cpu(), arena)
        if N <= 1216:
            assert torch.equal(h1, h1r)
        assert torch.equal(y, yr)
    finally:
        L.vmm_ffn_keep_h1(0)
        L.vmm_xfer_destroy(xf)


@pytest.mark.parametrize("n,k,E,H,with_y", [(1, 8, 128, 2048, True), (2, 8, 128, 2048, True), (1, 8, 128, 2048, False),
                                             (2, 2, 8, 256, True), (4, 4, 64, 2560, True)])
def test_decode_glue_bit_identical_to_separate_kernels(n, k, E, H, with_y):
    """vmm_decode_glue == combine -> rmsnorm -> trace gathers -> permute (plan + row copy)."""
    g = torch.Generator(device="cuda").manual_seed(n * 100 + k)
    T_tr = 50
    tr = torch.stack([torch.randperm(E, generator=torch.Generator().manual_seed(i))[:k] for i in range(T_tr)]) \
        .to(torch.int32).cuda()
    tg = torch.rand(T_tr, k, generator=g, device="cuda")
    rows = torch.tensor([7, 31, 2, 44][:n], dtype=torch.int32, device="cuda")
    resid = torch.randn(n, H, generator=g, device="cuda").to(torch.bfloat16)
    M = n * k
    y = torch.randn(M, H, generator=g, device="cuda").to(torch.bfloat16)
    pos_prev = torch.randperm(M, generator=torch.Generator().manual_seed(3)).to(torch.int32).cuda().view(n, k)
    gates_prev = torch.rand(n, k, generator=g, device="cuda")
    # separate kernels
    if with_y:
        out_ref = kernels.combine(y, pos_prev, gates_prev, resid)
    else:
        out_ref = resid
    xn_ref = kernels.rmsnorm(out_ref)
    ids_ref = tr[rows.long()].contiguous()
    gates_ref = tg[rows.long()].contiguous()
    off_ref, src_ref, pos_ref, xp_ref = kernels.permute(ids_ref, xn_ref, E)
    # one launch (pos/gates of the previous layer are overwritten in place, as in the executor)
    out, xn, ids, gates, off, src, pos, xp = kernels.decode_glue(y if with_y else None, pos_prev.clone(),
                                                                 gates_prev.clone(), resid, tr, tg, rows, E)
    if with_y:
        assert torch.equal(out, out_ref)
    assert torch.equal(xn, xn_ref)
    assert torch.equal(ids, ids_ref) and torch.equal(gates, gates_ref)
    assert torch.equal(off, off_ref[: E + 1]) and torch.equal(src, src_ref[:M]) and torch.equal(pos, pos_ref[:M])
    assert torch.equal(xp, xp_ref)


def test_refill_of_a_slab_lands_last_across_copy_streams():
    """Fills alternate over two copy streams; a slab filled twice with no reader in
    between (evict + refill) must end with the second fill's bytes (write-after-write)."""
    import ctypes as C

    from paper_2605_05899_b200 import _lib

    L = _lib.lib()
    nbytes = 64 << 20
    a = torch.full((nbytes,), 1, dtype=torch.uint8).pin_memory()
    b = torch.full((nbytes,), 2, dtype=torch.uint8).pin_memory()
    dst = torch.zeros(2, nbytes, dtype=torch.uint8, device="cuda")
    xf = C.c_void_p()
    _lib.check(L.vmm_xfer_create(2, nbytes, 1, C.byref(xf)))
    try:
        for i in range(4):
            # fill 2k+1 -> stream 0 (slab 0, bytes of a), fill 2k+2 -> stream 1 (slab 0 again, bytes of b)
            _lib.check(L.vmm_xfer_copy(xf, 0, a.data_ptr(), dst[0].data_ptr(), nbytes, 0))
            _lib.check(L.vmm_xfer_copy(xf, 0, b.data_ptr(), dst[0].data_ptr(), nbytes, 0))
            _lib.check(L.vmm_xfer_sync(xf))
            assert int(dst[0].min()) == 2 and int(dst[0].max()) == 2
            # the slab's ready flag ends at the LAST fill's sequence (never moves backwards)
            flags = torch.zeros(2, dtype=torch.int32, device="cuda")
            _lib.check(L.vmm_copy_async(flags.data_ptr(), L.vmm_xfer_ready(xf), 8,
                                        torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            assert int(flags[0]) == 2 * i + 2, (int(flags[0]), 2 * i + 2)
            dst.zero_()
            torch.cuda.synchronize()
    finally:
        L.vmm_xfer_destroy(xf)
