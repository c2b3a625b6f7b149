"""The G > 1 data path on one GPU: G contexts (ranks) with the external
transport, the two exchanges done by host-ordered device copies between the
contexts' layout buffers (all on one stream: no kernel ever waits on another).
Every rank-dependent index — per-destination send blocks, the
[source rank][segment][worker] receive layout, owner-side merge/sum, the
all-gather placement, decode of the local workers — runs on the real kernels
and must reproduce the single-context round bit for bit (fixed M, any G:
SURVEY §8e consistency requirement)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2204_06787_b200 as mb  # noqa: E402

DEV = "cuda:0"
ETA = 2.0 ** -10


def raw(ptr, nbytes):
    """uint8 view of library-owned device memory."""
    class _H:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_H(), device=DEV)


def run_ranks(ctxs, G, ml, t, period, seed, grads, comps, dense_mean=None):
    """One round on G emulated ranks; returns full_precision."""
    full = False
    for phase in range(3):
        for r, ctx in enumerate(ctxs):
            loc = slice(r * ml, (r + 1) * ml)
            full = ctx.round_phase(phase, t, period, ETA, seed, grads[loc], comps[loc],
                                   update=dense_mean[r] if dense_mean is not None else None)
        dense = full
        if phase == 0:  # exchange: block q of rank r's send -> block r of rank q's recv
            lays = [c.exchange_layout(dense) for c in ctxs]
            B = lays[0].block_bytes
            sends = [raw(l.send, B * G) for l in lays]
            recvs = [raw(l.recv, B * G) for l in lays]
            for r in range(G):
                for q in range(G):
                    recvs[q][r * B:(r + 1) * B].copy_(sends[r][q * B:(q + 1) * B])
        elif phase == 1:  # all-gather of the owned blocks
            lays = [c.exchange_layout(dense) for c in ctxs]
            B = lays[0].gather_block_bytes
            gath = [raw(l.gather, B * G) for l in lays]
            for r in range(G):
                for q in range(G):
                    if q != r:
                        gath[q][r * B:(r + 1) * B].copy_(gath[r][r * B:(r + 1) * B])
    return full


@pytest.mark.parametrize("topo,a,b,G,D", [
    ("ring", 8, 0, 2, 100_003),
    ("ring", 8, 0, 4, 65_536 * 3),
    ("ring", 8, 0, 8, 25_601),
    ("torus", 2, 4, 2, 60_211),
    ("torus", 2, 4, 8, 60_211),
    ("ring", 4, 0, 4, 1_000_000),
])
def test_emulated_ranks_match_single_context(topo, a, b, G, D):
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    W = sched.workers
    ml = W // G
    seed, period = 2026, 3
    single = mb.Context(D, sched, torch.float32, 0)
    ctxs = [mb.Context(D, sched, torch.float32, 0, nranks=G, rank=r, external_transport=True)
            for r in range(G)]
    assert [c.first_worker for c in ctxs] == [r * ml for r in range(G)]
    comp_1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    comp_g = [torch.zeros(D, device=DEV) for _ in range(W)]
    for t in range(0, 5):  # t = 0 and 3 are dense rounds (K = 3)
        grads = [torch.empty(D, device=DEV) for _ in range(W)]
        for w in range(W):
            mb.fill_recipe(grads[w], t % 2, seed, w, t)
        dense = t % period == 0
        if dense:
            mean_1 = torch.empty(D, device=DEV)
            single.dense_round(t, grads, comp_1, mean_1)
            means = [torch.empty(D, device=DEV) for _ in range(G)]
            full = run_ranks(ctxs, G, ml, t, period, seed, grads, comp_g, dense_mean=means)
            assert full
            for m in means:
                assert torch.equal(m, mean_1)
        else:
            agg_1 = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
            single.sign_round(t, ETA, seed, grads, comp_1, agg_bits=agg_1)
            full = run_ranks(ctxs, G, ml, t, period, seed, grads, comp_g)
            assert not full
            # every rank holds the full aggregate after the all-gather
            for c in ctxs:
                lay = c.exchange_layout(False)
                assert lay.gather is not None
        torch.cuda.synchronize()
        for w in range(W):
            assert torch.equal(comp_g[w], comp_1[w]), (t, w)
    single.check()
    for c in ctxs:
        c.check()


def test_external_transport_rejects_one_shot_rounds():
    sched = mb.build_ring_schedule(4)
    ctx = mb.Context(1000, sched, torch.float32, 0, nranks=2, rank=0, external_transport=True)
    g = [torch.zeros(1000, device=DEV) for _ in range(2)]
    with pytest.raises(mb.UnsupportedError):
        ctx.sign_round(1, ETA, 1, g, g)


@pytest.mark.slow
@pytest.mark.parametrize("topo,a,b,D", [("ring", 8, 0, 61_000_000), ("torus", 2, 4, 60_200_000)])
def test_full_size_c2_c4_ranks_bit_identical(topo, a, b, D):
    """C2 (ring 8, D = 61M: 40-bit segment tail) and C4 (torus 2x4, D = 60.2M:
    8-bit tail) at full size: the G = 8 rank decomposition reproduces the
    single-context round bit for bit, g_t = +-eta and c' = (g + c) - g_t hold
    exactly (fp32-exact dyadic inputs)."""
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    W, G, seed, t = sched.workers, 8, 2026, 1
    grads = [torch.empty(D, device=DEV) for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(grads[w], 0, seed, w, t)
    single = mb.Context(D, sched, torch.float32, 0)
    comp_1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    upd = torch.empty(D, device=DEV)
    single.sign_round(t, ETA, seed, grads, comp_1, update=upd)
    torch.cuda.synchronize()
    assert bool(((upd == ETA) | (upd == -ETA)).all())
    for w in (0, W - 1):
        assert torch.equal(comp_1[w], grads[w] - upd)  # c = 0: c' = g - g_t exactly
    ctxs = [mb.Context(D, sched, torch.float32, 0, nranks=G, rank=r, external_transport=True)
            for r in range(G)]
    comp_g = [torch.zeros(D, device=DEV) for _ in range(W)]
    run_ranks(ctxs, G, W // G, t, None, seed, grads, comp_g)
    torch.cuda.synchronize()
    for w in range(W):
        assert torch.equal(comp_g[w], comp_1[w]), w
    single.check()


# --------------------------------------------------------------------------
# P2P transport (fused over peer memory): on one GPU the G rank contexts'
# peer tables point at each other's buffers.  Phase-ordered on one stream,
# every stream wait is already satisfied when it is reached; the concurrent
# variant below runs each rank on its own stream so the waits really block.
# --------------------------------------------------------------------------
def p2p_contexts(D, sched, G, dtype=torch.float32):
    ctxs = [mb.Context(D, sched, dtype, 0, nranks=G, rank=r, transport="p2p") for r in range(G)]
    table = [c.p2p_buffers() for c in ctxs]
    for c in ctxs:
        c.set_peers(table)
    return ctxs


@pytest.mark.parametrize("topo,a,b,G,D", [
    ("ring", 8, 0, 2, 100_003),
    ("ring", 8, 0, 8, 25_601),
    ("torus", 2, 4, 4, 60_211),
    ("torus", 2, 4, 8, 1_000_003),
    ("ring", 4, 0, 4, 1_000_000),
])
def test_p2p_transport_matches_single_context(topo, a, b, G, D):
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    W = sched.workers
    ml = W // G
    seed, period = 2026, 3
    single = mb.Context(D, sched, torch.float32, 0)
    ctxs = p2p_contexts(D, sched, G)
    comp_1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    comp_g = [torch.zeros(D, device=DEV) for _ in range(W)]
    for t in range(0, 5):  # t = 0 and 3 are dense rounds (K = 3)
        grads = [torch.empty(D, device=DEV) for _ in range(W)]
        for w in range(W):
            mb.fill_recipe(grads[w], t % 2, seed, w, t)
        dense = t % period == 0
        agg_1 = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
        mean_1 = torch.empty(D, device=DEV)
        if dense:
            single.dense_round(t, grads, comp_1, mean_1)
        else:
            single.sign_round(t, ETA, seed, grads, comp_1, agg_bits=agg_1)
        aggs = [torch.empty_like(agg_1) for _ in range(G)]
        means = [torch.empty(D, device=DEV) for _ in range(G)]
        for phase in range(3):
            for r, ctx in enumerate(ctxs):
                loc = slice(r * ml, (r + 1) * ml)
                full = ctx.round_phase(phase, t, period, ETA, seed, grads[loc], comp_g[loc],
                                       agg_bits=None if dense else aggs[r],
                                       update=means[r] if dense else None)
                assert full == dense
        torch.cuda.synchronize()
        for w in range(W):
            assert torch.equal(comp_g[w], comp_1[w]), (t, w)
        for r in range(G):
            if dense:
                assert torch.equal(means[r], mean_1), (t, r)
            else:
                assert torch.equal(aggs[r], agg_1), (t, r)  # every rank reads every owner
    single.check()
    for c in ctxs:
        c.check()


@pytest.mark.parametrize("flag_kernel", ["0", "1"])
@pytest.mark.parametrize("G", [2, 4])
def test_p2p_transport_concurrent_streams(G, flag_kernel, monkeypatch):
    """Each rank's whole round on its own stream, enqueued rank by rank: rank
    0's stream blocks in its flag wait until the other ranks' extracts ran.
    Small D, so every rank's cooperative merge grid fits the GPU at once.
    flag_kernel = 1: the epoch flags are stored by a kernel (the fallback when
    stream writes to peer memory are unavailable)."""
    monkeypatch.setenv("MARSIT_P2P_FLAG_KERNEL", flag_kernel)
    sched = mb.build_ring_schedule(8)
    W, D, seed = 8, 50_003, 7
    ml = W // G
    single = mb.Context(D, sched, torch.float32, 0)
    ctxs = p2p_contexts(D, sched, G)
    streams = [torch.cuda.Stream() for _ in range(G)]
    comp_1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    comp_g = [torch.zeros(D, device=DEV) for _ in range(W)]
    for t in range(1, 4):
        grads = [torch.empty(D, device=DEV) for _ in range(W)]
        for w in range(W):
            mb.fill_recipe(grads[w], 0, seed, w, t)
        single.sign_round(t, ETA, seed, grads, comp_1)
        torch.cuda.synchronize()
        for r, ctx in enumerate(ctxs):
            loc = slice(r * ml, (r + 1) * ml)
            ctx.sign_round(t, ETA, seed, grads[loc], comp_g[loc], stream=streams[r].cuda_stream)
        torch.cuda.synchronize()
        for w in range(W):
            assert torch.equal(comp_g[w], comp_1[w]), (t, w)


def test_p2p_transport_requires_peers():
    sched = mb.build_ring_schedule(4)
    ctx = mb.Context(1000, sched, torch.float32, 0, nranks=2, rank=0, transport="p2p")
    g = [torch.zeros(1000, device=DEV) for _ in range(2)]
    with pytest.raises(mb.ParameterError):
        ctx.sign_round(1, ETA, 1, g, g)
    with pytest.raises(mb.ParameterError):
        ctx.set_peers([ctx.p2p_buffers()])  # one entry per rank
