"""Distributed failure handling and data consensus of multi-rank contexts
(SURVEY §5 "Failure detection"; the reference's contract for a broken wire is
protocol_error, errors.hpp:24-29, and its consensus check is
allreduce.hpp:32-43, called by marsit_round at sync.hpp:101).

* A rank whose peer never reports its epoch does not hang: the context's
  watchdog releases the stream waits after the timeout and every call
  raises ProtocolError; the peer that later runs sees the abort.
* Opt-in consensus: every rank re-hashes the aggregate it read against its
  owners' hashes; a corrupted owner row (after the owner hashed it) raises
  ProtocolError on every rank that read it, a clean round stays bit-exact.

Emulated ranks on one GPU: stream-ordered flag waits only (no kernel waits on
another), as in test_gpu_multirank_emulated.py."""
import time

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2204_06787_b200 as mb  # noqa: E402
from test_gpu_multirank_emulated import p2p_contexts, raw, run_ranks  # noqa: E402

DEV = "cuda:0"
ETA = 2.0 ** -10


def agg_row_offset(D, S, seg):
    """Byte offset of aggregate row `seg` (rows of wst + 4 u32 words)."""
    L = -(-D // S)
    words_proc = (2 * -(-L // 64) + 3) // 4 * 4
    wst = (words_proc + 31) // 32 * 32
    return seg * (wst + 4) * 4


def test_missing_peer_times_out_instead_of_hanging():
    sched = mb.build_ring_schedule(4)
    D, G, seed = 10_007, 2, 3
    ctxs = p2p_contexts(D, sched, G)
    ctxs[0].set_wait_timeout(1500)
    g = [torch.empty(D, device=DEV) for _ in range(4)]
    for w in range(4):
        mb.fill_recipe(g[w], 0, seed, w, 1)
    comp = [torch.zeros(D, device=DEV) for _ in range(4)]
    st0 = torch.cuda.Stream()
    t0 = time.time()
    ctxs[0].sign_round(1, ETA, seed, g[:2], comp[:2], stream=st0.cuda_stream)  # rank 1 never runs
    with pytest.raises(mb.ProtocolError, match="peer rank 1 has not reported"):
        ctxs[0].check(stream=st0.cuda_stream)
    waited = time.time() - t0
    assert 1.0 < waited < 60.0, waited
    torch.cuda.synchronize()  # the released stream drained
    with pytest.raises(mb.ProtocolError):  # latched: no new round is enqueued
        ctxs[0].sign_round(2, ETA, seed, g[:2], comp[:2], stream=st0.cuda_stream)
    with pytest.raises(mb.ProtocolError):
        ctxs[0].status()
    # the late peer's waits pass (abort value) and it reports the abort
    st1 = torch.cuda.Stream()
    ctxs[1].sign_round(1, ETA, seed, g[2:], comp[2:], stream=st1.cuda_stream)
    with pytest.raises(mb.ProtocolError, match="peer rank 0 aborted"):
        ctxs[1].check(stream=st1.cuda_stream)
    torch.cuda.synchronize()


@pytest.mark.parametrize("G", [2, 4])
def test_consensus_clean_round_is_bit_exact(G):
    sched = mb.build_ring_schedule(8)
    D, seed, W = 100_003, 9, 8
    ml = W // G
    single = mb.Context(D, sched, torch.float32, 0)
    single.set_consensus(True)
    ctxs = p2p_contexts(D, sched, G)
    for c in ctxs:
        c.set_consensus(True)
    comp_1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    comp_g = [torch.zeros(D, device=DEV) for _ in range(W)]
    for t in (1, 2):
        grads = [torch.empty(D, device=DEV) for _ in range(W)]
        for w in range(W):
            mb.fill_recipe(grads[w], 0, seed, w, t)
        single.sign_round(t, ETA, seed, grads, comp_1)
        for phase in range(3):
            for r, ctx in enumerate(ctxs):
                loc = slice(r * ml, (r + 1) * ml)
                ctx.round_phase(phase, t, None, ETA, seed, grads[loc], comp_g[loc])
        torch.cuda.synchronize()
        single.check()
        for c in ctxs:
            c.check()
        for w in range(W):
            assert torch.equal(comp_g[w], comp_1[w]), (t, w)


def test_consensus_detects_a_corrupted_owner_row_p2p():
    sched = mb.build_ring_schedule(4)
    D, G, seed, W = 40_000, 2, 5, 4
    S = sched.segments
    ctxs = p2p_contexts(D, sched, G)
    for c in ctxs:
        c.set_consensus(True)
    grads = [torch.empty(D, device=DEV) for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(grads[w], 0, seed, w, 1)
    comp = [torch.zeros(D, device=DEV) for _ in range(W)]
    for phase in (0, 1):
        for r, ctx in enumerate(ctxs):
            ctx.round_phase(phase, 1, None, ETA, seed, grads[2 * r:2 * r + 2], comp[2 * r:2 * r + 2])
    torch.cuda.synchronize()
    # rank 1 owns segments 2, 3: flip one bit of segment 3 after it was hashed
    buf = ctxs[1].p2p_buffers()
    off = agg_row_offset(D, S, 3)
    row = raw(buf.agg + off, 8)
    row[5] ^= 0x10
    for r, ctx in enumerate(ctxs):
        ctx.round_phase(2, 1, None, ETA, seed, grads[2 * r:2 * r + 2], comp[2 * r:2 * r + 2])
    torch.cuda.synchronize()
    for c in ctxs:  # both ranks read segment 3
        with pytest.raises(mb.ProtocolError, match="consensus"):
            c.check()


def test_consensus_detects_a_corrupted_gather_block_external():
    """Owner-computes with the caller's transport (as NCCL moves the blocks):
    a gather block damaged in transit is caught by the receiving rank only."""
    sched = mb.build_torus_schedule(2, 2)
    D, G, seed, W = 30_011, 2, 4, 4
    ml = W // G
    ctxs = [mb.Context(D, sched, torch.float32, 0, nranks=G, rank=r, external_transport=True)
            for r in range(G)]
    for c in ctxs:
        c.set_consensus(True)
    grads = [torch.empty(D, device=DEV) for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(grads[w], 1, seed, w, 1)
    comp = [torch.zeros(D, device=DEV) for _ in range(W)]
    run_ranks(ctxs, G, ml, 1, None, seed, grads, comp)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check()
    # next round: corrupt rank 0's copy of rank 1's block between the phases
    comp2 = [torch.zeros(D, device=DEV) for _ in range(W)]
    for phase in range(3):
        for r, ctx in enumerate(ctxs):
            ctx.round_phase(phase, 2, None, ETA, seed, grads[r * ml:(r + 1) * ml],
                            comp2[r * ml:(r + 1) * ml])
        lays = [c.exchange_layout(False) for c in ctxs]
        if phase == 0:
            B = lays[0].block_bytes
            sends = [raw(l.send, B * G) for l in lays]
            recvs = [raw(l.recv, B * G) for l in lays]
            for r in range(G):
                for q in range(G):
                    recvs[q][r * B:(r + 1) * B].copy_(sends[r][q * B:(q + 1) * B])
        elif phase == 1:
            B = lays[0].gather_block_bytes
            gath = [raw(l.gather, B * G) for l in lays]
            for r in range(G):
                for q in range(G):
                    if q != r:
                        gath[q][r * B:(r + 1) * B].copy_(gath[r][r * B:(r + 1) * B])
            gath[0][B + 3] ^= 0x01  # rank 0's copy of rank 1's block
    torch.cuda.synchronize()
    with pytest.raises(mb.ProtocolError, match="consensus"):
        ctxs[0].check()
    ctxs[1].check()
