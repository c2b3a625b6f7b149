#!/usr/bin/env python3
"""Small rounds through every kernel of the path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run):
sign rounds (cluster merge, coins, extract, decode, metrics decode, export,
consensus hashes), a dense round, a torus plan with a two-merge level, the
one-merge merge_signs entry, and 2 emulated P2P ranks phase-ordered on one
stream (stream-ordered flag waits already satisfied).  Exits 0 when every
result equals the single-context round."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

ETA, SEED = 2.0 ** -10, 2026
D = int(os.environ.get("SAN_DIM", "20011"))


def rounds(ctx, W, g, c, ts, period=None):
    for t in ts:
        if period and t % period == 0:
            ctx.dense_round(t, g, c, torch.empty(D, device="cuda"))
        else:
            ctx.sign_round(t, ETA, SEED, g, c, agg_bits=torch.empty((D + 63) // 64, dtype=torch.int64,
                                                                    device="cuda"),
                           update=torch.empty(D, device="cuda"))


ok = True
for topo, a, b in (("ring", 4, 0), ("torus", 2, 2)):
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    W = sched.workers
    g = [torch.empty(D, device="cuda") for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(g[w], 0, SEED, w, 1)
    c1 = [torch.zeros(D, device="cuda") for _ in range(W)]
    ctx = mb.Context(D, sched, torch.float32, 0)
    ctx.set_metrics(True)
    ctx.set_consensus(True)
    rounds(ctx, W, g, c1, range(1, 5), period=3)
    ctx.metrics()
    ctx.check()
    # P2P, 2 emulated ranks, phase-ordered
    ranks = [mb.Context(D, sched, torch.float32, 0, nranks=2, rank=r, transport="p2p") for r in (0, 1)]
    tab = [r.p2p_buffers() for r in ranks]
    for r in ranks:
        r.set_peers(tab)
        r.set_consensus(True)
    cg = [torch.zeros(D, device="cuda") for _ in range(W)]
    ml = W // 2
    for t in range(1, 5):
        for ph in range(3):
            for q, r in enumerate(ranks):
                r.round_phase(ph, t, 3, ETA, SEED, g[q * ml:(q + 1) * ml], cg[q * ml:(q + 1) * ml],
                              update=torch.empty(D, device="cuda"))
    torch.cuda.synchronize()
    for r in ranks:
        r.check()
    ok &= all(torch.equal(x, y) for x, y in zip(c1, cg))
# merge_signs (one-merge plan, inline draws)
x = torch.randint(-2**62, 2**62, ((D + 63) // 64,), dtype=torch.int64, device="cuda")
y = torch.randint(-2**62, 2**62, ((D + 63) // 64,), dtype=torch.int64, device="cuda")
if D % 64:
    x[-1] &= (1 << (D % 64)) - 1
    y[-1] &= (1 << (D % 64)) - 1
mb.merge_signs(mb.AggregateSign(x, 3, D), mb.AggregateSign(y, 1, D), key=12345, used=7)
torch.cuda.synchronize()
print("SANITIZE ROUNDS", "OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
