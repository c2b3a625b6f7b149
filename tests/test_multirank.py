"""Multi-rank decomposition on CPU (gloo, world_size 2 and 4).

The B200 path on G GPUs (runtime.cu: run_exchange / run_merge / run_allgather)
splits the M workers M/G per rank and gives rank q the contiguous segments
[q*S/G, (q+1)*S/G).  This test replays exactly that data movement with
torch.distributed (gloo) on packed words — per-destination contiguous send
blocks, receive layout [source rank][owned segment][local worker], owner-side
evaluation of the product's compiled merge DAG (sched.plan) with the oracle's
merge, in-place all-gather of the owned aggregates — and requires the result
to equal the single-process reference round (via the oracle pinned to it).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import pyoracle as O

ETA = 2.0 ** -10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _pack_local(g, c, M, L, D, w):
    u = g + c
    nw = O.words64(L)
    out = np.zeros((M, nw), np.uint64)  # [segment][words]
    for s in range(M):
        part = np.zeros(L)
        lo, hi = s * L, min((s + 1) * L, D)
        if hi > lo:
            part[:hi - lo] = u[lo:hi]
        out[s] = O.pack_signs(part)
    return out


def _rank_main(rank, world, port, topo, a, b, D, t, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2204_06787_b200 as mb
        sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
        M, S = sched.workers, sched.segments
        ml, s_own = M // world, S // world
        L = -(-D // S)
        nw = O.words64(L)
        first = rank * ml
        # K1 on the local workers: bits[segment][local worker][words]
        grads = {w: O.gen_dyadic(seed, w, t, D) for w in range(first, first + ml)}
        comp = {w: np.zeros(D) for w in grads}
        bits = np.zeros((S, ml, nw), np.uint64)
        for i, w in enumerate(range(first, first + ml)):
            bits[:, i, :] = _pack_local(grads[w], comp[w], S, L, D, w)
        # exchange: destination q gets segments [q*s_own, (q+1)*s_own) (contiguous)
        send = torch.from_numpy(bits.view(np.int64).copy()).reshape(world, s_own * ml * nw)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send)
        recv = recv.numpy().view(np.uint64).reshape(world, s_own, ml, nw)
        # owner-computes merge DAG of each owned segment (receiver keys)
        agg = np.zeros((S, nw), np.uint64)
        for sl in range(s_own):
            s = rank * s_own + sl
            merges, final, _ = sched.plan(s)
            nodes = {w: recv[w // ml, sl, w % ml] for w in range(M)}
            used_after = {}
            for k, m in enumerate(merges):
                key = O.stream_key(seed, 5, m["receiver"], t, s)
                used0 = used_after[m["offset_src"]] if m["offset_src"] >= 0 else 0
                res, used = O.merge_signs(nodes[m["recv_node"]], m["c_recv"],
                                          nodes[m["local_node"]], m["c_local"], L, key, used0)
                nodes[M + k] = res
                used_after[k] = used
            agg[s] = nodes[final]
        # in-place all-gather of the owned aggregate blocks
        mine = torch.from_numpy(agg[rank * s_own:(rank + 1) * s_own].view(np.int64).copy())
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        full = torch.cat(parts).numpy().view(np.uint64).reshape(S, nw)
        q.put((rank, full.tobytes()))
    finally:
        dist.destroy_process_group()


def _spawn_gloo_all_to_all_available():
    return hasattr(dist, "all_to_all_single")


@pytest.mark.parametrize("world,topo,a,b,D", [
    (2, "ring", 4, 0, 1001),
    (2, "torus", 2, 2, 777),
    (4, "ring", 8, 0, 3001),
    (2, "torus", 2, 4, 803),
])
def test_rank_decomposition_matches_single_process(world, topo, a, b, D):
    if not _spawn_gloo_all_to_all_available():
        pytest.skip("torch.distributed.all_to_all_single missing")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    t, seed = 3, 2026
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, topo, a, b, D, t, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference round (the oracle is pinned to the reference)
    T = O.schedule(topo, a, b)
    M = T.workers
    L = -(-D // M)
    nw = O.words64(L)
    signs = np.stack([_pack_local(O.gen_dyadic(seed, w, t, D), np.zeros(D), M, L, D, w)
                      for w in range(M)])
    ref = O.allreduce_sign(T, signs, L, seed, t)
    want = ref.state[0].reshape(M, nw)
    for r in range(world):
        got = np.frombuffer(results[r], np.uint64).reshape(M, nw)
        assert np.array_equal(got, want), f"rank {r}"
