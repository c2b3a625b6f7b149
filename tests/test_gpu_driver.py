"""GPU tests of the multi-step sync driver (marsit_driver_*): compensation
carry-over, dense cadence, fused replica update, buckets, checkpoint/resume,
reference-format params checkpoint — against the oracle (pinned to the
reference) replaying trainer.hpp's loop."""
import os
import struct
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2204_06787_b200 as mb  # noqa: E402
import pyoracle as O  # noqa: E402

DEV = "cuda:0"
M64 = (1 << 64) - 1
GAMMA = 0x9e3779b97f4a7c15


def mix64(z):
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M64
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M64
    return z ^ (z >> 31)


def bucket_seed(seed, b, nb):
    return seed if nb == 1 else mix64(seed ^ (((b + 1) * GAMMA) & M64))


def oracle_trainer(T, D, rounds, seed, eta, period, bucket, first_round, grads_fn, x0):
    """trainer.hpp:184-307 sync part: per round, per bucket marsit_round, comp
    carried, params -= update on every replica."""
    W = T.workers
    comp = np.zeros((W, D))
    x = np.array(x0, dtype=np.float64)
    bounds = [(o, min(o + bucket, D)) for o in range(0, D, bucket)] if bucket else [(0, D)]
    bits = 0
    for t in range(first_round, first_round + rounds):
        g = grads_fn(t)
        upd = np.zeros(D)
        for bi, (lo, hi) in enumerate(bounds):
            r = O.marsit_round(T, t, period, eta, g[:, lo:hi], comp[:, lo:hi],
                               bucket_seed(seed, bi, len(bounds)))
            assert r.status == 0
            comp[:, lo:hi] = r.comp
            upd[lo:hi] = r.update
            bits += int(r.bits_per_worker.sum())
        x = x - upd
    return comp, x, bits


@pytest.mark.parametrize("topo,a,b,D,bucket,period", [
    ("ring", 4, 0, 10_007, 0, None),
    ("ring", 4, 0, 10_007, 4000, None),
    ("torus", 2, 3, 9_001, 2500, 3),
    ("ring", 8, 0, 65_537, 0, 2),
])
def test_driver_matches_reference_trainer_loop(topo, a, b, D, bucket, period):
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    T = O.schedule(topo, a, b)
    W, seed, eta, rounds = sched.workers, 2026, 2.0 ** -10, 5
    first = 0 if period else 1

    def grads_fn(t):
        return np.stack([O.gen_correlated(seed, w, t, D) for w in range(W)])

    rng = np.random.default_rng(0)
    x0 = rng.standard_normal(D)
    drv = mb.Driver(D, sched, eta_s=eta, global_seed=seed, period=period, bucket_elems=bucket,
                    dtype=torch.float64, first_round=first)
    xs = [torch.tensor(x0, dtype=torch.float64, device=DEV) for _ in range(W)]
    for t in range(first, first + rounds):
        g = [torch.tensor(v, dtype=torch.float64, device=DEV) for v in grads_fn(t)]
        full = drv.step(g, params=xs)
        assert full == (period is not None and t % period == 0)
    torch.cuda.synchronize()
    comp_w, x_w, bits_w = oracle_trainer(T, D, rounds, seed, eta, period, bucket, first, grads_fn,
                                         x0)
    for w in range(W):
        assert np.array_equal(drv.compensation(w).cpu().numpy(), comp_w[w])
        assert np.array_equal(xs[w].cpu().numpy(), x_w)  # identical replicas (consensus)
    st = drv.state()
    assert st["next_round"] == first + rounds
    assert st["cum_bits"] == bits_w
    assert st["buckets"] == (-(-D // bucket) if bucket else 1)


def test_driver_checkpoint_resume_is_bit_identical():
    sched = mb.build_ring_schedule(4)
    D, seed, eta = 20_011, 7, 2.0 ** -10
    grads = {t: [torch.empty(D, device=DEV) for _ in range(4)] for t in range(1, 7)}
    for t, gs in grads.items():
        for w, g in enumerate(gs):
            mb.fill_recipe(g, 1, seed, w, t)
    kw = dict(eta_s=eta, global_seed=seed, period=4, bucket_elems=6000, first_round=1)
    a = mb.Driver(D, sched, **kw)
    xa = [torch.zeros(D, device=DEV) for _ in range(4)]
    for t in (1, 2, 3):
        a.step(grads[t], params=xa)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "sync.state")
        a.save(path)
        x_saved = [x.clone() for x in xa]
        for t in (4, 5, 6):
            a.step(grads[t], params=xa)
        b = mb.Driver(D, sched, **kw)
        b.load(path)
        assert b.state()["next_round"] == 4
        xb = x_saved
        for t in (4, 5, 6):
            b.step(grads[t], params=xb)
        torch.cuda.synchronize()
        for w in range(4):
            assert torch.equal(a.compensation(w), b.compensation(w))
            assert torch.equal(xa[w], xb[w])
        assert a.state() == b.state()
        # a state from a different configuration is refused
        c = mb.Driver(D, sched, **{**kw, "global_seed": 8})
        with pytest.raises(mb.ParameterError):
            c.load(path)
        # so is a truncated file or one with trailing bytes
        blob = open(path, "rb").read()
        for bad in (blob[:-4], blob + b"\0"):
            with open(path, "wb") as f:
                f.write(bad)
            with pytest.raises(mb.ParameterError):
                b.load(path)


def test_params_checkpoint_uses_reference_format():
    x = torch.randn(1001, dtype=torch.float64, device=DEV)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "params.ckpt")
        mb.write_params_checkpoint(path, x)
        blob = open(path, "rb").read()
        # checkpoint.hpp:18-24: magic, u32 version, u64 D, D little-endian doubles
        assert blob[:12] == b"marsit-ckpt\0"
        assert struct.unpack("<I", blob[12:16])[0] == 1
        assert struct.unpack("<Q", blob[16:24])[0] == 1001
        assert np.array_equal(np.frombuffer(blob[24:], "<f8"), x.cpu().numpy())
        y = torch.empty_like(x)
        mb.read_params_checkpoint(path, y)
        assert torch.equal(x, y)
        with pytest.raises(mb.ParameterError):
            mb.read_params_checkpoint(path, torch.empty(1000, dtype=torch.float64, device=DEV))
        # read_checkpoint rejects a file whose size is not 24 + 8 D (checkpoint.hpp:84)
        for bad in (blob + b"\0", blob[:-1], blob[:20]):
            with open(path, "wb") as f:
                f.write(bad)
            with pytest.raises(mb.ParameterError):
                mb.read_params_checkpoint(path, y)


@pytest.mark.slow
def test_c5_bucketed_round_properties():
    """C5 size (D = 355M, M = 8, 4 buckets): per-step properties that hold at any
    size — compensation identity c' = (g + c) - g_t bit for bit, g_t = +-eta,
    the replica update x' = x - g_t, unanimous coordinates keep their sign."""
    D, W, eta = 355_000_000, 8, 2.0 ** -10
    sched = mb.build_ring_schedule(W)
    drv = mb.Driver(D, sched, eta_s=eta, global_seed=5, bucket_elems=100_000_000, first_round=1)
    g = [torch.empty(D, device=DEV) for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(g[w], 1, 5, w, 1)
    x = [torch.zeros(D, device=DEV)]
    upd = torch.empty(D, device=DEV)
    c_before = [drv.compensation(w).clone() for w in (0, 7)]
    drv.step(g, update=upd)
    torch.cuda.synchronize()
    assert bool(((upd == eta) | (upd == -eta)).all())
    for i, w in enumerate((0, 7)):
        want = (g[w] + c_before[i]) - upd
        assert torch.equal(drv.compensation(w), want)
    # coordinates where all 8 workers agree on the sign of u = g (c = 0)
    pos = torch.stack([gw >= 0 for gw in g]).all(0)
    neg = torch.stack([gw < 0 for gw in g]).all(0)
    assert bool((upd[pos] == eta).all()) and bool((upd[neg] == -eta).all())
    assert drv.state()["buckets"] == 4
    del x


@pytest.mark.parametrize("G,bucket", [(2, 4000), (4, 0)])
def test_driver_p2p_transport_matches_single_driver(G, bucket):
    """G rank drivers with the P2P transport on one GPU (each rank's steps on
    its own stream; the stream flag waits block until the other ranks'
    phases ran) against one driver holding every worker: compensation and
    replicas bit-identical over sign and dense rounds."""
    sched = mb.build_ring_schedule(8)
    W, D, seed, eta = 8, 10_007, 5, 2.0 ** -10
    ml = W // G
    kw = dict(eta_s=eta, global_seed=seed, period=3, bucket_elems=bucket, first_round=1)
    one = mb.Driver(D, sched, **kw)
    ranks = [mb.Driver(D, sched, nranks=G, rank=r, transport="p2p", **kw) for r in range(G)]
    for b in range(ranks[0].state()["buckets"]):
        table = [d.p2p_buffers(b) for d in ranks]
        for d in ranks:
            d.set_peers(b, table)
    streams = [torch.cuda.Stream() for _ in range(G)]
    x1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    xg = [torch.zeros(D, device=DEV) for _ in range(W)]
    for t in range(1, 6):  # t = 3 dense
        g = [torch.empty(D, device=DEV) for _ in range(W)]
        for w in range(W):
            mb.fill_recipe(g[w], 1, seed, w, t)
        one.step(g, params=x1)
        torch.cuda.synchronize()
        for r, d in enumerate(ranks):
            loc = slice(r * ml, (r + 1) * ml)
            d.step(g[loc], params=xg[loc], stream=streams[r].cuda_stream)
        torch.cuda.synchronize()
    for r, d in enumerate(ranks):
        for i in range(ml):
            assert torch.equal(d.compensation(i), one.compensation(r * ml + i)), (r, i)
    for w in range(W):
        assert torch.equal(xg[w], x1[w])
    assert all(d.state()["next_round"] == one.state()["next_round"] for d in ranks)
