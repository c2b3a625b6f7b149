"""On-device round metrics against the oracle: the matching
count of analysis.hpp:244-253 on the trainer's input mean (trainer.hpp:241-251),
the merge disagreement counters (coins drawn = sum of the streams' positions
after the round, allreduce.hpp:170-177) and the round's BitsAccount.  Integer
counters: exact.  The metrics variant of the decode must not change any result
bit."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2204_06787_b200 as mb  # noqa: E402
import pyoracle as O  # noqa: E402

DEV = "cuda:0"
ETA = 2.0 ** -10


def sched_pair(topo, a, b):
    s = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    return s, O.schedule(topo, a, b)


def gen(recipe, seed, w, t, D):
    return (O.gen_dyadic if recipe == 0 else O.gen_correlated)(seed, w, t, D)


@pytest.mark.parametrize("topo,a,b,D,recipe,dtype", [
    ("ring", 8, 0, 100_003, 0, torch.float32),
    ("ring", 4, 0, 65_536, 1, torch.float32),
    ("torus", 2, 4, 60_211, 1, torch.float64),
    ("ring", 5, 0, 37, 0, torch.float64),
    ("ring", 2, 0, 4_099, 0, torch.float32),
    ("ring", 8, 0, 262_144, 1, torch.float32),    # aligned quads
    ("ring", 16, 0, 50_001, 0, torch.float32),
])
def test_metrics_match_oracle_over_rounds(topo, a, b, D, recipe, dtype):
    sched, T = sched_pair(topo, a, b)
    W, seed, period = sched.workers, 2026, 4
    ctx = mb.Context(D, sched, dtype, 0)
    ref = mb.Context(D, sched, dtype, 0)  # same rounds without metrics
    ctx.set_metrics(True)
    comp = [torch.zeros(D, dtype=dtype, device=DEV) for _ in range(W)]
    comp_ref = [torch.zeros(D, dtype=dtype, device=DEV) for _ in range(W)]
    comp_o = np.zeros((W, D))
    for t in range(1, 6):  # t = 4 is dense
        g = np.stack([gen(recipe, seed, w, t, D) for w in range(W)])
        gd = [torch.tensor(x, dtype=dtype, device=DEV) for x in g]
        upd = torch.empty(D, dtype=dtype, device=DEV)
        agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
        upd_r = torch.empty_like(upd)
        agg_r = torch.empty_like(agg)
        f1 = _round(ctx, t, period, seed, gd, comp, agg, upd)
        f2 = _round(ref, t, period, seed, gd, comp_ref, agg_r, upd_r)
        assert f1 == f2 == (t % period == 0)
        r = O.marsit_round(T, t, period, ETA, g, comp_o, seed)
        assert r.status == 0
        m = ctx.metrics()
        assert m.valid and m.round == t and m.full_precision == f1 and m.dim == D
        assert m.round_bits == int(r.bits_per_worker.sum())
        for w in range(W):
            assert torch.equal(comp[w], comp_ref[w]), (t, w)
        assert torch.equal(upd, upd_r)
        if not f1:
            assert torch.equal(agg, agg_r)
            assert m.has_matching
            assert m.matches == O.matching_count(r.agg_bits, g, comp_o), t
            assert m.matching_rate == m.matches / D
            assert m.disagreements == r.draws and m.merges == r.merges, t
            L = -(-D // sched.segments)
            assert m.compared_bits == r.merges * L
            assert m.disagreement_rate == pytest.approx(r.draws / (r.merges * L), rel=0, abs=0)
        else:
            assert not m.has_matching and m.matching_rate is None and m.merges == 0
        comp_o = r.comp
    ctx.check()


def _round(ctx, t, period, seed, g, comp, agg, upd):
    res = mb._native.lib()
    import ctypes as C
    gp = mb._native.ptr_array([x.data_ptr() for x in g])
    cp = mb._native.ptr_array([x.data_ptr() for x in comp])
    fp = C.c_int(0)
    mb._check(res.marsit_round(ctx._h, t, period, ETA, seed, gp, cp, cp,
                               C.c_void_p(agg.data_ptr()), C.c_void_p(upd.data_ptr()),
                               C.byref(fp), mb._stream_ptr(0)))
    return bool(fp.value)


def test_driver_metrics_sum_buckets():
    sched, T = sched_pair("ring", 4, 0)
    W, D, seed, bucket = 4, 10_007, 11, 4000
    drv = mb.Driver(D, sched, eta_s=ETA, global_seed=seed, bucket_elems=bucket, first_round=1)
    drv.set_metrics(True)
    comp_o = np.zeros((W, D))
    bounds = [(o, min(o + bucket, D)) for o in range(0, D, bucket)]
    for t in (1, 2):
        g = np.stack([O.gen_correlated(seed, w, t, D) for w in range(W)])
        drv.step([torch.tensor(x, dtype=torch.float32, device=DEV) for x in g])
        m = drv.metrics()
        matches = draws = merges = bits = 0
        for bi, (lo, hi) in enumerate(bounds):
            bs = seed if len(bounds) == 1 else _bucket_seed(seed, bi)
            r = O.marsit_round(T, t, None, ETA, g[:, lo:hi], comp_o[:, lo:hi], bs)
            matches += O.matching_count(r.agg_bits, g[:, lo:hi], comp_o[:, lo:hi])
            draws += r.draws
            merges += r.merges
            bits += int(r.bits_per_worker.sum())
            comp_o[:, lo:hi] = r.comp
        assert m.round == t and m.has_matching and m.dim == D
        assert (m.matches, m.disagreements, m.merges, m.round_bits) == (matches, draws, merges,
                                                                        bits)


def _bucket_seed(seed, b):
    M = (1 << 64) - 1
    z = seed ^ (((b + 1) * 0x9e3779b97f4a7c15) & M)
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
    return z ^ (z >> 31)


def test_rank_local_disagreements_sum_to_single_context():
    """G = 2 external-transport ranks: each reports its owned segments'
    disagreements (rank_local); they sum to the single-context count."""
    from test_gpu_multirank_emulated import run_ranks
    sched = mb.build_ring_schedule(8)
    W, D, G, seed = 8, 50_003, 2, 5
    single = mb.Context(D, sched, torch.float32, 0)
    single.set_metrics(True)
    ctxs = [mb.Context(D, sched, torch.float32, 0, nranks=G, rank=r, external_transport=True)
            for r in range(G)]
    for c in ctxs:
        c.set_metrics(True)
    grads = [torch.empty(D, device=DEV) for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(grads[w], 0, seed, w, 1)
    c1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    cg = [torch.zeros(D, device=DEV) for _ in range(W)]
    single.sign_round(1, ETA, seed, grads, c1)
    run_ranks(ctxs, G, W // G, 1, None, seed, grads, cg)
    m1 = single.metrics()
    ms = [c.metrics() for c in ctxs]
    assert all(m.rank_local and not m.has_matching for m in ms)
    assert sum(m.disagreements for m in ms) == m1.disagreements
    assert sum(m.merges for m in ms) == m1.merges


@pytest.mark.parametrize("pipeline", ["0", "1"])
def test_c3_matching_count_full_size(pipeline, monkeypatch):
    """C3 (D = 25.6M, M = 8): the fused count equals the count recomputed from
    the fp64 worker-order mean (torch, fp64), on both single-GPU schedules."""
    monkeypatch.setenv("MARSIT_PIPELINE", pipeline)
    D, W, seed = 25_600_000, 8, 2026
    sched = mb.build_ring_schedule(W)
    ctx = mb.Context(D, sched, torch.float32, 0)
    ctx.set_metrics(True)
    g = [torch.empty(D, device=DEV) for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(g[w], 1, seed, w, 1)
    c = [torch.zeros(D, device=DEV) for _ in range(W)]
    agg = torch.empty(D // 64, dtype=torch.int64, device=DEV)
    mean = torch.zeros(D, dtype=torch.float64, device=DEV)
    for w in range(W):
        mean += g[w].double() + c[w].double()
    mean /= W
    ctx.sign_round(1, ETA, seed, g, c, agg_bits=agg)
    m = ctx.metrics()
    shifts = torch.arange(64, device=DEV, dtype=torch.int64)
    bits = ((agg.view(-1, 1) >> shifts) & 1).view(-1).bool()
    want = int((bits == (mean >= 0)).sum())
    assert m.has_matching and m.matches == want
    # correlated inputs: most coordinates agree with the mean sign, and the
    # disagreement rate is well below the independent-sign 50 %
    assert m.matching_rate > 0.6 and 0.0 < m.disagreement_rate < 0.5
    assert m.merges == W * (W - 1) and m.compared_bits == m.merges * (D // W)


@pytest.mark.parametrize("case", range(3))
def test_matching_pinned_to_reference_golden(golden, case):
    """The fused matching count against the REAL reference's figure
    (analysis.hpp:244-253 on trainer.hpp:241-251's fp64 mean of add(g, c),
    tests/golden/metrics.json): fp32 Gaussian inputs plus coordinates where
    the fp32-rounded u = g + c flips the sign of the mean — the device forms
    the mean from the fp64 sum of the two fp32 values, like the trainer."""
    c = golden("metrics")[case]
    sched = (mb.build_ring_schedule(c["a"]) if c["topology"] == "ring"
             else mb.build_torus_schedule(c["a"], c["b"]))
    W, D = sched.workers, c["dim"]
    g, cc = O.gen_metrics_inputs(c["seed"], W, D)
    ctx = mb.Context(D, sched, torch.float32, 0)
    ctx.set_metrics(True)
    gd = [torch.tensor(x, dtype=torch.float32, device=DEV) for x in g]
    cd = [torch.tensor(x, dtype=torch.float32, device=DEV) for x in cc]
    out = [torch.empty_like(x) for x in cd]
    agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
    ctx.sign_round(c["round"], ETA, c["global_seed"], gd, cd, comp_out=out, agg_bits=agg)
    m = ctx.metrics()
    want = np.array([int(x, 16) for x in c["agg_words"]], dtype=np.uint64)
    assert np.array_equal(agg.cpu().numpy().view(np.uint64), want)
    assert m.has_matching and m.matches == c["matches"]
    assert float.fromhex(c["rate"]) == m.matching_rate
