"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
fixtures and the C oracle, bit-exact for sign words / aggregate bits, exact
for compensation when the inputs are fp32-exact (dyadic recipe) and within
1e-6 relative (+ tiny absolute floor) for Gaussian fp32 inputs."""
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2204_06787_b200 as mb  # noqa: E402
import pyoracle as O  # noqa: E402
from conftest import load_golden  # noqa: E402

DEV = "cuda:0"
ETA = 2.0 ** -10


def fx(lst):
    return np.array([float.fromhex(x) for x in lst], np.float64)


def wx(lst):
    return np.array([int(x, 16) for x in lst], np.uint64)


def sched_of(topo, a, b):
    return mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)


def to_dev(arr, dtype):
    return [torch.tensor(x, dtype=dtype, device=DEV) for x in arr]


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, "<f8").tobytes()).hexdigest()


def golden_inputs(case, rnd, W):
    if "grads" in rnd:
        return fx(rnd["grads"]).reshape(W, case["dim"])
    gen = O.gen_dyadic if case["recipe"] == "dyadic" else O.gen_correlated
    return np.stack([gen(case["seed"], w, rnd["t"], case["dim"]) for w in range(W)])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_rounds_match_reference_golden(dtype):
    for case in load_golden("rounds"):
        exact_inputs = case["recipe"] in ("dyadic", "correlated")
        if dtype == torch.float32 and case["recipe"] == "special":
            continue  # its subnormal doubles are not fp32-representable
        sched = sched_of(case["topology"], case["a"], case["b"])
        W, D = sched.workers, case["dim"]
        cfg = mb.SyncConfig(case["period"], case["eta_s"])
        comp = [torch.zeros(D, dtype=dtype, device=DEV) for _ in range(W)]
        for rnd in case["rounds"]:
            g = golden_inputs(case, rnd, W)
            prev_c = np.stack([c.double().cpu().numpy() for c in comp])
            res = mb.marsit_round(rnd["t"], cfg, to_dev(g, dtype), comp, sched, case["seed"])
            assert res.full_precision == rnd["full_precision"]
            assert res.bits.per_worker == rnd["bits_per_worker"]
            assert (res.bits.reduce_bits, res.bits.gather_bits) == (rnd["reduce_bits"],
                                                                   rnd["gather_bits"])
            if not rnd["full_precision"]:
                assert u64(res.aggregate_bits).tolist() == wx(rnd["agg_bits"]).tolist(), case
            got_c = np.stack([c.c.double().cpu().numpy() for c in res.compensation])
            got_u = res.global_update.double().cpu().numpy()
            exact = dtype == torch.float64 or (exact_inputs and not rnd["full_precision"])
            if "comp" in rnd:
                want_c = fx(rnd["comp"]).reshape(W, D)
                want_u = fx(rnd["update"])
                if exact:
                    assert np.array_equal(got_c, want_c), case
                    assert np.array_equal(got_u, want_u), case
                else:
                    # fp32 arithmetic vs the reference's fp64 (north_star: 1e-6
                    # relative).  Sign rounds: g_t = +-eta_s exactly.  c' = (g + c)
                    # - g_t cancels (c' can be ~0 while its operands are ~eta_s), so
                    # "relative" is taken against the operands of the reference's
                    # last operation, per element: |err| <= 1e-6 (|c'| + |g| + eta_s)
                    # (|c| <= |c'| + |g| + eta_s), i.e. no input-independent floor.
                    # (dense rounds: the update is a mean of u and cancels too; its
                    # operands are bounded by max_w |g_w| + |c_w|)
                    bu = 1e-6 * (np.abs(want_u) + np.abs(g).max(0) + np.abs(prev_c).max(0))
                    assert np.all(np.abs(got_u - want_u) <= bu), float((np.abs(got_u - want_u) / bu).max())
                    bound = 1e-6 * (np.abs(want_c) + np.abs(g) + case["eta_s"])
                    err = np.abs(got_c - want_c)
                    assert np.all(err <= bound), (case["name"] if "name" in case else case,
                                                  float((err / bound).max()))
            else:
                assert exact
                assert sha(got_c) == rnd["comp_sha256"], case
                assert sha(got_u) == rnd["update_sha256"], case
            comp = [c.c for c in res.compensation]


def test_survey_anchors_c1():
    """SURVEY §8c known answers for C1 (ring D=1M, M=4, rounds 1..3, fp32)."""
    sched = mb.build_ring_schedule(4)
    D = 1_000_000
    cfg = mb.SyncConfig(None, ETA)
    comp = [torch.zeros(D, device=DEV) for _ in range(4)]
    gold = [g for g in load_golden("anchors") if g["dim"] == D]
    for gd in gold:
        t = gd["t"]
        g = [torch.empty(D, device=DEV) for _ in range(4)]
        for w in range(4):
            mb.fill_recipe(g[w], 0, 2026, w, t)
        res = mb.marsit_round(t, cfg, g, comp, sched, 2026, inplace=True)
        bits = u64(res.aggregate_bits)
        assert int(sum(bin(int(x)).count("1") for x in bits)) == gd["popcount"]
        assert "%016x" % O.fnv1a64(bits) == gd["fnv1a64"]
        assert float(comp[0][0]) == float.fromhex(gd["c00"])
        assert float(comp[0].double().sum()) == pytest.approx(float.fromhex(gd["sum_c0"]),
                                                              abs=1e-12)


def test_device_recipe_matches_oracle_recipe():
    out = torch.empty(10_007, device=DEV)
    for recipe, gen in ((0, O.gen_dyadic), (1, O.gen_correlated)):
        mb.fill_recipe(out, recipe, 2026, 3, 7)
        assert np.array_equal(out.double().cpu().numpy(), gen(2026, 3, 7, 10_007))


@pytest.mark.parametrize("topo,a,b,D,rounds", [
    ("ring", 4, 0, 1_000_000, 3),        # C1
    ("ring", 8, 0, 1_000_003, 2),        # odd D: L % 4 != 0 -> scalar path
    ("torus", 2, 4, 602_001, 2),         # torus with stream continuation
    ("ring", 2, 0, 64 * 1024 * 3 + 17, 2),
    ("ring", 3, 0, 5, 3),
    ("ring", 4, 0, 3, 2),                # one segment is pure padding
])
def test_multi_round_vs_oracle(topo, a, b, D, rounds):
    sched = sched_of(topo, a, b)
    T = O.schedule(topo, a, b)
    W = sched.workers
    cfg = mb.SyncConfig(None, ETA)
    comp_d = [torch.zeros(D, device=DEV) for _ in range(W)]
    comp_h = np.zeros((W, D))
    for t in range(1, rounds + 1):
        gh = np.stack([O.gen_correlated(77, w, t, D) if t % 2 else O.gen_dyadic(77, w, t, D)
                       for w in range(W)])
        res = mb.marsit_round(t, cfg, to_dev(gh, torch.float32), comp_d, sched, 77, inplace=True)
        want = O.marsit_round(T, t, None, ETA, gh, comp_h, 77)
        assert want.status == 0
        assert np.array_equal(u64(res.aggregate_bits), want.agg_bits)
        got = np.stack([c.double().cpu().numpy() for c in comp_d])
        assert np.array_equal(got, want.comp)
        assert np.array_equal(res.global_update.double().cpu().numpy(), want.update)
        comp_h = want.comp


@pytest.mark.slow
def test_c3_full_size_round_vs_oracle():
    """The bench workload (ring M=8, D=25.6M): one round bit-exact vs the oracle."""
    D, W = 25_600_000, 8
    sched = mb.build_ring_schedule(W)
    g = [torch.empty(D, device=DEV) for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(g[w], 0, 2026, w, 1)
    comp = [torch.zeros(D, device=DEV) for _ in range(W)]
    res = mb.marsit_round(1, mb.SyncConfig(None, ETA), g, comp, sched, 2026, want_update=False)
    gh = np.stack([O.gen_dyadic(2026, w, 1, D) for w in range(W)])
    want = O.marsit_round(O.schedule("ring", W), 1, None, ETA, gh, np.zeros((W, D)), 2026)
    assert np.array_equal(u64(res.aggregate_bits), want.agg_bits)
    for w in (0, W - 1):
        assert np.array_equal(res.compensation[w].c.double().cpu().numpy(), want.comp[w])


def test_merge_signs_matches_reference_golden():
    for rec in load_golden("merges"):
        L = rec["length"]
        key = mb.stream_key(rec["seed"], 5, rec["w"], rec["t"], rec["s"])
        r = torch.tensor(wx(rec["recv"]).view(np.int64), device=DEV)
        l_ = torch.tensor(wx(rec["local"]).view(np.int64), device=DEV)
        out, used = mb.merge_signs(mb.AggregateSign(r, rec["c_recv"], L),
                                   mb.AggregateSign(l_, rec["c_local"], L), key, rec["skip"])
        assert u64(out.bits).tolist() == wx(rec["out"]).tolist()
        assert used == rec["consumed"]
        assert out.count == rec["c_recv"] + rec["c_local"]


def test_merge_signs_large_multi_tile_vs_oracle():
    rng = np.random.default_rng(1)
    for L in (32768 * 3 + 5, 200_000):
        nw = (L + 63) // 64
        r = rng.integers(0, 2**63, nw, dtype=np.uint64) * 2 + rng.integers(0, 2, nw, dtype=np.uint64)
        l_ = rng.integers(0, 2**63, nw, dtype=np.uint64)
        r[-1] &= np.uint64((1 << (L % 64)) - 1)
        l_[-1] &= np.uint64((1 << (L % 64)) - 1)
        key = O.stream_key(5, 5, 1, 2, 3)
        want, used = O.merge_signs(r, 3, l_, 2, L, key, 17)
        out, consumed = mb.merge_signs(
            mb.AggregateSign(torch.tensor(r.view(np.int64), device=DEV), 3, L),
            mb.AggregateSign(torch.tensor(l_.view(np.int64), device=DEV), 2, L), key, 17)
        assert np.array_equal(u64(out.bits), want)
        assert consumed == used - 17


def test_allreduce_sign_matches_reference_golden():
    for rec in load_golden("allreduce"):
        sched = sched_of(rec["topology"], rec["a"], rec["b"])
        L = rec["seg_len"]
        nw = (L + 63) // 64
        signs = torch.tensor(wx(rec["signs"]).view(np.int64).reshape(sched.workers,
                                                                    sched.segments, nw),
                             device=DEV)
        out, counts = mb.allreduce_sign(signs, sched, rec["seed"], rec["round"], L)
        state = wx(rec["state"]).reshape(sched.workers, sched.segments, nw)
        assert u64(out).reshape(sched.segments, nw).tolist() == state[0].tolist()
        assert counts == rec["counts"][:sched.segments]


def test_pack_signs_matches_oracle_with_zeros_and_subnormals():
    rng = np.random.default_rng(2)
    W, D = 5, 10_001
    sched = mb.build_ring_schedule(W)
    g = rng.standard_normal((W, D)).astype(np.float32)
    c = rng.standard_normal((W, D)).astype(np.float32)
    g[:, ::5] = 0.0
    g[:, 1::5] = -0.0
    c[:, ::5] = 0.0
    c[:, 1::5] = -0.0  # -0.0 + -0.0 = -0.0 -> bit 1
    g[:, 2::5] = np.float32(1e-45)
    c[:, 2::5] = 0.0
    g[:, 3::5] = np.float32(-1e-45)
    c[:, 3::5] = 0.0
    out = mb.pack_signs(to_dev(g, torch.float32), to_dev(c, torch.float32), sched)
    L = -(-D // W)
    u = g.astype(np.float64) + c.astype(np.float64)
    for w in range(W):
        for s in range(W):
            part = np.zeros(L)
            lo, hi = s * L, min((s + 1) * L, D)
            part[:hi - lo] = u[w, lo:hi]
            assert u64(out[w, s]).tolist() == O.pack_signs(part).tolist()


def test_errors_map_to_reference_exceptions():
    sched = mb.build_ring_schedule(2)
    g = [torch.ones(8, device=DEV), torch.ones(8, device=DEV)]
    c = [torch.zeros(8, device=DEV), torch.zeros(8, device=DEV)]
    with pytest.raises(mb.ParameterError):
        mb.marsit_round(1, mb.SyncConfig(0, 0.1), g, c, sched, 1)
    with pytest.raises(mb.ParameterError):
        mb.marsit_round(1, mb.SyncConfig(None, 0.0), g, c, sched, 1)
    with pytest.raises(mb.ParameterError):
        mb.marsit_round(1, mb.SyncConfig(None, 0.1), g[:1], c, sched, 1)
    bad = [torch.ones(8, device=DEV), torch.tensor([1.0] * 7 + [float("nan")], device=DEV)]
    with pytest.raises(mb.NonFiniteError):
        mb.marsit_round(1, mb.SyncConfig(None, 0.1), bad, c, sched, 1)
    big = [torch.full((8,), 3e38, device=DEV)] * 2
    with pytest.raises(mb.NonFiniteError):  # u = g + c overflows
        mb.marsit_round(1, mb.SyncConfig(None, 0.1), big, big, sched, 1)
    # the latch is cleared: the next good round succeeds
    mb.marsit_round(2, mb.SyncConfig(None, 0.1), g, c, sched, 1)
    with pytest.raises(mb.ParameterError):
        mb.build_ring_schedule(1)
    with pytest.raises(mb.ParameterError):
        mb.build_torus_schedule(1, 3)


def test_value_semantics_and_inplace_agree():
    sched = mb.build_torus_schedule(2, 3)
    D = 4099
    g = [torch.empty(D, device=DEV) for _ in range(6)]
    for w in range(6):
        mb.fill_recipe(g[w], 0, 9, w, 1)
    c0 = [torch.zeros(D, device=DEV) for _ in range(6)]
    a = mb.marsit_round(1, mb.SyncConfig(None, ETA), g, c0, sched, 9)
    assert all(float(c.abs().sum()) == 0.0 for c in c0)  # inputs untouched
    c1 = [torch.zeros(D, device=DEV) for _ in range(6)]
    b = mb.marsit_round(1, mb.SyncConfig(None, ETA), g, c1, sched, 9, inplace=True)
    for x, y in zip(a.compensation, c1):
        assert torch.equal(x.c, y)
    assert torch.equal(a.aggregate_bits, b.aggregate_bits)


@pytest.mark.parametrize("frac", ["0", "0.2", "0.5", "2"])
@pytest.mark.parametrize("topo,a,b", [("ring", 8, 0), ("torus", 2, 4)])
def test_coin_precompute_budget_and_inline_fallback(frac, topo, a, b, monkeypatch):
    """Precomputed coin bits, the inline-draw fallback beyond the budget, and
    mixtures of both must give identical results (the budget is a tuning knob)."""
    monkeypatch.setenv("MARSIT_COIN_FRAC", frac)
    sched = sched_of(topo, a, b)
    W, D = sched.workers, 300_001
    ctx = mb.Context(D, sched, torch.float32, 0)
    T = O.schedule(topo, a, b)
    comp_d = [torch.zeros(D, device=DEV) for _ in range(W)]
    comp_h = np.zeros((W, D))
    agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
    for t in (1, 2):
        gh = np.stack([O.gen_dyadic(5, w, t, D) for w in range(W)])
        ctx.sign_round(t, ETA, 5, to_dev(gh, torch.float32), comp_d, agg_bits=agg)
        ctx.check()
        want = O.marsit_round(T, t, None, ETA, gh, comp_h, 5)
        assert np.array_equal(u64(agg), want.agg_bits)
        assert np.array_equal(np.stack([c.double().cpu().numpy() for c in comp_d]), want.comp)
        comp_h = want.comp


def test_cpp_dropin_bit_identical_to_reference_in_process():
    """build/dropin_parity (built where the reference headers exist) runs the
    reference's marsit_round/allreduce_sign and marsit::gpu:: versions on the
    same inputs in one process and requires bit-identical results."""
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "build", "dropin_parity")
    if not os.path.exists(exe):
        pytest.skip("dropin_parity binary not shipped")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROP-IN PARITY OK" in r.stdout


def test_coin_prefetch_speculation_is_safe():
    """Round t+1's coins are precomputed during round t; rounds that do not
    follow that guess (jumps in t, a new seed) must still be bit-exact."""
    sched = mb.build_ring_schedule(4)
    D = 100_003
    T = O.schedule("ring", 4)
    ctx = mb.Context(D, sched, torch.float32, 0)
    comp_d = [torch.zeros(D, device=DEV) for _ in range(4)]
    comp_h = np.zeros((4, D))
    agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
    for t, seed in [(1, 7), (2, 7), (5, 7), (3, 7), (4, 7), (4, 8), (5, 8), (6, 9)]:
        gh = np.stack([O.gen_dyadic(seed, w, t, D) for w in range(4)])
        ctx.sign_round(t, ETA, seed, to_dev(gh, torch.float32), comp_d, agg_bits=agg)
        ctx.check()
        want = O.marsit_round(T, t, None, ETA, gh, comp_h, seed)
        assert np.array_equal(u64(agg), want.agg_bits), (t, seed)
        comp_h = want.comp
    assert np.array_equal(np.stack([c.double().cpu().numpy() for c in comp_d]), comp_h)


@pytest.mark.parametrize("wpt", [1, 2, 4, 8, 12, 16])
@pytest.mark.parametrize("topo,a,b,D", [("ring", 8, 0, 1_000_037), ("torus", 2, 4, 700_001),
                                        ("ring", 3, 0, 4_001)])
def test_merge_tilings_bit_exact(wpt, topo, a, b, D, monkeypatch):
    """Every merge tiling (words per thread incl. the 12/16-word tails that
    pass the segment end, balanced grids) of the cooperative merge gives the
    reference's bits."""
    monkeypatch.setenv("MARSIT_MERGE_KERNEL", "coop")
    monkeypatch.setenv("MARSIT_MERGE_WPT", str(wpt))
    monkeypatch.setenv("MARSIT_MERGE_BALANCE", "2" if wpt >= 12 else "0")
    sched = sched_of(topo, a, b)
    T = O.schedule(topo, a, b)
    W, seed = sched.workers, 99
    ctx = mb.Context(D, sched, torch.float32, 0)
    comp_o = np.zeros((W, D))
    comp = [torch.zeros(D, device=DEV) for _ in range(W)]
    for t in (1, 2):
        g = np.stack([O.gen_dyadic(seed, w, t, D) for w in range(W)])
        agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
        ctx.sign_round(t, ETA, seed, [torch.tensor(x, dtype=torch.float32, device=DEV) for x in g],
                       comp, agg_bits=agg)
        r = O.marsit_round(T, t, None, ETA, g, comp_o, seed)
        assert u64(agg).tolist() == r.agg_bits.tolist(), (wpt, topo, t)
        comp_o = r.comp
    ctx.check()


@pytest.mark.parametrize("kernel,csize", [("cluster", "0"), ("cluster", "16"), ("cluster", "4"),
                                          ("cluster", "1"), ("grid", "0"), ("grid", "3"),
                                          ("grid", "1"), ("grid", "100"), ("coop", "0")])
@pytest.mark.parametrize("topo,a,b,D", [("ring", 8, 0, 1_000_037), ("torus", 2, 4, 700_001),
                                        ("torus", 3, 3, 36_011), ("ring", 3, 0, 4_001),
                                        ("ring", 16, 0, 250_003)])
def test_cluster_merge_bit_exact(kernel, csize, topo, a, b, D, monkeypatch):
    """The level-loop merges give the reference's bits for every tile count,
    incl. torus continuation streams and ragged segment ends:
    MARSIT_MERGE_KERNEL=cluster (one thread-block cluster per segment, DSMEM
    totals, csize CTAs), =grid (the default: csize co-resident CTAs per
    segment, cooperative launch, level-tagged totals through global memory)
    and =coop (the cooperative stage merge)."""
    monkeypatch.setenv("MARSIT_MERGE_KERNEL", kernel)
    monkeypatch.setenv("MARSIT_MERGE_CSIZE", csize)
    sched = sched_of(topo, a, b)
    T = O.schedule(topo, a, b)
    W, seed = sched.workers, 77
    ctx = mb.Context(D, sched, torch.float32, 0)
    comp_o = np.zeros((W, D))
    comp = [torch.zeros(D, device=DEV) for _ in range(W)]
    for t in (1, 2, 3):
        g = np.stack([O.gen_dyadic(seed, w, t, D) for w in range(W)])
        agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
        ctx.sign_round(t, ETA, seed, [torch.tensor(x, dtype=torch.float32, device=DEV) for x in g],
                       comp, agg_bits=agg)
        r = O.marsit_round(T, t, None, ETA, g, comp_o, seed)
        assert u64(agg).tolist() == r.agg_bits.tolist(), (csize, topo, t)
        comp_o = r.comp
    ctx.check()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("topo,a,b,D", [("ring", 8, 0, 8192), ("ring", 4, 0, 1_000_000),
                                        ("ring", 8, 0, 8196), ("torus", 2, 4, 8192),
                                        ("torus", 2, 4, 60_224), ("torus", 3, 3, 36_036),
                                        ("torus", 2, 4, 8196), ("torus", 2, 2, 1003)])
def test_dense_round_vector_path_vs_oracle(dtype, topo, a, b, D):
    """Dense rounds whose L and D are multiples of 4 take the 16-byte kernels
    (ring: register chain; torus: the reduction DAG in shared memory), ragged
    sizes the scalar ones: exact vs the oracle, compensation reset to 0."""
    sched = sched_of(topo, a, b)
    T = O.schedule(topo, a, b)
    M = sched.workers
    rng = np.random.default_rng(D + M)
    if dtype == torch.float64:
        g = rng.standard_normal((M, D))
    else:
        g = np.stack([O.gen_dyadic(3, w, 1, D) for w in range(M)])
    comp_o = rng.standard_normal((M, D)) * 1e-3 if dtype == torch.float64 else np.zeros((M, D))
    r = O.marsit_round(T, 2, 2, ETA, g, comp_o, 5)
    assert r.status == 0 and r.full_precision
    ctx = mb.Context(D, sched, dtype, 0)
    comp = [torch.tensor(x, dtype=dtype, device=DEV) for x in comp_o]
    mean = torch.empty(D, dtype=dtype, device=DEV)
    ctx.dense_round(2, [torch.tensor(x, dtype=dtype, device=DEV) for x in g], comp, mean)
    torch.cuda.synchronize()
    want = r.update if dtype == torch.float64 else r.update.astype(np.float32).astype(np.float64)
    assert np.array_equal(mean.double().cpu().numpy(), want)
    assert all(bool((c == 0).all()) for c in comp)
    ctx.check()


@pytest.mark.parametrize("topo,a,b,D,period", [
    ("ring", 33, 0, 40_009, None),    # 32 merges per segment: descriptor cache limit
    ("ring", 64, 0, 70_001, 2),       # 63 merges: descriptors read from global memory
    ("torus", 4, 8, 50_021, 2),
    ("torus", 8, 8, 64 * 1024 + 5, None),
    ("torus", 16, 2, 30_011, 3),      # 16 row chains: more than kMaxLanes = 8 lanes
    ("torus", 2, 16, 40_003, None),   # two long row chains side by side
])
def test_large_worker_counts_vs_oracle(topo, a, b, D, period):
    """Many workers on one context (up to kMaxLocalWorkers = 64): long merge
    chains (more merges per stage than the shared-memory descriptor cache
    holds) and wide dense reduction trees, exact vs the oracle over rounds
    including dense ones."""
    sched = sched_of(topo, a, b)
    T = O.schedule(topo, a, b)
    W, seed = sched.workers, 4242
    ctx = mb.Context(D, sched, torch.float32, 0)
    comp_o = np.zeros((W, D))
    comp = [torch.zeros(D, device=DEV) for _ in range(W)]
    for t in (1, 2, 3):
        g = np.stack([O.gen_dyadic(seed, w, t, D) for w in range(W)])
        r = O.marsit_round(T, t, period, ETA, g, comp_o, seed)
        assert r.status == 0
        gd = [torch.tensor(x, dtype=torch.float32, device=DEV) for x in g]
        if r.full_precision:
            mean = torch.empty(D, device=DEV)
            ctx.dense_round(t, gd, comp, mean)
            got_update = mean
        else:
            agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
            upd = torch.empty(D, device=DEV)
            ctx.sign_round(t, ETA, seed, gd, comp, agg_bits=agg, update=upd)
            assert u64(agg).tolist() == r.agg_bits.tolist(), (topo, t)
            got_update = upd
        torch.cuda.synchronize()
        assert np.array_equal(got_update.double().cpu().numpy(), r.update), (topo, t)
        assert np.array_equal(np.stack([c.double().cpu().numpy() for c in comp]), r.comp)
        comp_o = r.comp
    ctx.check()


@pytest.mark.parametrize("frac", ["0.53", "0.2"])
def test_adaptive_coin_budget_over_rounds_vs_oracle(frac, monkeypatch):
    """Error feedback with a fixed Gaussian gradient drives the disagreement
    rate above 1/2 over rounds; the coin kernel sizes each merge's coins from
    the previous round's end index (first round: MARSIT_COIN_FRAC), and every
    draw beyond them is taken inline — bit-exact against the oracle either
    way, for 8 rounds (fp64, ring 8 and torus 2x4, ragged L)."""
    monkeypatch.setenv("MARSIT_COIN_FRAC", frac)
    for topo, a, b in (("ring", 8, 0), ("torus", 2, 4)):
        D = 300_007
        sched = sched_of(topo, a, b)
        T = O.schedule(topo, a, b)
        W, seed = sched.workers, 31
        rng = np.random.default_rng(5)
        g = rng.standard_normal((W, D)) * 1e-3
        gd = [torch.tensor(x, dtype=torch.float64, device=DEV) for x in g]
        ctx = mb.Context(D, sched, torch.float64, 0)
        comp = [torch.zeros(D, dtype=torch.float64, device=DEV) for _ in range(W)]
        comp_o = np.zeros((W, D))
        ctx.set_metrics(True)
        rates = []
        for t in range(1, 9):
            agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
            ctx.sign_round(t, ETA, seed, gd, comp, agg_bits=agg)
            rates.append(ctx.metrics().disagreement_rate)
            r = O.marsit_round(T, t, None, ETA, g, comp_o, seed)
            assert u64(agg).tolist() == r.agg_bits.tolist(), (topo, t)
            got = np.stack([c.cpu().numpy() for c in comp])
            assert np.array_equal(got, r.comp), (topo, t)
            comp_o = r.comp
        assert max(rates) > 0.5  # the drift the adaptive budget follows
        ctx.check()


@pytest.mark.parametrize("frac", ["0", "0.2", "2"])
def test_spread_round_coin_budgets_vs_oracle(frac, monkeypatch):
    """The spread round's own coins: computed in the launch when the buffer's
    (seed, round) tag misses (first round, a skipped or revisited round, a new seed),
    otherwise prefetched by the previous launch during its merge; budgets from
    the stream ends of the round before, anything beyond drawn inline (a
    Gaussian gradient with error feedback drives the disagreement above 1/2).
    Bit-exact against the oracle for fp64, ring 8 and torus 2x4."""
    monkeypatch.setenv("MARSIT_COIN_FRAC", frac)
    monkeypatch.setenv("MARSIT_SPREAD", "1")
    for topo, a, b in (("ring", 8, 0), ("torus", 2, 4)):
        D = 300_000
        sched = sched_of(topo, a, b)
        T = O.schedule(topo, a, b)
        W = sched.workers
        rng = np.random.default_rng(5)
        g = rng.standard_normal((W, D)) * 1e-3
        gd = [torch.tensor(x, dtype=torch.float64, device=DEV) for x in g]
        ctx = mb.Context(D, sched, torch.float64, 0)
        ctx.set_timing(True)
        comp = [torch.zeros(D, dtype=torch.float64, device=DEV) for _ in range(W)]
        comp_o = np.zeros((W, D))
        # skips, a revisit (3, 6, 4: round 6 misses and recomputes the buffer
        # round 4's prefetch had tagged) and a new seed
        rounds = [(31, t) for t in range(1, 7)] + [(31, 9), (31, 10), (31, 3), (31, 6), (31, 4),
                                                   (32, 11), (32, 12)]
        for seed, t in rounds:
            agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
            ctx.sign_round(t, ETA, seed, gd, comp, agg_bits=agg)
            r = O.marsit_round(T, t, None, ETA, g, comp_o, seed)
            assert u64(agg).tolist() == r.agg_bits.tolist(), (topo, seed, t)
            got = np.stack([c.cpu().numpy() for c in comp])
            assert np.array_equal(got, r.comp), (topo, seed, t)
            comp_o = r.comp
        ctx.check()
        assert ctx.timing()["spread_round"][1] == len(rounds)


def test_plain_c_program_round_trip():
    """build/sign_round_c (the C-ABI from plain C) runs 6 rounds, dense every
    4th, and checks c' = (g + c) - g_t bit for bit after every sign round."""
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "build", "sign_round_c")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools"), "sign_round_c"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "identity held exactly" in r.stdout
    assert r.stdout.count("dense") == 2 and r.stdout.count(" sign ") == 4


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("topo,a,b,D", [("ring", 4, 0, 1_000_000), ("ring", 8, 0, 262_142),
                                        ("torus", 2, 4, 60_224), ("ring", 16, 0, 640_000),
                                        ("torus", 3, 3, 36_036), ("ring", 2, 0, 8)])
@pytest.mark.parametrize("kernel", ["spread", "spread_nostash", "spread_tma", "cluster"])
def test_fused_small_round_vs_oracle(dtype, topo, a, b, D, kernel, monkeypatch):
    """Small one-GPU rounds run as ONE launch — over every SM with this
    round's coins inside (round_spread_kernel, the default) or one cluster per
    segment (round_cluster_kernel, MARSIT_SPREAD=0): bit-exact vs the oracle
    over carried rounds (value padding in the last segment when D % 4 != 0),
    the g_t output, and the same bits as the unfused kernels (MARSIT_FUSED=0)."""
    sched = sched_of(topo, a, b)
    T = O.schedule(topo, a, b)
    W, seed = sched.workers, 31
    monkeypatch.setenv("MARSIT_SPREAD", "0" if kernel == "cluster" else "1")
    monkeypatch.setenv("MARSIT_STASH", "0" if kernel == "spread_nostash" else "1")
    monkeypatch.setenv("MARSIT_SPREAD_TMA", "1" if kernel == "spread_tma" else "0")
    ctx = mb.Context(D, sched, dtype, 0)
    ctx.set_timing(True)
    monkeypatch.setenv("MARSIT_FUSED", "0")
    ref = mb.Context(D, sched, dtype, 0)
    comp = [torch.zeros(D, dtype=dtype, device=DEV) for _ in range(W)]
    comp_r = [torch.zeros(D, dtype=dtype, device=DEV) for _ in range(W)]
    comp_o = np.zeros((W, D))
    for t in (1, 2, 3, 5):
        g = np.stack([O.gen_correlated(seed, w, t, D) for w in range(W)])
        gd = [torch.tensor(x, dtype=dtype, device=DEV) for x in g]
        agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
        agg_r = torch.empty_like(agg)
        upd = torch.empty(D, dtype=dtype, device=DEV)
        ctx.sign_round(t, ETA, seed, gd, comp, agg_bits=agg, update=upd)
        ref.sign_round(t, ETA, seed, gd, comp_r, agg_bits=agg_r)
        r = O.marsit_round(T, t, None, ETA, g, comp_o, seed)
        assert u64(agg).tolist() == r.agg_bits.tolist(), (topo, t)
        assert torch.equal(agg, agg_r)
        assert np.array_equal(upd.double().cpu().numpy(), r.update)
        for w in range(W):
            assert torch.equal(comp[w], comp_r[w]), (t, w)
        comp_o = r.comp
    assert np.array_equal(np.stack([c.double().cpu().numpy() for c in comp]), comp_o)
    ctx.check()
    esize = 4 if dtype == torch.float32 else 8
    if W <= 16 and W * D * esize * 2 <= 96 << 20:
        ran = "fused_round" if kernel == "cluster" else "spread_round"
        assert ctx.timing()[ran][1] == 4  # the one-launch kernel ran every round


def test_spread_round_graph_replay_matches_eager():
    """The spread round keeps no host-side round state (its arrival count and
    generation live on the device and reset themselves), so rounds captured in
    a CUDA graph replay exactly: two replays of rounds t = 1, 2, 3 equal six
    eager rounds t = 1, 2, 3, 1, 2, 3 with the compensation carried."""
    W, D, seed = 4, 1_000_000, 7
    sched = mb.build_ring_schedule(W)
    g = [torch.empty(D, device=DEV) for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(g[w], 0, seed, w, 1)
    ctx, ref = mb.Context(D, sched, torch.float32, 0), mb.Context(D, sched, torch.float32, 0)
    comp = [torch.zeros(D, device=DEV) for _ in range(W)]
    comp_r = [torch.zeros(D, device=DEV) for _ in range(W)]
    agg = torch.zeros((D + 63) // 64, dtype=torch.int64, device=DEV)
    agg_r = torch.zeros_like(agg)
    warm = [torch.zeros(D, device=DEV) for _ in range(W)]
    ctx.sign_round(1, ETA, seed, g, warm)  # kernel attributes, coin tags settled outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for t in (1, 2, 3):
            ctx.sign_round(t, ETA, seed, g, comp, agg_bits=agg)
    for _ in range(2):
        graph.replay()
        for t in (1, 2, 3):
            ref.sign_round(t, ETA, seed, g, comp_r, agg_bits=agg_r)
        torch.cuda.synchronize()
        assert torch.equal(agg, agg_r)
        for w in range(W):
            assert torch.equal(comp[w], comp_r[w]), w
    ctx.check()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fused_round_zeros_negzero_subnormals_vs_oracle(dtype):
    """The fused small round (L % 4 == 0: D = 10,000, M = 5) on exact zeros,
    -0.0 + -0.0 (packs to 1, sign_vector.hpp:70), fp32 subnormals and their
    negatives: aggregate, g_t and compensation exactly the oracle's."""
    rng = np.random.default_rng(5)
    W, D, seed = 5, 10_000, 17
    sched = mb.build_ring_schedule(W)
    T = O.schedule("ring", W)
    g = rng.standard_normal((W, D)).astype(np.float32) * np.float32(1e-3)
    c = rng.standard_normal((W, D)).astype(np.float32) * np.float32(1e-3)
    g[:, ::5] = 0.0
    g[:, 1::5] = -0.0
    c[:, ::5] = 0.0
    c[:, 1::5] = -0.0
    g[:, 2::5] = np.float32(1e-45)
    c[:, 2::5] = 0.0
    g[:, 3::5] = np.float32(-1e-45)
    c[:, 3::5] = 0.0
    g64, c64 = g.astype(np.float64), c.astype(np.float64)
    ctx = mb.Context(D, sched, dtype, 0)
    ctx.set_timing(True)
    comp = [torch.tensor(x, dtype=dtype, device=DEV) for x in c64]
    agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
    upd = torch.empty(D, dtype=dtype, device=DEV)
    ctx.sign_round(1, ETA, seed, [torch.tensor(x, dtype=dtype, device=DEV) for x in g64], comp,
                   agg_bits=agg, update=upd)
    ctx.check()
    r = O.marsit_round(T, 1, None, ETA, g64, c64, seed)
    assert u64(agg).tolist() == r.agg_bits.tolist()
    assert np.array_equal(upd.double().cpu().numpy(), r.update)
    got = np.stack([x.double().cpu().numpy() for x in comp])
    if dtype == torch.float64:
        assert np.array_equal(got, r.comp)
    else:  # fp32 arithmetic: 1e-6 relative to the operands of c' = (g + c) - g_t
        bound = 1e-6 * (np.abs(r.comp) + np.abs(g64) + np.abs(c64) + ETA)
        assert np.all(np.abs(got - r.comp) <= bound)
    tm = ctx.timing()
    assert tm["fused_round"][1] + tm["spread_round"][1] == 1


def test_c3_cooperative_default_equals_grid_merge(monkeypatch):
    """C3 on one GPU (8 segments in one co-resident cooperative launch): the
    context picks the cooperative merge there (faster by a round's ~8 us) —
    its results equal the grid merge's (MARSIT_MERGE_KERNEL=grid) bit for bit
    over carried rounds, one merge launch per round each."""
    D, seed = 25_600_000, 2026
    sched = mb.build_ring_schedule(8)
    W = sched.workers
    auto = mb.Context(D, sched, torch.float32, 0)
    auto.set_timing(True)
    monkeypatch.setenv("MARSIT_MERGE_KERNEL", "grid")
    grid = mb.Context(D, sched, torch.float32, 0)
    grid.set_timing(True)
    monkeypatch.delenv("MARSIT_MERGE_KERNEL")
    g = [torch.empty(D, device=DEV) for _ in range(W)]
    c1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    c2 = [torch.zeros(D, device=DEV) for _ in range(W)]
    a1 = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
    a2 = torch.empty_like(a1)
    for t in (1, 2):
        for w in range(W):
            mb.fill_recipe(g[w], t % 2, seed, w, t)
        auto.sign_round(t, ETA, seed, g, c1, agg_bits=a1)
        grid.sign_round(t, ETA, seed, g, c2, agg_bits=a2)
        torch.cuda.synchronize()
        assert torch.equal(a1, a2), t
        for w in range(W):
            assert torch.equal(c1[w], c2[w]), (t, w)
    assert auto.timing()["merge"][1] == 2 and grid.timing()["merge"][1] == 2
    auto.check()
    grid.check()


@pytest.mark.slow
@pytest.mark.parametrize("topo,a,b,D", [("torus", 2, 4, 60_200_000), ("ring", 8, 0, 61_000_000)])
def test_large_segments_grid_merge_equals_cooperative(topo, a, b, D, monkeypatch):
    """C4 / C2 on one GPU: the segments are too large for one co-resident
    cooperative grid, so the context picks the grid merge (one launch); its
    aggregate and compensation equal the cooperative merge's (forced with
    MARSIT_MERGE_KERNEL=coop) bit for bit over carried rounds."""
    sched = sched_of(topo, a, b)
    W, seed = sched.workers, 2026
    auto = mb.Context(D, sched, torch.float32, 0)
    auto.set_timing(True)
    monkeypatch.setenv("MARSIT_MERGE_KERNEL", "coop")
    coop = mb.Context(D, sched, torch.float32, 0)
    monkeypatch.delenv("MARSIT_MERGE_KERNEL")
    g = [torch.empty(D, device=DEV) for _ in range(W)]
    c1 = [torch.zeros(D, device=DEV) for _ in range(W)]
    c2 = [torch.zeros(D, device=DEV) for _ in range(W)]
    a1 = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
    a2 = torch.empty_like(a1)
    for t in (1, 2):
        for w in range(W):
            mb.fill_recipe(g[w], t % 2, seed, w, t)
        auto.sign_round(t, ETA, seed, g, c1, agg_bits=a1)
        coop.sign_round(t, ETA, seed, g, c2, agg_bits=a2)
        torch.cuda.synchronize()
        assert torch.equal(a1, a2), t
        for w in range(W):
            assert torch.equal(c1[w], c2[w]), (t, w)
    assert auto.timing()["merge"][1] == 2  # one merge launch per round
    auto.check()
    coop.check()
