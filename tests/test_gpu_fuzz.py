"""Randomised GPU-vs-oracle rounds (the oracle is pinned to the reference in
tests/test_oracle.py): ring M in [2, 16], torus up to 4x4, D from 1 to a few
thousand incl. D < M and 64-bit word boundaries, fp64 Gaussian inputs with
zeros / -0.0 / subnormals, fp32 dyadic (fp32-exact) inputs, dense cadence,
compensation carried over 3 rounds.  Bit-exact: aggregate bits, update and
compensation."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2204_06787_b200 as mb  # noqa: E402
import pyoracle as O  # noqa: E402

DEV = "cuda:0"


def draw_case(seed):
    rng = np.random.default_rng(seed)
    if rng.random() < 0.6:
        topo, a, b = "ring", int(rng.integers(2, 17)), 0
        M = a
    else:
        topo, a, b = "torus", int(rng.integers(2, 5)), int(rng.integers(2, 5))
        M = a * b
    D = int(rng.choice([1, max(1, M - 1), M, M + 1, 64 * M - 1, 64 * M + 1,
                        int(rng.integers(1, 5000))]))
    f64 = bool(rng.random() < 0.5)
    period = None if rng.random() < 0.5 else int(rng.integers(2, 4))
    eta = float(2.0 ** -int(rng.integers(6, 12)))
    return rng, topo, a, b, M, D, f64, period, eta


def inputs(rng, f64, M, D, seed, t):
    if not f64:
        return np.stack([O.gen_dyadic(seed, w, t, D) for w in range(M)])
    g = rng.standard_normal((M, D)) * 1e-3
    flat = g.ravel()
    k = max(1, flat.size // 20)
    idx = rng.choice(flat.size, size=k, replace=False)
    flat[idx[: k // 3]] = 0.0
    flat[idx[k // 3: 2 * k // 3]] = -0.0
    flat[idx[2 * k // 3:]] = 1e-310 * np.sign(rng.standard_normal(len(idx) - 2 * k // 3))
    return g


# MARSIT_FUZZ_CASES widens the sweep (e.g. 1000 for a soak run on the GPU box)
@pytest.mark.parametrize("case", range(int(os.environ.get("MARSIT_FUZZ_CASES", "32"))))
def test_fuzz_rounds_vs_oracle(case):
    rng, topo, a, b, M, D, f64, period, eta = draw_case(7000 + case)
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    T = O.schedule(topo, a, b)
    dtype = torch.float64 if f64 else torch.float32
    ctx = mb.Context(D, sched, dtype, 0)
    seed = 100 + case
    comp_o = np.zeros((M, D))
    comp = [torch.zeros(D, dtype=dtype, device=DEV) for _ in range(M)]
    key = (topo, a, b, D, f64, period)
    for t in range(1, 4):
        g = inputs(rng, f64, M, D, seed, t)
        r = O.marsit_round(T, t, period, eta, g, comp_o, seed)
        assert r.status == 0, key
        gd = [torch.tensor(x, dtype=dtype, device=DEV) for x in g]
        upd = torch.empty(D, dtype=dtype, device=DEV)
        if r.full_precision:
            ctx.dense_round(t, gd, comp, upd)
            torch.cuda.synchronize()
            want = r.update
            got = upd.double().cpu().numpy()
            if f64:
                assert np.array_equal(got, want), key
            else:  # the fp32 mean of dyadic inputs is the fp64 mean rounded once
                assert np.array_equal(got, want.astype(np.float32).astype(np.float64)), key
        else:
            agg = torch.empty((D + 63) // 64, dtype=torch.int64, device=DEV)
            ctx.sign_round(t, eta, seed, gd, comp, agg_bits=agg, update=upd)
            torch.cuda.synchronize()
            assert agg.cpu().numpy().view(np.uint64).tolist() == r.agg_bits.tolist(), key
            assert np.array_equal(upd.double().cpu().numpy(), r.update), key
        got_c = np.stack([c.double().cpu().numpy() for c in comp])
        assert np.array_equal(got_c, r.comp), key
        comp_o = r.comp
    ctx.check()
