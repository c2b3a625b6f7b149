"""SSDM baseline collectives on the device against the
reference's golden fixtures (tests/golden/ssdm.json) and the oracle
(oracle/marsit_oracle.c, pinned to the reference in tests/test_oracle.py).

Bits, packet words, BitsAccount and max |sum| per step: exact.  Values: the
l2 norm is summed in a fixed parallel order instead of the reference's
sequential one, so it is exact whenever the sum of squares is (dyadic
recipe inputs: every first-hop norm) and within a few ulps otherwise; the
tolerance is stated per assertion."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2204_06787_b200 as mb  # noqa: E402
import pyoracle as O  # noqa: E402
from conftest import load_golden  # noqa: E402

DEV = "cuda:0"
REL = 1e-12  # relative tolerance for norms summed in a different order


def rel_tol(L, hops):
    """The reference sums the L squares sequentially: its own rounding error is
    up to ~L * 2^-53 relative per norm, compounded over the chain's hops."""
    return max(REL, 2.0 * hops * L * 2.0 ** -53)


def fx(lst):
    return np.array([float.fromhex(x) for x in lst], np.float64)


def wx(lst):
    return np.array([int(x, 16) for x in lst], np.uint64)


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def case_inputs(case):
    if case["vectors"] is not None:
        return fx(case["vectors"]).reshape(case["a"], case["dim"])
    return np.stack([O.gen_dyadic(case["seed"], w, case["round"], case["dim"])
                     for w in range(case["a"])])


def test_ssdm_compress_matches_reference_golden():
    for case in load_golden("ssdm")["compress"]:
        v = fx(case["v"])
        pk = mb.ssdm_compress(torch.tensor(v, device=DEV), case["seed"], case["worker"],
                              case["round"], case["segment"])
        want_norm = float.fromhex(case["norm"])
        assert u64(pk.bits).tolist() == wx(case["bits"]).tolist()
        assert pk.norm == pytest.approx(want_norm, rel=REL, abs=0)
        dec = mb.ssdm_decompress(pk).cpu().numpy()
        assert np.array_equal(dec, O.ssdm_decompress(u64(pk.bits), len(v), pk.norm))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_ssdm_allreduce_matches_reference_golden(dtype):
    for case in load_golden("ssdm")["allreduce"]:
        v = case_inputs(case)
        exact_in = case["recipe"] == "dyadic"
        if dtype == torch.float32 and not exact_in:
            continue  # Gaussian doubles are not fp32-representable
        sched = mb.build_ring_schedule(case["a"])
        vecs = [torch.tensor(x, dtype=dtype, device=DEV) for x in v]
        fn = mb.cascading_allreduce if case["mode"] == "cascading" else mb.sum_ssdm_allreduce
        res = fn(vecs, sched, case["seed"], case["round"])
        got = res.per_worker[0].double().cpu().numpy()
        want = fx(case["estimate"])
        if dtype == torch.float32:
            want = want.astype(np.float32).astype(np.float64)
        key = (case["mode"], case["a"], case["dim"], case["recipe"])
        if case["mode"] == "sum" and exact_in:
            # every norm is a first compression of dyadic inputs: exact sums
            assert np.array_equal(got, want), key
        else:
            # same signs everywhere, magnitudes within REL (norm summation order)
            assert np.array_equal(np.signbit(got), np.signbit(want)), key
            np.testing.assert_allclose(got, want, rtol=REL, atol=0, err_msg=str(key))
        assert res.bits.per_worker == case["bits_per_worker"], key
        assert (res.bits.reduce_bits, res.bits.gather_bits) == (case["reduce_bits"],
                                                               case["gather_bits"]), key
        if case["mode"] == "sum":
            assert res.max_abs_per_step == case["max_abs_per_step"], key


@pytest.mark.parametrize("mode", ["cascading", "sum"])
@pytest.mark.parametrize("M,D", [(8, 4_000_000), (5, 1_000_003)])
def test_ssdm_allreduce_large_vs_oracle(mode, M, D):
    """Sizes far beyond the fixtures (multi-CTA norms, ragged tails)."""
    seed, rnd = 2026, 4
    v = np.stack([O.gen_dyadic(seed, w, rnd, D) for w in range(M)])
    T = O.schedule("ring", M)
    want = O.ssdm_allreduce(mode, T, v, seed, rnd)
    assert want.status == 0
    sched = mb.build_ring_schedule(M)
    vecs = [torch.tensor(x, device=DEV) for x in v]
    fn = mb.cascading_allreduce if mode == "cascading" else mb.sum_ssdm_allreduce
    res = fn(vecs, sched, seed, rnd)
    got = res.per_worker[0].cpu().numpy()
    if mode == "sum":
        assert np.array_equal(got, want.estimate)
        assert res.max_abs_per_step == want.max_abs_per_step.tolist()
    else:
        assert np.array_equal(np.signbit(got), np.signbit(want.estimate))
        np.testing.assert_allclose(got, want.estimate, rtol=rel_tol(-(-D // M), M), atol=0)
    assert res.bits.per_worker == want.bits_per_worker.tolist()
    assert (res.bits.reduce_bits, res.bits.gather_bits) == (want.reduce_bits, want.gather_bits)


def test_ssdm_zero_and_one_hot_vectors():
    # allreduce.hpp / test_collective.cpp:264-278: unanimous one-hot inputs decode exactly
    sched = mb.build_ring_schedule(3)
    v = torch.tensor([0.0, 2.0, 0.0], dtype=torch.float64, device=DEV)
    res = mb.sum_ssdm_allreduce([v, v, v], sched, 11, 0)
    est = res.per_worker[0].cpu().numpy()
    assert est[0] == 0.0 and est[2] == 0.0 and est[1] == pytest.approx(2.0, rel=1e-12)
    z = torch.zeros(50, dtype=torch.float64, device=DEV)
    for fn in (mb.cascading_allreduce, mb.sum_ssdm_allreduce):
        r = fn([z] * 3, sched, 1, 1)
        assert bool((r.per_worker[0] == 0).all())  # zero norm decodes to zero
    pk = mb.ssdm_compress(z, 5, 0, 0, 0)
    assert pk.norm == 0.0 and bool((mb.ssdm_decompress(pk) == 0).all())


def test_ssdm_errors():
    v = [torch.ones(10, dtype=torch.float64, device=DEV) for _ in range(4)]
    with pytest.raises(mb.UnsupportedError):
        mb.cascading_allreduce(v, mb.build_torus_schedule(2, 2), 1, 1)
    with pytest.raises(mb.UnsupportedError):
        mb.sum_ssdm_allreduce(v, mb.build_torus_schedule(2, 2), 1, 1)
    with pytest.raises(mb.ParameterError):
        mb.sum_ssdm_allreduce(v[:3], mb.build_ring_schedule(4), 1, 1)
    bad = [x.clone() for x in v]
    bad[2][3] = float("nan")
    with pytest.raises(mb.NonFiniteError):
        mb.sum_ssdm_allreduce(bad, mb.build_ring_schedule(4), 1, 1)
    ctx = mb.Context(10, mb.build_ring_schedule(4), torch.float64, 0, nranks=2, rank=0,
                     external_transport=True)
    import ctypes as C
    st = mb._native.lib().marsit_ssdm_allreduce(
        ctx._h, 1, 1, 1, mb._native.ptr_array([x.data_ptr() for x in v[:2]]),
        C.c_void_p(v[0].data_ptr()), None, None, None, None, mb._stream_ptr(0))
    assert st == 4  # MARSIT_EUNSUPPORTED: every worker must be on the context
