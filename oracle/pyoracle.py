"""ctypes front-end for the CHECKER libraries — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  It wraps:

* ``oracle/liboracle.so``          — the C restatement (marsit_oracle.c), and
* ``oracle/_ref/libmarsit_ref.so`` — the unmodified reference headers compiled
  in place (ref_driver.cpp); present only where it was built from
  /root/reference (it travels to the GPU box as a prebuilt file).

All arrays are numpy; schedules are flat tables (phase, send_to, recv_from,
segment) exactly like the product's C-ABI takes them.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmarsit_ref.so")

STATUS = {0: "ok", 1: "parameter_error", 2: "non_finite_error", 3: "protocol_error",
          4: "unsupported_error", 9: "other"}

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the checker libraries (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_stream_key.restype = C.c_uint64
        L.orc_stream_key.argtypes = [C.c_uint64] * 5
        L.orc_draw.restype = C.c_uint64
        L.orc_draw.argtypes = [C.c_uint64, C.c_uint64]
        for f in (L.orc_ring_schedule,):
            f.restype = C.c_int
            f.argtypes = [C.c_uint32, _u8p, _u32p, _u32p, _u32p]
        L.orc_torus_schedule.restype = C.c_int
        L.orc_torus_schedule.argtypes = [C.c_uint32, C.c_uint32, _u8p, _u32p, _u32p, _u32p]
        L.orc_pack_signs.restype = None
        L.orc_pack_signs.argtypes = [_f64p, C.c_size_t, _u64p]
        L.orc_merge_signs.restype = C.c_int
        L.orc_merge_signs.argtypes = [_u64p, C.c_uint32, _u64p, C.c_uint32, C.c_size_t,
                                      C.c_uint64, C.POINTER(C.c_uint64), _u64p]
        L.orc_allreduce_sign.restype = C.c_int
        L.orc_allreduce_sign.argtypes = [C.c_uint32, C.c_uint32, C.c_size_t, _u64p, C.c_uint32,
                                         _u8p, _u32p, _u32p, _u32p, C.c_uint64, C.c_uint64,
                                         _u64p, _u32p, _u64p, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64)]
        L.orc_allreduce_dense.restype = C.c_int
        L.orc_allreduce_dense.argtypes = [C.c_uint32, C.c_uint32, C.c_size_t, _f64p,
                                          C.c_uint32, _u8p, _u32p, _u32p, _u32p, _f64p, _u64p,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.orc_marsit_round.restype = C.c_int
        L.orc_marsit_round.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_double, C.c_uint32,
                                       C.c_uint32, C.c_size_t, _f64p, _f64p, C.c_uint32, _u8p,
                                       _u32p, _u32p, _u32p, C.c_uint64, _f64p, _f64p, _u64p,
                                       C.POINTER(C.c_int), _u64p, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]
        L.orc_gen_dyadic.restype = None
        L.orc_gen_dyadic.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, _f64p]
        L.orc_gen_correlated.restype = None
        L.orc_gen_correlated.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, _f64p]
        L.orc_last_sign_stats.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.orc_last_sign_stats.restype = None
        L.orc_ssdm_compress.restype = C.c_double
        L.orc_ssdm_compress.argtypes = [_f64p, C.c_size_t, C.c_uint64, _u64p]
        L.orc_ssdm_decompress.restype = None
        L.orc_ssdm_decompress.argtypes = [_u64p, C.c_size_t, C.c_double, _f64p]
        for f in (L.orc_cascading_allreduce, L.orc_sum_ssdm_allreduce):
            f.restype = C.c_int
        _ss = [C.c_uint32, C.c_uint32, C.c_size_t, _f64p, C.c_uint32, _u8p, _u32p, _u32p, _u32p,
               C.c_int, C.c_uint64, C.c_uint64, _f64p, _u64p, C.POINTER(C.c_uint64),
               C.POINTER(C.c_uint64)]
        L.orc_cascading_allreduce.argtypes = _ss
        L.orc_sum_ssdm_allreduce.argtypes = _ss + [_i64p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference compiled from its own headers (None when not built)."""
    global _ref
    if _ref is None:
        if not ref_available():
            return None
        R = C.CDLL(REF_SO)
        R.ref_build_schedule.restype = C.c_int
        R.ref_build_schedule.argtypes = [C.c_int, C.c_uint32, C.c_uint32, _u8p, _u32p, _u32p,
                                         _u32p]
        R.ref_stream_draws.restype = None
        R.ref_stream_draws.argtypes = [C.c_uint64] * 5 + [C.c_size_t, _u64p]
        R.ref_pack_signs.restype = C.c_int
        R.ref_pack_signs.argtypes = [_f64p, C.c_size_t, _u64p]
        R.ref_merge_signs.restype = C.c_int
        R.ref_merge_signs.argtypes = [_u64p, C.c_uint32, _u64p, C.c_uint32, C.c_size_t,
                                      C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                      C.c_uint64, _u64p, C.POINTER(C.c_uint64)]
        R.ref_allreduce_sign.restype = C.c_int
        R.ref_allreduce_sign.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_size_t, _u64p,
                                         C.c_uint64, C.c_uint64, _u64p, _u32p, _u64p,
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        R.ref_marsit_round.restype = C.c_int
        R.ref_marsit_round.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_double, C.c_int,
                                       C.c_uint32, C.c_uint32, C.c_size_t, _f64p, _f64p,
                                       C.c_uint64, _f64p, _f64p, _u64p, C.POINTER(C.c_int),
                                       _u64p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        R.ref_ssdm_compress.restype = C.c_int
        R.ref_ssdm_compress.argtypes = [_f64p, C.c_size_t] + [C.c_uint64] * 4 + [
            _u64p, C.POINTER(C.c_double)]
        R.ref_ssdm_allreduce.restype = C.c_int
        R.ref_ssdm_allreduce.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_size_t,
                                         _f64p, C.c_uint64, C.c_uint64, _f64p, _u64p,
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _i64p]
        R.ref_matching.restype = C.c_int
        R.ref_matching.argtypes = [_u64p, C.c_size_t, C.c_uint32, _f64p, _f64p,
                                   C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        R.ref_bench_create.restype = C.c_void_p
        R.ref_bench_create.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_size_t, C.c_uint64]
        R.ref_bench_round.restype = C.c_double
        R.ref_bench_round.argtypes = [C.c_void_p, C.c_uint64]
        R.ref_bench_destroy.restype = None
        R.ref_bench_destroy.argtypes = [C.c_void_p]
        _ref = R
    return _ref


# ----------------------------------------------------------------------------
# Schedules
# ----------------------------------------------------------------------------
@dataclass
class Tables:
    topology: int  # 0 ring, 1 torus
    a: int
    b: int
    workers: int
    segments: int
    phase: np.ndarray      # [steps] uint8 (0 reduce, 1 gather)
    send_to: np.ndarray    # [steps, workers] uint32
    recv_from: np.ndarray
    segment: np.ndarray

    @property
    def steps(self) -> int:
        return int(self.phase.shape[0])


def schedule(topology: str, a: int, b: int = 0, use_ref: bool = False) -> Tables:
    m = a if topology == "ring" else a * b
    n = max(2 * (m - 1), 1)
    ph = np.zeros(n, np.uint8)
    st = np.zeros(n * m, np.uint32)
    rf = np.zeros(n * m, np.uint32)
    sg = np.zeros(n * m, np.uint32)
    if use_ref:
        k = ref().ref_build_schedule(0 if topology == "ring" else 1, a, b, ph, st, rf, sg)
    elif topology == "ring":
        k = lib().orc_ring_schedule(a, ph, st, rf, sg)
    else:
        k = lib().orc_torus_schedule(a, b, ph, st, rf, sg)
    if k < 0:
        raise ValueError(STATUS[-k])
    return Tables(0 if topology == "ring" else 1, a, b, m, m, ph[:k].copy(),
                  st[:k * m].reshape(k, m).copy(), rf[:k * m].reshape(k, m).copy(),
                  sg[:k * m].reshape(k, m).copy())


def _flat(t: Tables):
    return (np.ascontiguousarray(t.phase), np.ascontiguousarray(t.send_to.ravel()),
            np.ascontiguousarray(t.recv_from.ravel()), np.ascontiguousarray(t.segment.ravel()))


# ----------------------------------------------------------------------------
# Primitives
# ----------------------------------------------------------------------------
def words64(n_bits: int) -> int:
    return (n_bits + 63) // 64


def stream_key(seed, purpose, w, t, s) -> int:
    return lib().orc_stream_key(seed, purpose, w, t, s)


def draw(key: int, n: int) -> int:
    return lib().orc_draw(key, n)


def pack_signs(v: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float64)
    out = np.zeros(max(words64(v.size), 1), np.uint64)
    lib().orc_pack_signs(v, v.size, out)
    return out[:words64(v.size)]


def merge_signs(recv, c_recv, local, c_local, length, key, used=0):
    out = np.zeros(max(words64(length), 1), np.uint64)
    u = C.c_uint64(used)
    rc = lib().orc_merge_signs(np.ascontiguousarray(recv, np.uint64), c_recv,
                               np.ascontiguousarray(local, np.uint64), c_local, length, key,
                               C.byref(u), out)
    if rc:
        raise RuntimeError(STATUS[rc])
    return out[:words64(length)], u.value


def gen_dyadic(seed, w, t, dim) -> np.ndarray:
    out = np.zeros(dim, np.float64)
    lib().orc_gen_dyadic(seed, w, t, dim, out)
    return out


def gen_correlated(seed, w, t, dim) -> np.ndarray:
    out = np.zeros(dim, np.float64)
    lib().orc_gen_correlated(seed, w, t, dim, out)
    return out


@dataclass
class SignResult:
    state: np.ndarray      # [workers, segments, words] uint64
    counts: np.ndarray     # [workers, segments] uint32
    bits_per_worker: np.ndarray
    reduce_bits: int
    gather_bits: int


def allreduce_sign(tables: Tables, signs: np.ndarray, seg_len: int, seed: int, rnd: int,
                   use_ref: bool = False) -> SignResult:
    W, S = tables.workers, tables.segments
    nw = words64(seg_len)
    signs = np.ascontiguousarray(signs, np.uint64).reshape(W * S * nw)
    state = np.zeros(W * S * nw + 1, np.uint64)
    counts = np.zeros(W * S, np.uint32)
    bpw = np.zeros(W, np.uint64)
    rb, gb = C.c_uint64(), C.c_uint64()
    if use_ref:
        rc = ref().ref_allreduce_sign(tables.topology, tables.a, tables.b, seg_len, signs, seed,
                                      rnd, state, counts, bpw, C.byref(rb), C.byref(gb))
    else:
        ph, st, rf, sg = _flat(tables)
        rc = lib().orc_allreduce_sign(W, S, seg_len, signs, tables.steps, ph, st, rf, sg, seed,
                                      rnd, state, counts, bpw, C.byref(rb), C.byref(gb))
    if rc:
        raise RuntimeError(STATUS[rc])
    return SignResult(state[:W * S * nw].reshape(W, S, nw), counts.reshape(W, S), bpw,
                      rb.value, gb.value)


@dataclass
class RoundResult:
    status: int
    update: np.ndarray
    comp: np.ndarray
    agg_bits: np.ndarray
    full_precision: bool
    bits_per_worker: np.ndarray
    reduce_bits: int
    gather_bits: int
    draws: int = 0    # coins drawn over all merges (sign rounds, oracle path)
    merges: int = 0   # merges evaluated


def marsit_round(tables: Tables, t: int, period, eta_s: float, grads: np.ndarray,
                 comp: np.ndarray, seed: int, use_ref: bool = False) -> RoundResult:
    """grads/comp: [workers, dim] float64.  period None = never."""
    W = tables.workers
    grads = np.ascontiguousarray(grads, np.float64)
    comp = np.ascontiguousarray(comp, np.float64)
    dim = grads.shape[1]
    upd = np.zeros(dim, np.float64)
    cout = np.zeros((W, dim), np.float64)
    agg = np.zeros(words64(dim) + 1, np.uint64)
    fp = C.c_int(0)
    bpw = np.zeros(W, np.uint64)
    rb, gb = C.c_uint64(), C.c_uint64()
    hp = 0 if period is None else 1
    K = 0 if period is None else int(period)
    if use_ref:
        rc = ref().ref_marsit_round(t, hp, K, eta_s, tables.topology, tables.a, tables.b, dim,
                                    grads.ravel(), comp.ravel(), seed, upd, cout.ravel(), agg,
                                    C.byref(fp), bpw, C.byref(rb), C.byref(gb))
    else:
        ph, st, rf, sg = _flat(tables)
        rc = lib().orc_marsit_round(t, hp, K, eta_s, W, tables.segments, dim, grads.ravel(),
                                    comp.ravel(), tables.steps, ph, st, rf, sg, seed, upd,
                                    cout.ravel(), agg, C.byref(fp), bpw, C.byref(rb),
                                    C.byref(gb))
    draws = merges = 0
    if not use_ref and not fp.value:
        d, m = C.c_uint64(), C.c_uint64()
        lib().orc_last_sign_stats(C.byref(d), C.byref(m))
        draws, merges = d.value, m.value
    return RoundResult(rc, upd, cout, agg[:words64(dim)], bool(fp.value), bpw, rb.value,
                       gb.value, draws, merges)


def matching_count(agg_bits: np.ndarray, grads: np.ndarray, comp: np.ndarray) -> int:
    """analysis.hpp:244-253 on the input mean of trainer.hpp:241-251: the number
    of coordinates whose aggregate bit equals (mean_w(g_w + c_w) >= 0), the mean
    summed in fp64 in worker order from 0.0 and divided by M."""
    grads = np.asarray(grads, np.float64)
    comp = np.asarray(comp, np.float64)
    W, dim = grads.shape
    mean = np.zeros(dim)
    for w in range(W):
        mean += grads[w] + comp[w]
    mean /= float(W)
    bits = np.unpackbits(np.ascontiguousarray(agg_bits, "<u8").view(np.uint8),
                         bitorder="little")[:dim].astype(bool)
    return int(np.count_nonzero(bits == (mean >= 0.0)))


def gen_metrics_inputs(seed: int, workers: int, dim: int):
    """fp32-valued (g, c) for the matching-rate fixtures: Gaussian values
    rounded to fp32, plus every 7th coordinate a cancellation case where
    fp32(g + c) loses the bits that decide the sign of the fp64 mean
    (worker 0: 1 + 2^-30, worker 1: -1 - 2^-29, the rest 0), so a mean formed
    from fp32-rounded u differs from trainer.hpp:241-251's fp64 add(g, c)."""
    rs = np.random.RandomState(seed)
    g = rs.standard_normal((workers, dim)).astype(np.float32).astype(np.float64) * 1e-3
    c = rs.standard_normal((workers, dim)).astype(np.float32).astype(np.float64) * 1e-3
    g = g.astype(np.float32).astype(np.float64)
    c = c.astype(np.float32).astype(np.float64)
    idx = np.arange(0, dim, 7)
    g[:, idx] = 0.0
    c[:, idx] = 0.0
    g[0, idx], c[0, idx] = 1.0, 2.0 ** -30
    g[1, idx], c[1, idx] = -1.0, -(2.0 ** -29)
    return g, c


def ref_matching(agg_bits: np.ndarray, grads: np.ndarray, comp: np.ndarray):
    """The REAL reference's matching figure (oracle/_ref: analysis.hpp:244-253
    on trainer.hpp:241-251's mean): (rate, count)."""
    grads = np.ascontiguousarray(grads, np.float64)
    comp = np.ascontiguousarray(comp, np.float64)
    W, dim = grads.shape
    words = np.ascontiguousarray(agg_bits, np.uint64)
    rate, cnt = C.c_double(), C.c_uint64()
    rc = ref().ref_matching(words, dim, W, grads.ravel(), comp.ravel(), C.byref(rate), C.byref(cnt))
    assert rc == 0, rc
    return rate.value, cnt.value


# ----------------------------------------------------------------------------
# SSDM baselines (ssdm.hpp:29-56, allreduce.hpp:198-339)
# ----------------------------------------------------------------------------
PURPOSE_SSDM = 4  # rng.hpp:18


def ssdm_compress(v: np.ndarray, seed: int, w: int, t: int, s: int, use_ref: bool = False):
    """(bits words, norm) of ssdm_compress(v, RngStream(seed, ssdm, w, t, s))."""
    v = np.ascontiguousarray(v, np.float64)
    bits = np.zeros(words64(len(v)) + 1, np.uint64)
    if use_ref:
        nrm = C.c_double()
        rc = ref().ref_ssdm_compress(v, len(v), seed, w, t, s, bits, C.byref(nrm))
        assert rc == 0
        return bits[:words64(len(v))], nrm.value
    key = stream_key(seed, PURPOSE_SSDM, w, t, s)
    nrm = lib().orc_ssdm_compress(v, len(v), key, bits)
    return bits[:words64(len(v))], nrm


def ssdm_decompress(bits: np.ndarray, length: int, norm: float) -> np.ndarray:
    out = np.zeros(length, np.float64)
    lib().orc_ssdm_decompress(np.ascontiguousarray(bits, np.uint64), length, norm, out)
    return out


@dataclass
class SsdmResult:
    status: int
    estimate: np.ndarray
    bits_per_worker: np.ndarray
    reduce_bits: int
    gather_bits: int
    max_abs_per_step: np.ndarray


def ssdm_allreduce(mode: str, tables: Tables, vectors: np.ndarray, seed: int, rnd: int,
                   use_ref: bool = False) -> SsdmResult:
    """mode 'cascading' (allreduce.hpp:205-262) or 'sum' (275-339)."""
    W = tables.workers
    vectors = np.ascontiguousarray(vectors, np.float64)
    dim = vectors.shape[1]
    out = np.zeros(dim, np.float64)
    bpw = np.zeros(W, np.uint64)
    rb, gb = C.c_uint64(), C.c_uint64()
    mx = np.zeros(max(tables.steps, 1), np.int64)
    m = 0 if mode == "cascading" else 1
    if use_ref:
        rc = ref().ref_ssdm_allreduce(m, tables.topology, tables.a, tables.b, dim, vectors.ravel(),
                                      seed, rnd, out, bpw, C.byref(rb), C.byref(gb), mx)
    else:
        ph, st, rf, sg = _flat(tables)
        args = (W, tables.segments, dim, vectors.ravel(), tables.steps, ph, st, rf, sg,
                int(tables.topology == 0), seed, rnd, out, bpw, C.byref(rb), C.byref(gb))
        rc = (lib().orc_cascading_allreduce(*args) if m == 0
              else lib().orc_sum_ssdm_allreduce(*args, mx))
    return SsdmResult(rc, out, bpw, rb.value, gb.value, mx[:tables.steps])


def fnv1a64(words: np.ndarray) -> int:
    """FNV-1a-64 over the little-endian bytes of u64 words (SURVEY §8c anchors)."""
    h = 0xcbf29ce484222325
    for byte in np.ascontiguousarray(words, "<u8").tobytes():
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h
