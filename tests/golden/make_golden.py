#!/usr/bin/env python3
"""Generate tests/golden/*.json from the REAL reference (oracle/_ref/libmarsit_ref.so,
compiled in place from /root/reference/proj/include by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The GPU box never runs this; it only reads the committed JSON.

Doubles are stored as float.hex() strings, u64 words as 16-digit hex strings.
Inputs are either regenerated from a recipe ("dyadic"/"correlated", see
oracle/marsit_oracle.h — the recipe draws themselves are pinned in streams.json)
or stored explicitly ("explicit").
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as O  # noqa: E402

ETA = 2.0 ** -10


def hx(a):
    return [float(x).hex() for x in np.asarray(a, np.float64).ravel()]


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, "<f8").tobytes()).hexdigest()


def wx(a):
    return ["%016x" % int(x) for x in np.asarray(a, np.uint64).ravel()]


def inputs(recipe, seed, W, t, D, rng=None):
    if recipe == "dyadic":
        return np.stack([O.gen_dyadic(seed, w, t, D) for w in range(W)])
    if recipe == "correlated":
        return np.stack([O.gen_correlated(seed, w, t, D) for w in range(W)])
    raise ValueError(recipe)


def special_values(g, rng):
    """Sprinkle exact zeros, negative zeros and tiny values (fp32 subnormal range)."""
    g = g.copy()
    flat = g.ravel()
    n = flat.size
    idx = rng.choice(n, size=max(1, n // 16), replace=False)
    for k, i in enumerate(idx):
        flat[i] = [0.0, -0.0, 1e-40, -1e-40, 2.0 ** -149, -(2.0 ** -149)][k % 6]
    return g


def round_cases():
    rng = np.random.default_rng(7)
    cases = []
    specs = [
        # (topology, a, b, D, recipe, rounds, period, seed)
        ("ring", 2, 0, 2, "unanimous", 1, None, 42),
        ("ring", 5, 0, 37, "dyadic", 4, None, 2026),
        ("ring", 3, 0, 1, "dyadic", 2, None, 11),
        ("ring", 4, 0, 3, "dyadic", 2, None, 12),
        ("ring", 4, 0, 130, "dyadic", 3, None, 13),
        ("ring", 8, 0, 1000, "dyadic", 3, None, 14),
        ("ring", 8, 0, 1000, "correlated", 2, None, 15),
        ("ring", 6, 0, 1031, "special", 2, None, 16),
        ("ring", 16, 0, 3001, "dyadic", 2, None, 17),
        ("torus", 2, 3, 97, "dyadic", 3, None, 18),
        ("torus", 2, 4, 100, "dyadic", 2, None, 2026),
        ("torus", 3, 3, 500, "dyadic", 2, None, 19),
        ("torus", 4, 2, 257, "gaussian", 2, None, 20),
        ("ring", 4, 0, 77, "gaussian", 5, 3, 21),      # dense rounds at t=0,3
        ("torus", 2, 3, 61, "dyadic", 4, 2, 22),       # dense rounds at t=0,2
        ("ring", 7, 0, 2048 + 5, "dyadic", 2, None, 23),
    ]
    for topo, a, b, D, recipe, rounds, period, seed in specs:
        T = O.schedule(topo, a, b, use_ref=True)
        W = T.workers
        comp = np.zeros((W, D))
        case = dict(topology=topo, a=a, b=b, dim=D, recipe=recipe, period=period, seed=seed,
                    eta_s=ETA if recipe != "unanimous" else 0.1, rounds=[])
        t0 = 0 if period is not None else 1
        for t in range(t0, t0 + rounds):
            if recipe == "unanimous":
                g = np.array([[0.4, -0.2], [0.4, -0.2]])
            elif recipe == "gaussian":
                g = rng.standard_normal((W, D)) * 1e-3
            elif recipe == "special":
                g = special_values(inputs("dyadic", seed, W, t, D), rng)
            else:
                g = inputs(recipe, seed, W, t, D)
            r = O.marsit_round(T, t, period, case["eta_s"], g, comp, seed, use_ref=True)
            assert r.status == 0, (topo, a, b, D, t, r.status)
            rec = dict(t=t, full_precision=r.full_precision,
                       bits_per_worker=[int(x) for x in r.bits_per_worker],
                       reduce_bits=r.reduce_bits, gather_bits=r.gather_bits)
            if W * D <= 4000:
                rec["update"] = hx(r.update)
                rec["comp"] = hx(r.comp)
            else:  # large: digests of the little-endian float64 bytes
                rec["update_sha256"] = sha(r.update)
                rec["comp_sha256"] = sha(r.comp)
                rec["comp_head"] = hx(r.comp[:, :8])
            if recipe in ("gaussian", "special", "unanimous"):
                rec["grads"] = hx(g)
            if not r.full_precision:
                rec["agg_bits"] = wx(r.agg_bits)
            case["rounds"].append(rec)
            comp = r.comp
        cases.append(case)
    return cases


def anchors():
    """SURVEY §8c known-answer table, recomputed with the reference."""
    out = []
    for topo, a, b, D, rounds in [("ring", 5, 0, 37, 2), ("torus", 2, 4, 100, 1),
                                  ("ring", 4, 0, 1_000_000, 3)]:
        T = O.schedule(topo, a, b, use_ref=True)
        comp = np.zeros((T.workers, D))
        for t in range(1, rounds + 1):
            g = inputs("dyadic", 2026, T.workers, t, D)
            r = O.marsit_round(T, t, None, ETA, g, comp, 2026, use_ref=True)
            assert r.status == 0
            comp = r.comp
            out.append(dict(topology=topo, a=a, b=b, dim=D, t=t,
                            popcount=int(sum(bin(int(x)).count("1") for x in r.agg_bits)),
                            fnv1a64="%016x" % O.fnv1a64(r.agg_bits),
                            word0="%016x" % int(r.agg_bits[0]),
                            words_head=wx(r.agg_bits[:4]),
                            sum_c0=float(comp[0].sum()).hex(), c00=float(comp[0][0]).hex()))
    return out


def streams():
    R = O.ref()
    out = []
    for seed, purpose, w, t, s in [(2026, 5, 0, 1, 0), (2026, 5, 7, 3, 5), (42, 5, 0, 0, 0),
                                   (2026, 6, 3, 1, 0), (0, 6, 0xFFFF, 9, 0),
                                   (2**64 - 1, 5, 2**32, 2**40, 17)]:
        d = np.zeros(16, np.uint64)
        R.ref_stream_draws(seed, purpose, w, t, s, 16, d)
        out.append(dict(seed="%x" % seed, purpose=purpose, w="%x" % w, t="%x" % t, s="%x" % s,
                        draws=wx(d)))
    return out


def merges():
    import ctypes as C
    R = O.ref()
    rng = np.random.default_rng(99)
    out = []
    for length, cr, cl, skip in [(1, 1, 1, 0), (64, 1, 1, 0), (65, 2, 1, 3), (200, 3, 1, 0),
                                 (1000, 7, 1, 11), (4096, 4, 4, 0), (333, 1, 15, 5),
                                 (4099, 5, 3, 100)]:
        nw = O.words64(length)
        r = rng.integers(0, 2**63, size=nw, dtype=np.uint64) * 2 + rng.integers(0, 2, size=nw, dtype=np.uint64)
        l = rng.integers(0, 2**63, size=nw, dtype=np.uint64) * 2 + rng.integers(0, 2, size=nw, dtype=np.uint64)
        if length % 64:
            mask = np.uint64((1 << (length % 64)) - 1)
            r[-1] &= mask
            l[-1] &= mask
        o = np.zeros(nw, np.uint64)
        used = C.c_uint64()
        seed, w, t, s = 77, 3, 5, 2
        rc = R.ref_merge_signs(r, cr, l, cl, length, seed, w, t, s, skip, o, C.byref(used))
        assert rc == 0
        out.append(dict(length=length, c_recv=cr, c_local=cl, seed=seed, w=w, t=t, s=s,
                        skip=skip, recv=wx(r), local=wx(l), out=wx(o), consumed=used.value))
    return out


def allreduces():
    rng = np.random.default_rng(5)
    out = []
    for topo, a, b, L, rounds in [("ring", 6, 0, 17, 3), ("torus", 2, 3, 17, 3),
                                  ("ring", 9, 0, 70, 2), ("torus", 3, 3, 70, 2),
                                  ("torus", 4, 2, 129, 2), ("ring", 2, 0, 64, 2)]:
        T = O.schedule(topo, a, b, use_ref=True)
        nw = O.words64(L)
        for rnd in range(rounds):
            signs = rng.integers(0, 2**63, size=(T.workers, T.segments, nw), dtype=np.uint64)
            signs = signs * 2 + rng.integers(0, 2, size=signs.shape, dtype=np.uint64)
            if L % 64:
                signs[..., -1] &= np.uint64((1 << (L % 64)) - 1)
            res = O.allreduce_sign(T, signs, L, 1234, rnd, use_ref=True)
            out.append(dict(topology=topo, a=a, b=b, seg_len=L, seed=1234, round=rnd,
                            signs=wx(signs), state=wx(res.state),
                            counts=[int(x) for x in res.counts.ravel()],
                            bits_per_worker=[int(x) for x in res.bits_per_worker],
                            reduce_bits=res.reduce_bits, gather_bits=res.gather_bits))
    return out


def ssdm_cases():
    """ssdm_compress (ssdm.hpp:29-40) and the two baseline all-reduces
    (allreduce.hpp:205-262, 275-339) from the reference."""
    rng = np.random.default_rng(11)
    comp, allr = [], []
    for n, kind in [(1, "gauss"), (21, "gauss"), (64, "gauss"), (100, "dyadic"), (130, "zero"),
                    (33, "onehot")]:
        if kind == "gauss":
            v = rng.standard_normal(n)
        elif kind == "dyadic":
            v = O.gen_dyadic(3, 0, 1, n)
        elif kind == "zero":
            v = np.zeros(n)
        else:
            v = np.zeros(n)
            v[n // 2] = 2.5
        bits, norm = O.ssdm_compress(v, 77, 2, 5, 1, use_ref=True)
        comp.append(dict(v=hx(v), seed=77, worker=2, round=5, segment=1, bits=wx(bits),
                         norm=float(norm).hex()))
    for mode in ("cascading", "sum"):
        for a, D, recipe in [(4, 21, "gauss"), (5, 40, "gauss"), (3, 3, "dyadic"),
                             (8, 1001, "dyadic"), (6, 5, "gauss"), (4, 4096, "dyadic"),
                             (2, 7, "gauss")]:
            T = O.schedule("ring", a, 0, use_ref=True)
            if recipe == "dyadic":
                v = inputs("dyadic", 2026, a, 3, D)
                vec = None
            else:
                v = rng.standard_normal((a, D))
                vec = hx(v)
            r = O.ssdm_allreduce(mode, T, v, 2026, 3, use_ref=True)
            assert r.status == 0
            allr.append(dict(mode=mode, a=a, dim=D, recipe=recipe, vectors=vec, seed=2026,
                             round=3, estimate=hx(r.estimate),
                             bits_per_worker=[int(x) for x in r.bits_per_worker],
                             reduce_bits=r.reduce_bits, gather_bits=r.gather_bits,
                             max_abs_per_step=[int(x) for x in r.max_abs_per_step]))
    return dict(compress=comp, allreduce=allr)


def metrics_cases():
    """The trainer's matching figure (analysis.hpp:244-253 on trainer.hpp:241-251's
    fp64 mean of add(g, c)) from the REAL reference, on fp32-valued inputs with
    cancellation coordinates (O.gen_metrics_inputs): one sign round each."""
    out = []
    for topo, a, b, D, seed in [("ring", 4, 0, 4_099, 11), ("torus", 2, 4, 60_211, 12),
                                ("ring", 8, 0, 100_003, 13)]:
        T = O.schedule(topo, a, b)
        g, c = O.gen_metrics_inputs(seed, T.workers, D)
        r = O.marsit_round(T, 1, None, ETA, g, c, 2026, use_ref=True)
        assert r.status == 0
        rate, matches = O.ref_matching(r.agg_bits, g, c)
        # what a mean of fp32-rounded u would give (the pre-fix device figure)
        u32 = (g.astype(np.float32) + c.astype(np.float32)).astype(np.float64)
        m32 = O.matching_count(r.agg_bits, u32, np.zeros_like(u32))
        out.append({"topology": topo, "a": a, "b": b, "dim": D, "seed": seed, "round": 1,
                    "global_seed": 2026, "inputs_sha256": sha(np.concatenate([g, c])),
                    "agg_words": wx(r.agg_bits), "matches": int(matches), "rate": float(rate).hex(),
                    "matches_fp32_mean": int(m32)})
    return out


def schedules():
    out = []
    for topo, a, b in [("ring", 2, 0), ("ring", 3, 0), ("ring", 8, 0), ("torus", 2, 2),
                       ("torus", 2, 3), ("torus", 2, 4), ("torus", 3, 3), ("torus", 4, 2)]:
        T = O.schedule(topo, a, b, use_ref=True)
        out.append(dict(topology=topo, a=a, b=b, phase=[int(x) for x in T.phase],
                        send_to=T.send_to.tolist(), recv_from=T.recv_from.tolist(),
                        segment=T.segment.tolist()))
    return out


def main():
    if not O.ref_available():
        O.build()
    assert O.ref_available(), "oracle/_ref/libmarsit_ref.so not built (needs /root/reference)"
    makers = dict(anchors=anchors, streams=streams, merges=merges, allreduce=allreduces,
                  schedules=schedules, rounds=round_cases, ssdm=ssdm_cases, metrics=metrics_cases)
    names = sys.argv[1:] or list(makers)  # e.g. `make_golden.py metrics`
    blobs = {n: makers[n]() for n in names}
    for name, obj in blobs.items():
        with open(os.path.join(HERE, name + ".json"), "w") as f:
            json.dump(obj, f, separators=(",", ":"))
        print(name, os.path.getsize(os.path.join(HERE, name + ".json")), "bytes")


if __name__ == "__main__":
    main()
