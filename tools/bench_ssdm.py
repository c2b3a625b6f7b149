#!/usr/bin/env python3
"""SSDM baselines at C3 (ring M=8, D=25.6M) on the device vs the reference's
own CPU implementation (oracle/_ref, when built) on a D/10 sample."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2204_06787_b200 as mb  # noqa: E402

D, M, seed = 25_600_000, 8, 2026
sched = mb.build_ring_schedule(M)
vecs = [torch.empty(D, device="cuda") for _ in range(M)]
for w in range(M):
    mb.fill_recipe(vecs[w], 0, seed, w, 1)
for name, fn in (("cascading", mb.cascading_allreduce), ("sum", mb.sum_ssdm_allreduce)):
    for t in range(3):
        fn(vecs, sched, seed, t)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    a.record()
    for t in range(n):
        fn(vecs, sched, seed, t)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    print(f"{name}: {ms * 1e3:.0f} us per all-reduce (D={D}, M={M}, fp32, incl. host bits "
          f"accounting), {D / ms / 1e6:.2f} Gelem/s")
try:
    import pyoracle as O
    if O.ref_available():
        Ds = D // 10
        v = np.stack([O.gen_dyadic(seed, w, 1, Ds) for w in range(M)])
        T = O.schedule("ring", M)
        for mode in ("cascading", "sum"):
            t0 = time.perf_counter()
            r = O.ssdm_allreduce(mode, T, v, seed, 1, use_ref=True)
            dt = time.perf_counter() - t0
            print(f"reference CPU {mode}: {dt * 1e3:.0f} ms for D={Ds} (1 thread), "
                  f"{Ds / dt / 1e9:.4f} Gelem/s")
except Exception as e:  # pragma: no cover
    print("reference CPU timing skipped:", e)
