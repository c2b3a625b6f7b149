#!/usr/bin/env python3
"""Small rounds over every kernel family (ring / torus, ragged / aligned,
fp32 / fp64, dense, metrics, driver with replica update, SSDM), each
followed by the context's error-latch check: a quick whole-library smoke
on the GPU (compute-sanitizer is not available on the GPU pool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

ETA = 2.0 ** -10
for topo, a, b, D, dt in (("ring", 8, 0, 40_960, torch.float32), ("ring", 5, 0, 10_007, torch.float64),
                          ("torus", 2, 4, 32_768, torch.float32), ("torus", 3, 3, 9_001, torch.float32),
                          ("ring", 4, 0, 3, torch.float32)):
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    W = sched.workers
    ctx = mb.Context(D, sched, dt, 0)
    g = [torch.randn(D, device="cuda", dtype=dt) * 1e-3 for _ in range(W)]
    c = [torch.zeros(D, device="cuda", dtype=dt) for _ in range(W)]
    agg = torch.empty((D + 63) // 64, dtype=torch.int64, device="cuda")
    upd = torch.empty(D, device="cuda", dtype=dt)
    for t in range(1, 4):
        ctx.set_metrics(t == 2)
        ctx.sign_round(t, ETA, 7, g, c, agg_bits=agg, update=upd)
    mean = torch.empty(D, device="cuda", dtype=dt)
    ctx.dense_round(4, g, c, mean)
    torch.cuda.synchronize()
    ctx.check()
    drv = mb.Driver(D, sched, eta_s=ETA, global_seed=3, period=3, bucket_elems=max(D // 3, 1),
                    dtype=dt, first_round=1)
    x = [torch.zeros(D, device="cuda", dtype=dt) for _ in range(W)]
    for _ in range(4):
        drv.step(g, params=x)
    torch.cuda.synchronize()
    print("ok", topo, a, b, D, dt, flush=True)
if True:
    sched = mb.build_ring_schedule(4)
    v = [torch.randn(5000, device="cuda", dtype=torch.float64) for _ in range(4)]
    mb.cascading_allreduce(v, sched, 1, 1)
    mb.sum_ssdm_allreduce(v, sched, 1, 1)
    torch.cuda.synchronize()
    print("ok ssdm", flush=True)
