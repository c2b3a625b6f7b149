#!/usr/bin/env python3
"""Time sign rounds, dense rounds and driver steps on the BASELINE configs
(device time with CUDA events, inputs resident)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c3,c2,c4")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--dense", action="store_true")
ap.add_argument("--c5", action="store_true")
args = ap.parse_args()
CFG = {"c1": (1_000_000, "ring", 4, 0), "c2": (61_000_000, "ring", 8, 0),
       "c3": (25_600_000, "ring", 8, 0), "c4": (60_200_000, "torus", 2, 4)}


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


for name in args.configs.split(","):
    D, topo, a, b = CFG[name]
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    W = sched.workers
    ctx = mb.Context(D, sched, torch.float32, 0)
    g = [torch.empty(D, device="cuda") for _ in range(W)]
    for w in range(W):
        mb.fill_recipe(g[w], 0, 2026, w, 1)
    c = [torch.zeros(D, device="cuda") for _ in range(W)]
    state = {"t": 1}

    def sign():
        ctx.sign_round(state["t"], 2 ** -10, 2026, g, c)
        state["t"] += 1
    ms = timed(sign, args.iters)
    line = f"{name}: {topo} M={W} D={D}: sign round {ms*1e3:8.1f} us  {D/ms/1e6:7.2f} Gelem/s"
    if args.dense:
        mean = torch.empty(D, device="cuda")
        msd = timed(lambda: ctx.dense_round(0, g, c, mean), args.iters)
        line += f" | dense round {msd*1e3:8.1f} us"
    print(line, flush=True)
    del ctx, g, c
    torch.cuda.empty_cache()

if args.c5:
    D, W = 355_000_000, 8
    sched = mb.build_ring_schedule(W)
    for bucket in (0, 100_000_000):
        drv = mb.Driver(D, sched, eta_s=2 ** -10, global_seed=5, bucket_elems=bucket,
                        first_round=1)
        g = [torch.empty(D, device="cuda") for _ in range(W)]
        for w in range(W):
            mb.fill_recipe(g[w], 0, 5, w, 1)
        x = [torch.zeros(D, device="cuda") for _ in range(W)]
        ms = timed(lambda: drv.step(g, params=x), 3)
        print(f"c5: ring M=8 D=355M bucket={bucket}: driver step (+ replica update) "
              f"{ms:8.2f} ms  {D/ms/1e6:7.2f} Gelem/s", flush=True)
        del drv, g, x
        torch.cuda.empty_cache()
