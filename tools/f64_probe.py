#!/usr/bin/env python3
"""fp64 sign rounds (the drop-in's default instantiation) at C3 / C4 sizes:
round time against the 40.25 B/worker-element floor, per-phase times, and
the same Gaussian data through an fp32 context for comparison."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

PEAK = 6548.2


def timed(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


for D, topo, A, B in ((25_600_000, "ring", 8, 0), (60_200_000, "torus", 2, 4)):
    s = mb.build_ring_schedule(A) if topo == "ring" else mb.build_torus_schedule(A, B)
    M = s.workers
    for dt, eb in ((torch.float64, 8), (torch.float32, 4)):
        ctx = mb.Context(D, s, dt, 0)
        gen = torch.Generator(device="cuda").manual_seed(1)
        g = [(torch.randn(D, device="cuda", generator=gen, dtype=torch.float64) * 1e-3).to(dt)
             for _ in range(M)]
        c = [torch.zeros(D, device="cuda", dtype=dt) for _ in range(M)]
        st = {"t": 1}

        def r():
            ctx.sign_round(st["t"], 2 ** -10, 5, g, c)
            st["t"] += 1

        us = timed(r)
        floor = (2 * eb + 0.125 + 2 * eb + eb + 0.125) * M * D / PEAK / 1e3
        ctx.set_timing(True)
        ctx.timing(reset=True)
        for _ in range(5):
            r()
        torch.cuda.synchronize()
        ph = {k: round(v[0] / 5 * 1e3, 1) for k, v in ctx.timing(reset=True).items() if v[1]}
        print(json.dumps({"D": D, "topo": topo, "dtype": str(dt), "sign_round_us": round(us, 1),
                          "floor_us": round(floor, 1), "frac": round(floor / us, 3),
                          "phases_us": ph}), flush=True)
        del ctx, g, c
        torch.cuda.empty_cache()
