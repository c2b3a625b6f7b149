#!/usr/bin/env python3
"""Cost of the fused round metrics at C3 (ring M=8, D=25.6M, fp32): sign
round and decode-phase times with and without marsit_ctx_set_metrics."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

D, W, seed, eta = 25_600_000, 8, 2026, 2.0 ** -10
sched = mb.build_ring_schedule(W)
g = [torch.empty(D, device="cuda") for _ in range(W)]
for w in range(W):
    mb.fill_recipe(g[w], 0, seed, w, 1)
for on in (False, True, False, True):
    ctx = mb.Context(D, sched, torch.float32, 0)
    ctx.set_metrics(on)
    c = [torch.zeros(D, device="cuda") for _ in range(W)]
    for t in range(1, 6):
        ctx.sign_round(t, eta, seed, g, c)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.timing(reset=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for t in range(6, 6 + n):
        ctx.sign_round(t, eta, seed, g, c)
    b.record()
    torch.cuda.synchronize()
    tm = ctx.timing()
    m = ctx.metrics()
    print(f"metrics={on}: round {a.elapsed_time(b) / n * 1e3:.1f} us, decode "
          f"{tm['decode_comp'][0] / n * 1e3:.1f} us, matching {m.matching_rate}, "
          f"disagreement {m.disagreement_rate:.4f}")
