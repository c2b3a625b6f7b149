"""ncu helper: C3 sign rounds, two with the fused metrics decode, two without."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

D, W, seed = 25_600_000, 8, 2026
sched = mb.build_ring_schedule(W)
g = [torch.empty(D, device="cuda") for _ in range(W)]
for w in range(W):
    mb.fill_recipe(g[w], 0, seed, w, 1)
for on in (True, False):
    ctx = mb.Context(D, sched, torch.float32, 0)
    ctx.set_metrics(on)
    c = [torch.zeros(D, device="cuda") for _ in range(W)]
    for t in range(1, 3):
        ctx.sign_round(t, 2 ** -10, seed, g, c)
    torch.cuda.synchronize()
    print(ctx.metrics())
