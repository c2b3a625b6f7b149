#!/usr/bin/env python3
"""Workload for ncu captures beyond the bench's four kernels: the C3 dense
round (dense_chain4_kernel), a G = 8 rank round (merge at 2 words/thread,
extract/decode of one worker) and a driver step with the fused replica
update (decode_kernel<float, 1, 1>).  Each runs a few times after warm-up.

  ncu --set full -k regex:"dense_chain4|merge_coop|decode_kernel<float, 1, 1>" ... python tools/prof_misc.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

D, ETA = 25_600_000, 2.0 ** -10
sched = mb.build_ring_schedule(8)
g = [torch.empty(D, device="cuda") for _ in range(8)]
for w in range(8):
    mb.fill_recipe(g[w], 0, 2026, w, 1)
c = [torch.zeros(D, device="cuda") for _ in range(8)]
ctx = mb.Context(D, sched, torch.float32, 0)
mean = torch.empty(D, device="cuda")
for t in range(4):
    ctx.dense_round(t, g, c, mean)
torch.cuda.synchronize()
del ctx
# one rank of a G = 8 job (external transport; the exchange is not run)
rk = mb.Context(D, sched, torch.float32, 0, nranks=8, rank=0, external_transport=True)
for t in range(1, 5):
    for p in range(3):
        rk.round_phase(p, t, None, ETA, 2026, g[:1], c[:1])
torch.cuda.synchronize()
del rk
drv = mb.Driver(D, sched, eta_s=ETA, global_seed=5, first_round=1)
x = [torch.zeros(D, device="cuda") for _ in range(8)]
for _ in range(3):
    drv.step(g, params=x)
torch.cuda.synchronize()
print("done")
