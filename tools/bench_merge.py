#!/usr/bin/env python3
"""Micro-benchmark of the merge DAG kernel alone (allreduce_sign lower entry on
random packed signs), reporting device time per merge launch and coins/s."""
import argparse
import os
import sys

import torch

# the next round's coin prefetch would co-run with the following merge here
# (in a real round it runs underneath the decode): measure the merge alone
os.environ.setdefault("MARSIT_COIN_PREFETCH", "0")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=25_600_000)
ap.add_argument("--topo", default="ring")
ap.add_argument("--a", type=int, default=8)
ap.add_argument("--b", type=int, default=0)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--segs", type=int, default=0, help="emulate owning only this many segments")
args = ap.parse_args()

sched = mb.build_ring_schedule(args.a) if args.topo == "ring" else mb.build_torus_schedule(args.a, args.b)
M, S = sched.workers, sched.segments
L = -(-args.dim // S)
nw = (L + 63) // 64
ctx = mb.Context(args.dim, sched, torch.float32, 0)
g = torch.Generator(device="cuda").manual_seed(1)
signs = torch.randint(-2**63, 2**63 - 1, (M, S, nw), dtype=torch.int64, device="cuda", generator=g)
if L % 64:
    signs[..., -1] &= (1 << (L % 64)) - 1
out = torch.empty((S, nw), dtype=torch.int64, device="cuda")
for _ in range(3):
    ctx.allreduce_sign(1, 7, signs, out)
torch.cuda.synchronize()
ctx.set_timing(True)
ctx.timing(reset=True)
for i in range(args.iters):
    ctx.allreduce_sign(i + 2, 7, signs, out)
torch.cuda.synchronize()
t = ctx.timing(reset=True)
ms, n = t["merge"]
coins = (M - 1) * L * S * 0.5
print(f"merge: {ms / args.iters * 1e3:.1f} us per round ({n // args.iters} launches), "
      f"~{coins / (ms / args.iters * 1e-3) / 1e9:.2f} Gcoins/s")
