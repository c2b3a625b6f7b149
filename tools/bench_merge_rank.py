#!/usr/bin/env python3
"""Merge time of ONE rank of a G-GPU job (external-transport context, random
received packed bits): the multi-GPU critical-path merge, measured on 1 GPU."""
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
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--topo", default="ring")
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
sched = mb.build_ring_schedule(8) if args.topo == "ring" else mb.build_torus_schedule(2, 4)
G = args.ranks
ml = 8 // G
ctx = mb.Context(args.dim, sched, torch.float32, 0, nranks=G, rank=0, external_transport=True)
lay = ctx.exchange_layout(False)


class _H:
    __cuda_array_interface__ = {"shape": (lay.block_bytes * G // 8,), "typestr": "<i8",
                                "data": (lay.recv, False), "version": 3, "strides": None}


recv = torch.as_tensor(_H(), device="cuda")
recv.copy_(torch.randint(-2**62, 2**62, recv.shape, device="cuda"))
D = args.dim
g = [torch.zeros(D, device="cuda") for _ in range(ml)]
c = [torch.zeros(D, device="cuda") for _ in range(ml)]
# phase 0 first every round: it computes the round's coins (adaptive budget:
# the coin kernel sizes each merge's coins from the previous merge)
for t in range(1, 4):
    ctx.round_phase(0, t, None, 2 ** -10, 7, g, c)
    ctx.round_phase(1, t, None, 2 ** -10, 7, g, c)
torch.cuda.synchronize()
ctx.set_timing(True)
ctx.timing(reset=True)
for t in range(4, 4 + args.iters):
    ctx.round_phase(0, t, None, 2 ** -10, 7, g, c)
    ctx.round_phase(1, t, None, 2 ** -10, 7, g, c)
torch.cuda.synchronize()
ms, n = ctx.timing(reset=True)["merge"]
print(f"rank merge (G={G}, D={D}, {args.topo}): {ms / args.iters * 1e3:.1f} us per round "
      f"({n // args.iters} launches)")
