"""Phase times of the spread small round (MARSIT_FUSED_PROF build, MARSIT_SO=
...libmarsit_b200_prof.so): CTA 0 (in merge cluster 0) and the last CTA (a
streaming-only CTA), per launch, from %globaltimer."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402
from paper_2204_06787_b200 import _native as N  # noqa: E402

L = N.lib()
L.marsit_debug_coop_prof.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 16)()
for D, M in ((1_000_000, 4), (4_000_000, 4), (1_000_000, 8)):
    sched = mb.build_ring_schedule(M)
    ctx = mb.Context(D, sched, torch.float32, 0)
    g = [torch.empty(D, device="cuda") for _ in range(M)]
    for w in range(M):
        mb.fill_recipe(g[w], 0, 2026, w, 1)
    c = [torch.zeros(D, device="cuda") for _ in range(M)]
    for t in range(1, 6):
        ctx.sign_round(t, 2 ** -10, 2026, g, c)
    torch.cuda.synchronize()
    L.marsit_debug_coop_prof(buf, 1)
    for t in range(6, 26):
        ctx.sign_round(t, 2 ** -10, 2026, g, c)
    torch.cuda.synchronize()
    L.marsit_debug_coop_prof(buf, 1)
    n, nl = max(buf[3], 1), max(buf[7], 1)
    us = lambda i: buf[i] / n / 1e3  # noqa: E731
    print(f"D={D} M={M}: CTA0 start {us(8):.2f} +extract (+coins on a tag miss) {us(0)-us(8):.2f} | wait-arrivals {us(9):.2f} "
          f"merge(incl wait) {us(1):.2f} | wait-aggregates {us(10):.2f} decode(incl wait) {us(2):.2f} || "
          f"last CTA: start {us(12):.2f} wait-aggregates {us(14):.2f} whole {us(15):.2f} | per level "
          f"({nl // n}): pass1+scan {buf[4]/nl/1e3:.2f} barrier {buf[5]/nl/1e3:.2f} pass2 {buf[6]/nl/1e3:.2f} us",
          flush=True)
