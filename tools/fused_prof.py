"""Phase times of CTA 0 of the fused small round (MARSIT_FUSED_PROF build,
MARSIT_SO=...libmarsit_b200_prof.so): extract / merge / decode per launch and,
inside the merge, pass 1 + CTA scan / cluster barrier / pass 2 per level."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402
from paper_2204_06787_b200 import _native as N  # noqa: E402

L = N.lib()
L.marsit_debug_coop_prof.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 8)()
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
    print(f"D={D} M={M}: launches {buf[3]} extract {buf[0]/n/1e3:.2f} us  merge {buf[1]/n/1e3:.2f} us  "
          f"decode {buf[2]/n/1e3:.2f} us | per level ({nl // n} levels): pass1+scan {buf[4]/nl/1e3:.2f}  "
          f"cluster barrier {buf[5]/nl/1e3:.2f}  pass2 {buf[6]/nl/1e3:.2f} us")
