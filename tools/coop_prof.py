"""Per-step phase times of CTA 0 of the cooperative merge (debug build)."""
import ctypes as C, os, subprocess, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb
from paper_2204_06787_b200 import _native as N
L = N.lib(); buf = (C.c_ulonglong * 16)()
def run(G, D):
    sched = mb.build_ring_schedule(8)
    ctx = mb.Context(D, sched, torch.float32, 0, nranks=G, rank=0, external_transport=(G > 1))
    lay = ctx.exchange_layout(False)
    class _H:
        __cuda_array_interface__ = {"shape": (lay.block_bytes * G // 8,), "typestr": "<i8",
                                    "data": (lay.recv, False), "version": 3, "strides": None}
    recv = torch.as_tensor(_H(), device="cuda")
    recv.copy_(torch.randint(-2**62, 2**62, recv.shape, device="cuda"))
    ml = 8 // G
    g = [torch.zeros(D, device="cuda") for _ in range(ml)]
    c = [torch.zeros(D, device="cuda") for _ in range(ml)]
    for t in range(1, 4):
        ctx.round_phase(0, t, None, 2**-10, 7, g, c); ctx.round_phase(1, t, None, 2**-10, 7, g, c)
    torch.cuda.synchronize(); L.marsit_debug_coop_prof(buf, 1)
    for t in range(4, 14):
        ctx.round_phase(0, t, None, 2**-10, 7, g, c); ctx.round_phase(1, t, None, 2**-10, 7, g, c)
    torch.cuda.synchronize(); L.marsit_debug_coop_prof(buf, 1)
    n = buf[4]
    print(f"G={G} D={D}: steps {n}  avg ns: load+scan {buf[0]/n:.0f}  grid.sync {buf[1]/n:.0f}  "
          f"prefix {buf[2]/n:.0f}  coins+deposit+store {buf[3]/n:.0f}")
for G in (8, 2, 1):
    run(G, 25_600_000)
