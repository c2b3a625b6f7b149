"""Average per-phase time of one merge step (tile x merge), debug build."""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb
from paper_2204_06787_b200 import _native as N
D = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
sched = mb.build_ring_schedule(8)
ctx = mb.Context(D, sched, torch.float32, 0)
g = [torch.empty(D, device="cuda") for _ in range(8)]
for w in range(8): mb.fill_recipe(g[w], 0, 2026, w, 1)
c = [torch.zeros(D, device="cuda") for _ in range(8)]
for t in range(1, 4): ctx.sign_round(t, 2**-10, 2026, g, c)
torch.cuda.synchronize()
L = N.lib(); buf = (C.c_ulonglong * 8)()
L.marsit_debug_merge_prof(buf, 1)
for t in range(4, 8): ctx.sign_round(t, 2**-10, 2026, g, c)
torch.cuda.synchronize()
L.marsit_debug_merge_prof(buf, 1)
n = buf[4]
print("merge steps:", n, " avg ns: load+scan", buf[0] / n, " lookback", buf[1] / n,
      " coins+deposit", buf[2] / n, " store+sync", buf[3] / n)
