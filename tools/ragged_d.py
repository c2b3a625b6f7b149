"""Sign-round time at C3-like sizes whose segment length is not a multiple
of 4 (real models: ResNet-50 has D = 25,557,032, L = 3,194,629) vs 25.6M."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

for D in (25_600_000, 25_557_032, 25_600_001):
    sched = mb.build_ring_schedule(8)
    ctx = mb.Context(D, sched, torch.float32, 0)
    g = [torch.empty(D, device="cuda") for _ in range(8)]
    for w in range(8):
        mb.fill_recipe(g[w], 0, 2026, w, 1)
    c = [torch.zeros(D, device="cuda") for _ in range(8)]
    for t in range(1, 5):
        ctx.sign_round(t, 2 ** -10, 2026, g, c)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.timing(reset=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 10
    for t in range(5, 5 + n):
        ctx.sign_round(t, 2 ** -10, 2026, g, c)
    b.record()
    torch.cuda.synchronize()
    tm = ctx.timing()
    L = -(-D // 8)
    print(f"D={D} L%4={L % 4}: {a.elapsed_time(b) / n * 1e3:.0f} us/round; extract "
          f"{tm['sign_extract'][0] / n * 1e3:.0f}, decode {tm['decode_comp'][0] / n * 1e3:.0f} us")
    del ctx, g, c
