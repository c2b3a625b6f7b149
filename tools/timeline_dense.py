#!/usr/bin/env python3
"""CUPTI timeline of dense (full-precision K-th) rounds at C3: every kernel
and memset / memcpy on the device, relative to the round's first one."""
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

D, M = 25_600_000, 8
sched = mb.build_ring_schedule(M)
ctx = mb.Context(D, sched, torch.float32, 0)
g = [torch.empty(D, device="cuda") for _ in range(M)]
for w in range(M):
    mb.fill_recipe(g[w], 0, 2026, w, 1)
c = [torch.zeros(D, device="cuda") for _ in range(M)]
mean = torch.empty(D, device="cuda")
for t in range(3):
    ctx.dense_round(t, g, c, mean)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for t in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.dense_round(t, g, c, mean)
        b.record()
        torch.cuda.synchronize()
        print(f"dense round {t}: {a.elapsed_time(b) * 1e3:.1f} us")
path = os.path.join(tempfile.gettempdir(), "marsit_dense_trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"]
      if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev[: len(ev) // 3 + 1]:
    print(f"{e['name'].split('(')[0][-40:]:40s} {e['ts'] - t0:9.1f} .. {e['ts'] + e['dur'] - t0:9.1f} us "
          f"({e['dur']:.1f})")
