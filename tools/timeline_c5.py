#!/usr/bin/env python3
"""CUPTI kernel timeline (torch.profiler) of one C5 driver step: D = 355M,
M = 8, 4 buckets of 88.75M, fused replica update.  Prints every kernel of the
middle step relative to its first kernel, and the busy time per kernel kind."""
import collections
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

D, M = int(os.environ.get("C5_D", 355_000_000)), 8
bucket = int(os.environ.get("C5_BUCKET", 88_750_000))
sched = mb.build_ring_schedule(M)
g = [torch.empty(D, device="cuda") for _ in range(M)]
for w in range(M):
    mb.fill_recipe(g[w], 0, 5, w, 1)
x = [torch.zeros(D, device="cuda") for _ in range(M)]
drv = mb.Driver(D, sched, eta_s=2 ** -10, global_seed=5, bucket_elems=bucket, first_round=1)
for _ in range(3):
    drv.step(g, params=x)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        drv.step(g, params=x)
        torch.cuda.synchronize()
path = os.path.join(tempfile.gettempdir(), "marsit_c5_trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel" and "marsit" in e.get("name", "")]
ev.sort(key=lambda e: e["ts"])
# steps are separated by host synchronisation gaps (> 200 us without a kernel)
steps, cur, last_end = [], [], None
for e in ev:
    if cur and e["ts"] - last_end > 200:
        steps.append(cur)
        cur = []
    cur.append(e)
    last_end = max(last_end or 0, e["ts"] + e["dur"])
steps.append(cur)
step = steps[len(steps) // 2]
t0 = step[0]["ts"]
busy = collections.defaultdict(float)
for e in step:
    name = e["name"].split("::")[-1].split("(")[0].split("<")[0]
    busy[name] += e["dur"]
    print(f"{name:26s} stream {e['args'].get('stream', '?'):>4}  {e['ts'] - t0:9.1f} .. "
          f"{e['ts'] + e['dur'] - t0:9.1f} us  ({e['dur']:.1f})")
span = max(e["ts"] + e["dur"] for e in step) - t0
print("step span %.1f us; busy per kernel kind: %s" % (span, {k: round(v, 1) for k, v in busy.items()}))
