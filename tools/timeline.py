#!/usr/bin/env python3
"""Kernel timeline of a few sign rounds via torch.profiler (CUPTI activity
records: real device start/end of every kernel, all streams).  Prints one
step's kernels relative to the step's first kernel."""
import argparse
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=25_600_000)
ap.add_argument("--workers", type=int, default=8)
ap.add_argument("--steps", type=int, default=4)
args = ap.parse_args()

D, M = args.dim, args.workers
sched = mb.build_ring_schedule(M)
ctx = mb.Context(D, sched, torch.float32, 0)
if os.environ.get("TL_METRICS"):
    ctx.set_metrics(True)
g = [torch.empty(D, device="cuda") for _ in range(M)]
for w in range(M):
    mb.fill_recipe(g[w], 0, 2026, w, 1)
c = [torch.zeros(D, device="cuda") for _ in range(M)]
for t in range(1, 6):
    ctx.sign_round(t, 2 ** -10, 2026, g, c)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for t in range(10, 10 + args.steps):
        ctx.sign_round(t, 2 ** -10, 2026, g, c)
    torch.cuda.synchronize()
path = os.path.join(tempfile.gettempdir(), "marsit_trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"]
      if e.get("cat") == "kernel" and "marsit" in e.get("name", "")]
ev.sort(key=lambda e: e["ts"])
# split into steps at each extract kernel
steps, cur = [], []
for e in ev:
    if "extract_kernel" in e["name"] and cur:
        steps.append(cur)
        cur = []
    cur.append(e)
steps.append(cur)
step = steps[len(steps) // 2]
t0 = step[0]["ts"]
for e in step:
    name = e["name"].split("::")[-1].split("(")[0]
    print(f"{name:28s} stream {e['args'].get('stream', '?'):>4}  "
          f"{e['ts'] - t0:9.1f} .. {e['ts'] + e['dur'] - t0:9.1f} us  ({e['dur']:.1f})")
def span(st):
    return round(max(e["ts"] + e["dur"] for e in st) - st[0]["ts"], 1)


print("step span:", span(step), "us; steps:", [span(s) for s in steps],
      "; extract-to-extract:", [round(b[0]["ts"] - a[0]["ts"], 1) for a, b in zip(steps, steps[1:])])
