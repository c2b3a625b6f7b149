"""C1-size one-launch rounds: eager (Python enqueue per round) vs CUDA-graph
replay (device time only), spread round vs the cluster-per-segment round.
Usage: python tools/spread_probe.py [D] [M]"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2204_06787_b200 as mb

D = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ETA, SEED, N = 2.0 ** -10, 2026, 200
sched = mb.build_ring_schedule(M)
g = [torch.empty(D, device="cuda") for _ in range(M)]
for w in range(M):
    mb.fill_recipe(g[w], 0, SEED, w, 1)
ctx = mb.Context(D, sched, torch.float32, 0)
c = [torch.zeros(D, device="cuda") for _ in range(M)]
for t in range(1, 20):
    ctx.sign_round(t, ETA, SEED, g, c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for t in range(20, 20 + N):
    ctx.sign_round(t, ETA, SEED, g, c)
e1.record()
torch.cuda.synchronize()
eager = e0.elapsed_time(e1) / N * 1e3
ctx.set_timing(True)
ctx.timing(reset=True)  # launches are counted with timing off too
for t in range(20, 20 + N):
    ctx.sign_round(t, ETA, SEED, g, c)
torch.cuda.synchronize()
tm = {k: v for k, v in ctx.timing().items() if v[1]}
ctx.set_timing(False)
kern = {k: round(v[0] / v[1] * 1e3, 2) for k, v in tm.items()}
graph_us = None
if os.environ.get("SPREAD_NO_GRAPH"):  # under ncu: eager rounds only
    print({"D": D, "M": M, "eager_us": round(eager, 2), "per_kernel_us": kern}, flush=True)
    sys.exit(0)
try:
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for t in range(1, 51):
            ctx.sign_round(t, ETA, SEED, g, c)
    gr.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_us = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
except Exception as ex:  # the cluster path forks a side stream per round
    graph_us = f"n/a ({type(ex).__name__})"
print({"D": D, "M": M, "spread": os.environ.get("MARSIT_SPREAD", "1"),
       "csize": os.environ.get("MARSIT_SPREAD_CSIZE", "auto"), "eager_us": round(eager, 2),
       "per_kernel_us": kern, "graph_us": graph_us}, flush=True)
