"""One dense round (allreduce_dense, the K-th round) at C2 (ring 8, 61M) and
C4 (torus 2x4, 60.2M) for ncu: python tools/dense_probe.py c2|c4"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2204_06787_b200 as mb
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
D, sched = (61_000_000, mb.build_ring_schedule(8)) if cfg == "c2" else (60_200_000, mb.build_torus_schedule(2, 4))
M = sched.workers
ctx = mb.Context(D, sched, torch.float32, 0)
g = [torch.empty(D, device="cuda") for _ in range(M)]
for w in range(M):
    mb.fill_recipe(g[w], 0, 5, w, 1)
c = [torch.zeros(D, device="cuda") for _ in range(M)]
mean = torch.empty(D, device="cuda")
for _ in range(4):
    ctx.dense_round(0, g, c, mean)
torch.cuda.synchronize()
print("ok", cfg)
