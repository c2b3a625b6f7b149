"""ncu helper: one cascading and one sum SSDM all-reduce at C3 (fp32)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402

D, M, seed = 25_600_000, 8, 2026
sched = mb.build_ring_schedule(M)
vecs = [torch.empty(D, device="cuda") for _ in range(M)]
for w in range(M):
    mb.fill_recipe(vecs[w], 0, seed, w, 1)
for fn in (mb.cascading_allreduce, mb.sum_ssdm_allreduce):
    fn(vecs, sched, seed, 1)
torch.cuda.synchronize()
