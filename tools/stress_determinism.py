#!/usr/bin/env python3
"""Race evidence without compute-sanitizer (closed on this GPU pool): random
configurations (ring / torus, M, ragged D, merge kernel, tiling, coin budget,
emulated P2P ranks on concurrent streams), several carried rounds each, every
result compared bit for bit with the oracle.  Run it against the checked build
(MARSIT_SO=paper_2204_06787_b200/libmarsit_b200_checked.so: random sleeps at
every barrier / cluster barrier of the merge kernels + index bound latches),
where any missing ordering or out-of-bound index shows up as a mismatch or a
latched error.  Prints one JSON summary line."""
import json
import os
import random
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2204_06787_b200 as mb  # noqa: E402
import pyoracle as O  # noqa: E402

ETA = 2.0 ** -10
rng = random.Random(int(os.environ.get("STRESS_SEED", "2026")))
n_cfg = int(os.environ.get("STRESS_CONFIGS", "40"))
t0 = time.time()
rounds = mism = 0
kinds = {}
for i in range(n_cfg):
    topo = rng.choice(["ring", "ring", "torus"])
    if topo == "ring":
        a, b = rng.choice([2, 3, 4, 8, 16]), 0
    else:
        a, b = rng.choice([(2, 2), (2, 4), (3, 3), (4, 2)])
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    T = O.schedule(topo, a, b)
    W = sched.workers
    D = rng.choice([rng.randint(W, 5000), rng.randint(5000, 400_000), rng.randint(400_000, 2_000_000)])
    kernel = rng.choice(["coop", "cluster", "grid"])
    env = {"MARSIT_MERGE_KERNEL": kernel, "MARSIT_COIN_FRAC": rng.choice(["0", "0.2", "0.53", "2"]),
           "MARSIT_FUSED": rng.choice(["0", "1"])}
    if kernel == "cluster":
        env["MARSIT_MERGE_CSIZE"] = rng.choice(["0", "2", "8", "16"])
    elif kernel == "grid":
        env["MARSIT_MERGE_CSIZE"] = rng.choice(["0", "0", "5"])
    else:
        env["MARSIT_MERGE_WPT"] = rng.choice(["0", "1", "4", "12"])
    G = rng.choice([g for g in (1, 2, 4) if W % g == 0 and sched.segments % g == 0])
    for k, v in env.items():
        os.environ[k] = v
    seed = rng.randrange(1 << 32)
    kinds[f"{kernel}/G{G}"] = kinds.get(f"{kernel}/G{G}", 0) + 1
    if G == 1:
        ctxs = [mb.Context(D, sched, torch.float32, 0)]
    else:
        ctxs = [mb.Context(D, sched, torch.float32, 0, nranks=G, rank=r, transport="p2p")
                for r in range(G)]
        tab = [c.p2p_buffers() for c in ctxs]
        for c in ctxs:
            c.set_peers(tab)
    streams = [torch.cuda.Stream() for _ in ctxs]
    ml = W // G
    comp = [torch.zeros(D, device="cuda") for _ in range(W)]
    comp_o = np.zeros((W, D))
    for t in (1, 2, 3):
        g = np.stack([O.gen_dyadic(seed, w, t, D) for w in range(W)])
        gd = [torch.tensor(x, dtype=torch.float32, device="cuda") for x in g]
        torch.cuda.synchronize()
        for r, c in enumerate(ctxs):  # each rank on its own stream: the flag waits really block
            c.sign_round(t, ETA, seed, gd[r * ml:(r + 1) * ml], comp[r * ml:(r + 1) * ml],
                         stream=streams[r].cuda_stream)
        torch.cuda.synchronize()
        for r, c in enumerate(ctxs):
            c.check(stream=streams[r].cuda_stream)
        ref = O.marsit_round(T, t, None, ETA, g, comp_o, seed)
        got = np.stack([x.double().cpu().numpy() for x in comp])
        rounds += 1
        if not np.array_equal(got, ref.comp):
            mism += 1
            print("MISMATCH", topo, a, b, D, env, G, t, flush=True)
        comp_o = ref.comp
    for k in env:
        os.environ.pop(k)
    del ctxs
print(json.dumps({"library": os.path.basename(mb._native.SO_PATH), "configs": n_cfg,
                  "rounds": rounds, "mismatches": mism, "kinds": kinds,
                  "seconds": round(time.time() - t0, 1)}))
sys.exit(1 if mism else 0)
