#!/usr/bin/env python3
"""Every BASELINE config on one B200 (device time with CUDA events, inputs
resident in HBM, fp32, SURVEY §8d recipes):

  A. one GPU, all M workers simulated: sign round (independent and correlated
     recipes, with the measured disagreement rate), sign round with the fused
     metrics, dense round; each against its HBM floor at MEASURED_PEAKS.json;
  B. C5 (355M) driver step, bucketed, with the fused replica update;
  C. per-rank device time of a G-rank job (G = 2/4/8; C3 ring, C4 torus): the
     three phases of rank 0 with its M/G local workers, the merge on received
     packed bits (external-transport context, exchange itself not included),
     and the rank's NVLink payload.

  python tools/bench_configs.py [--iters N] [--skip-c5]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2204_06787_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--skip-c5", action="store_true")
ap.add_argument("--configs", default="c1,c2,c3,c4")
args = ap.parse_args()

CFG = {"c1": (1_000_000, "ring", 4, 0), "c2": (61_000_000, "ring", 8, 0),
       "c3": (25_600_000, "ring", 8, 0), "c4": (60_200_000, "torus", 2, 4)}
ETA, SEED = 2.0 ** -10, 2026
try:
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    PEAK = 6650.0
NVLINK = 900.0  # GB/s per direction


def sched_of(topo, a, b):
    return mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)


def timed(fn, iters, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


def emit(rec):
    print(json.dumps(rec), flush=True)


# A. one GPU, all workers -----------------------------------------------------
for name in args.configs.split(","):
    D, topo, a, b = CFG[name]
    sched = sched_of(topo, a, b)
    M = sched.workers
    ctx = mb.Context(D, sched, torch.float32, 0)
    g = [torch.empty(D, device="cuda") for _ in range(M)]
    c = [torch.zeros(D, device="cuda") for _ in range(M)]
    st = {"t": 1}

    def sign():
        ctx.sign_round(st["t"], ETA, SEED, g, c)
        st["t"] += 1

    sign_floor = 20.25 * M * D / PEAK / 1e3  # us
    for recipe in (0, 1):
        for w in range(M):
            mb.fill_recipe(g[w], recipe, SEED, w, 1)
        for x in c:
            x.zero_()
        ctx.set_metrics(True)
        sign()
        met = ctx.metrics()
        us_m = timed(sign, args.iters)  # metrics on
        ctx.set_metrics(False)
        us = timed(sign, args.iters)
        emit({"part": "A", "config": name, "topology": topo, "workers": M, "D": D,
              "recipe": ["independent", "correlated"][recipe], "sign_round_us": round(us, 1),
              "gelem_s": round(D / us / 1e3, 2), "worker_gelem_s": round(M * D / us / 1e3, 1),
              "hbm_floor_us": round(sign_floor, 1), "frac_of_floor": round(sign_floor / us, 3),
              "metrics_round_us": round(us_m, 1),
              "disagreement_rate": round(met.disagreement_rate, 4),
              "matching_rate": met.matching_rate})
    mean = torch.empty(D, device="cuda")
    us_d = timed(lambda: ctx.dense_round(0, g, c, mean), max(args.iters // 2, 3))
    dense_floor = (12.0 * M * D + 4.0 * D) / PEAK / 1e3
    emit({"part": "A", "config": name, "dense_round_us": round(us_d, 1),
          "hbm_floor_us": round(dense_floor, 1), "frac_of_floor": round(dense_floor / us_d, 3)})
    del ctx, g, c, mean
    torch.cuda.empty_cache()

# B. C5 -------------------------------------------------------------------------
if not args.skip_c5:
    D, M = 355_000_000, 8
    sched = mb.build_ring_schedule(M)
    drv = mb.Driver(D, sched, eta_s=ETA, global_seed=5, bucket_elems=100_000_000, first_round=1)
    g = [torch.empty(D, device="cuda") for _ in range(M)]
    for w in range(M):
        mb.fill_recipe(g[w], 0, 5, w, 1)
    x = [torch.zeros(D, device="cuda") for _ in range(M)]
    us = timed(lambda: drv.step(g, params=x), 3, warm=2)
    floor = 28.25 * M * D / PEAK / 1e3  # + read/write of the replica (8 B)
    emit({"part": "B", "config": "c5", "D": D, "workers": M, "buckets": 4,
          "driver_step_us": round(us, 1), "gelem_s": round(D / us / 1e3, 2),
          "hbm_floor_us": round(floor, 1), "frac_of_floor": round(floor / us, 3),
          "note": "sign step with carried compensation and fused replica update x -= g_t"})
    del drv, g, x
    torch.cuda.empty_cache()

# C. per-rank device time of a G-rank job ----------------------------------------
os.environ.setdefault("MARSIT_COIN_PREFETCH", "1")
for name, G in (("c3", 2), ("c3", 4), ("c3", 8), ("c4", 8)):
    D, topo, a, b = CFG[name]
    sched = sched_of(topo, a, b)
    M = sched.workers
    ml = M // G
    ctx = mb.Context(D, sched, torch.float32, 0, nranks=G, rank=0, external_transport=True)
    g = [torch.empty(D, device="cuda") for _ in range(ml)]
    for w in range(ml):
        mb.fill_recipe(g[w], 0, SEED, w, 1)
    c = [torch.zeros(D, device="cuda") for _ in range(ml)]
    lay = ctx.exchange_layout(False)

    class _H:
        __cuda_array_interface__ = {"shape": (lay.block_bytes * G // 8,), "typestr": "<i8",
                                    "data": (lay.recv, False), "version": 3, "strides": None}

    recv = torch.as_tensor(_H(), device="cuda")
    recv.copy_(torch.randint(-2 ** 62, 2 ** 62, recv.shape, device="cuda"))
    st = {"t": 1}

    def rank_round():  # rank 0's three phases in round order (exchange not included)
        for p in range(3):
            ctx.round_phase(p, st["t"], None, ETA, SEED, g, c)
        st["t"] += 1

    tot = timed(rank_round, args.iters)
    ctx.set_timing(True)
    ctx.timing(reset=True)
    for _ in range(args.iters):
        rank_round()
    torch.cuda.synchronize()
    tm = ctx.timing(reset=True)
    ctx.set_timing(False)
    ph = {i: tm[k][0] * 1e3 / args.iters  # us per round
          for i, k in enumerate(("sign_extract", "merge", "decode_comp"))}
    S = M  # segments
    L = -(-D // M)
    wbytes = -(-L // 32) * 4
    # P2P/NCCL payload per rank: received leaves of the owned segments from
    # the other ranks, then the owned aggregates to every other rank
    nv_in = (S // G) * (M - ml) * wbytes + (S - S // G) * wbytes
    floor = 20.25 * ml * D / PEAK / 1e3
    emit({"part": "C", "config": name, "topology": topo, "G": G, "local_workers": ml,
          "extract_us": round(ph[0], 1), "merge_us": round(ph[1], 1),
          "decode_us": round(ph[2], 1), "device_us": round(tot, 1),
          "hbm_floor_us": round(floor, 1), "frac_of_floor": round(floor / tot, 3),
          "nvlink_bytes_in": nv_in, "nvlink_us_at_900": round(nv_in / NVLINK / 1e3, 1),
          "gelem_s_if_exchange_hidden": round(D / tot / 1e3, 1)})
    del ctx, g, c, recv
    torch.cuda.empty_cache()
