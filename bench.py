#!/usr/bin/env python3
"""Marsit sign all-reduce round on B200 — the driver's benchmark.

Default (N=1): BASELINE config C3 — ring all-reduce of a 25.6M-element fp32
gradient over M=8 workers (all simulated on the one GPU), with the global
compensation update, one step = one marsit_round sign round (t >= 1).
With N ranks (torchrun, or `--gpus N` which re-launches itself under
torchrun) the same M=8 workers are split 8/N per GPU (strong scaling: total
work fixed); the packed segments move over NVLink peer memory inside the
merge and decode kernels (--transport p2p, default) or with NCCL
(--transport nccl).  The N > 1 line carries `parity_vs_g1` (the G-rank
round against one context holding all M workers), per-rank phase times and
the NVLink payload.

Metric: sign-allreduce Gelem/s = D / step time (all-reduce algbw convention).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sign-allreduce Gelem/s (25.6M grad, 1/2/4/8 B200) + % HBM/NVLink roofline"
ETA = 2.0 ** -10
SEED = 2026

L2_BYTES = 126 << 20  # B200 L2 (MEASURED_PEAKS / B200_PROFILING)

CONFIGS = {
    # id: (D, topology, a, b)
    "c1": (1_000_000, "ring", 4, 0),
    "c2": (61_000_000, "ring", 8, 0),
    "c3": (25_600_000, "ring", 8, 0),
    "c4": (60_200_000, "torus", 2, 4),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p",
                    help="N > 1: fused over NVLink peer memory (p2p) or NCCL send/recv + all-gather")
    ap.add_argument("--recipe", type=int, default=0, help="0 dyadic (independent), 1 correlated")
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32",
                    help="element type of gradients and compensation (f64: the drop-in's)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--min-busy-s", type=float, default=1.5,
                    help="keep the GPU busy at least this long before timing (clock sampling)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ----------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = []
        for ts, line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 10:
                continue
            rows.append((ts, parts))
        sel = [p for ts, p in rows if t0 - 0.15 <= ts <= t1 + 0.15] or [p for _, p in rows]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        busy = [p for p in sel if p[4].isdigit() and int(p[4]) > 0] or sel
        sm = [float(p[1]) for p in busy if p[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for p in busy:
            for n, v in zip(names, p[6:10]):
                if "Active" in v and "Not" not in v:
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(busy[0][2]) if busy[0][2].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(busy)}


# ----------------------------------------------------------------------------
# CPU baselines
# ----------------------------------------------------------------------------
def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class RefBuckets:
    """The reference's own marsit_round (oracle/_ref, compiled from the unmodified
    headers) on every host thread at once: the D-coordinate sample is split into
    `threads` contiguous buckets and each thread runs the reference's round on its
    bucket (the reference is single-threaded per round; buckets are the only way
    it can use more than one core). ctypes releases the GIL around each call."""

    def __init__(self, cfg_id: str, sample_dim: int, threads: int):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle as O
        from concurrent.futures import ThreadPoolExecutor
        _, topo, a, b = CONFIGS[cfg_id]
        self.R = O.ref()
        self.threads = threads
        self.dims = [sample_dim // threads + (1 if i < sample_dim % threads else 0)
                     for i in range(threads)]
        self.h = [self.R.ref_bench_create(0 if topo == "ring" else 1, a, b, d, SEED + i)
                  for i, d in enumerate(self.dims)]
        self.pool = ThreadPoolExecutor(threads)

    def round(self, t: int) -> float:
        t0 = time.perf_counter()
        rcs = list(self.pool.map(lambda h: self.R.ref_bench_round(h, t), self.h))
        ms = (time.perf_counter() - t0) * 1e3
        if any(rc < 0 for rc in rcs):
            raise RuntimeError(f"reference round failed: {rcs}")
        return ms

    def close(self):
        self.pool.shutdown()
        for h in self.h:
            self.R.ref_bench_destroy(h)


def cpu_baseline(cfg_id: str, sample_dim: int, rounds: int = 3):
    """The reference's own marsit_round (oracle/_ref) on all host threads (see
    RefBuckets), plus its single-thread time on the unsplit sample; the C
    restatement (1 thread) where the reference was not built."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import pyoracle as O
    D, topo, a, b = CONFIGS[cfg_id]
    single = None
    if O.ref_available():
        R = O.ref()
        h = R.ref_bench_create(0 if topo == "ring" else 1, a, b, sample_dim, SEED)
        R.ref_bench_round(h, 1)  # warm-up round
        st = min(R.ref_bench_round(h, t) for t in range(2, 2 + rounds))
        R.ref_bench_destroy(h)
        single = {"value": sample_dim / (st * 1e-3) / 1e9, "ms_per_round": st, "cores": 1}
        cores = host_threads()
        rb = RefBuckets(cfg_id, sample_dim, cores)
        rb.round(1)
        times = [rb.round(t) for t in range(2, 2 + rounds)]
        rb.close()
        kind = "reference"
        how = (f"{cores} threads, each the reference's marsit_round on a contiguous "
               f"{sample_dim // cores}-coordinate bucket")
    else:
        O.build() if not os.path.exists(O.ORACLE_SO) else None
        T = O.schedule(topo, a, b)
        g = np.stack([O.gen_dyadic(SEED, w, 1, sample_dim) for w in range(T.workers)])
        comp = np.zeros_like(g)
        times = []
        for t in range(1, 2 + rounds):
            t0 = time.perf_counter()
            r = O.marsit_round(T, t, None, ETA, g, comp, SEED)
            dt = (time.perf_counter() - t0) * 1e3
            comp = r.comp
            if t > 1:
                times.append(dt)
        kind, cores, how = "port", 1, "1 thread (C restatement)"
    ms = min(times)
    out = {"value": sample_dim / (ms * 1e-3) / 1e9, "unit": "Gelem/s", "cores": cores,
           "kind": kind, "ms_per_round": ms,
           "sample": f"{topo} M={a * (b or 1)} D={sample_dim} sign round (t>=1, K=never), "
                     f"best of {rounds} warm rounds, {how}",
           "host_cpu": _cpu_model(), "nproc": os.cpu_count()}
    if single is not None:
        out["single_thread"] = single
    return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    """The reference's own CPU path (oracle/_ref: its unmodified headers compiled
    with the Release flags) on the arm's config: each step is ONE stock
    marsit_round (sync.hpp:60-120) over the full D and all M workers — the
    reference is single-threaded, so this is 1 host core.  A secondary figure
    times the same round on all host threads, the D/10 sample split into one
    contiguous bucket per thread (the only way the reference uses more cores;
    bucketed semantics, reported as `bucketed_all_threads`)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    D, topo, a, b = CONFIGS[args.config]
    M = a * (b or 1)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    steps = []
    secondary = None
    if O.ref_available():
        R = O.ref()
        h = R.ref_bench_create(0 if topo == "ring" else 1, a, b, D, SEED)
        t = 1
        for _ in range(args.warmup):
            ms = R.ref_bench_round(h, t)
            if ms < 0:
                raise RuntimeError(f"reference round failed: {ms}")
            t += 1
        for _ in range(args.steps):
            ms = R.ref_bench_round(h, t)
            if ms < 0:
                raise RuntimeError(f"reference round failed: {ms}")
            steps.append(ms)
            t += 1
        R.ref_bench_destroy(h)
        kind, cores = "reference", 1
        how = (f"the reference's own marsit_round over the full D={D}, M={M} workers, one "
               f"round per step (single-threaded, as the reference is)")
        if not args.no_cpu_baseline:
            try:
                sample = max(D // 10, 1000)
                threads = host_threads()
                rb = RefBuckets(args.config, sample, threads)
                rb.round(1)
                bt = [rb.round(tt) for tt in range(2, 5)]
                rb.close()
                secondary = {"value": sample / (min(bt) * 1e-3) / 1e9, "unit": "Gelem/s",
                             "cores": threads, "ms_per_round": min(bt),
                             "sample": f"D={sample} sample split into {threads} contiguous "
                                       f"buckets, each the reference's marsit_round on its own "
                                       f"host thread (bucketed semantics, not one round)"}
            except Exception as e:  # pragma: no cover
                secondary = {"error": str(e)}
    else:
        cb = cpu_baseline(args.config, max(D // 10, 1000), rounds=max(args.steps, 1))
        steps = [cb["ms_per_round"] * 10]
        kind, cores, how = "port", 1, "1 thread (C restatement, D/10 sample x 10)"
    ms = sum(steps) / len(steps)
    val = D / (ms * 1e-3) / 1e9
    line = {"metric": METRIC, "value": val, "unit": "Gelem/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY §8c dyadic recipe)", "impl": "reference",
            "config": {"workload": f"{args.config}: {topo} all-reduce M={M} workers, D={D}, "
                                   f"sign round + compensation",
                       "D": D, "workers": M, "topology": topo, "same_config": kind == "reference"},
            "cpu_baseline": {"value": val, "unit": "Gelem/s", "cores": cores, "kind": kind,
                             "sample": f"one step = {how}", "host_cpu": _cpu_model(),
                             "nproc": os.cpu_count()},
            "e2e": {"value": val, "unit": "Gelem/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if secondary is not None:
        line["bucketed_all_threads"] = secondary
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
class Comm:
    """torch.distributed plumbing of the bench (barriers, max over ranks, the
    warm-up decision, small objects).  NCCL over the ranks' GPUs; gloo with CPU
    tensors when the ranks share one device (MARSIT_BENCH_DEVICE, tests)."""

    def __init__(self, world, rank, dev, shared):
        import torch
        import torch.distributed as dist
        self.dist, self.world, self.rank = dist, world, rank
        self.tdev = torch.device("cpu")
        if world > 1:
            if shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=dev)
                self.tdev = dev

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.tdev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def bcast(self, v: int) -> int:
        if self.world == 1:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.int64, device=self.tdev)
        self.dist.broadcast(t, 0)
        return int(t.item())

    def gather(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def warm_up(comm, step, sync, warmup: int, min_busy_s: float) -> int:
    """Untimed rounds 1..n: at least max(W, 3) and at least min_busy_s of GPU
    work (clock sampling).  Rank 0 decides after every chunk whether to go on
    and broadcasts it, so every rank runs the same number of rounds — the
    lock-step delivery of transport.hpp:27-35 (P2P flag waits and NCCL
    collectives pair round by round; a rank that ran ahead would wait for
    flags its peers never write).  Returns n."""
    n = 0
    t0 = time.time()
    chunk = max(warmup, 3)
    while True:
        for _ in range(chunk):
            n += 1
            step(n)
        sync()
        more = int(time.time() - t0 < min_busy_s) if comm.rank == 0 else 0
        if not comm.bcast(more):
            return n
        chunk = 20


def _digest(t) -> str:
    import hashlib
    return hashlib.blake2b(t.contiguous().view(-1).cpu().numpy().tobytes(), digest_size=16).hexdigest()


def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    shared = os.environ.get("MARSIT_BENCH_DEVICE") is not None
    dev_index = int(os.environ["MARSIT_BENCH_DEVICE"]) if shared else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    comm = Comm(world, rank, dev, shared)

    import paper_2204_06787_b200 as mb

    D, topo, a, b = CONFIGS[args.config]
    sched = mb.build_ring_schedule(a) if topo == "ring" else mb.build_torus_schedule(a, b)
    M, S = sched.workers, sched.segments
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    esize = 8 if dt == torch.float64 else 4
    nccl_id = None
    if world > 1 and args.transport == "nccl":
        ids = comm.gather(bytes(mb.nccl_unique_id()) if rank == 0 else None)
        nccl_id = ids[0]
    ctx = mb.Context(D, sched, dt, dev_index, nranks=world, rank=rank, nccl_id=nccl_id,
                     transport=args.transport if world > 1 else None)
    opened = []
    if world > 1 and args.transport == "p2p":
        opened = mb.exchange_p2p_buffers(ctx)  # CUDA IPC handles over torch.distributed
    ml, w0 = ctx.local_workers, ctx.first_worker
    grads = [torch.empty(D, device=dev, dtype=dt) for _ in range(ml)]
    for i in range(ml):
        mb.fill_recipe(grads[i], args.recipe, SEED, w0 + i, 1)
    comp = [torch.zeros(D, device=dev, dtype=dt) for _ in range(ml)]
    stream = torch.cuda.current_stream(dev)

    def step(t):
        ctx.sign_round(t, ETA, SEED, grads, comp)

    sampler = ClockSampler(dev_index)
    sampler.start()
    n_warm = warm_up(comm, step, lambda: torch.cuda.synchronize(dev), args.warmup, args.min_busy_s)
    t = 1 + n_warm
    ctx.check()
    comm.barrier()
    torch.cuda.synchronize(dev)
    # headline: K steps, no per-phase instrumentation inside the timed region.
    # Inputs larger than L2 stream from HBM every step; smaller ones (C1)
    # would be L2-resident from the step before, so then L2 is flushed
    # (a 512 MB write) before every step, outside per-step events.
    in_bytes = 2 * ml * D * esize
    flush_l2 = in_bytes <= L2_BYTES
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    if flush_l2:
        scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for k in range(args.steps):
            scratch.fill_(k & 0xFF)
            ev[k][0].record(stream)
            step(t)
            ev[k][1].record(stream)
            t += 1
        torch.cuda.synchronize(dev)
        ms_rank = sum(a.elapsed_time(b) for a, b in ev) / args.steps
        del scratch
    else:
        e0.record(stream)
        for k in range(args.steps):
            step(t)
            t += 1
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_rank = e0.elapsed_time(e1) / args.steps
    wall1 = time.time()
    comm.barrier()
    # breakdown: K more steps with CUDA events around every phase on its
    # stream (the roofline's per-launch kernel times)
    ctx.set_timing(True)
    ctx.timing(reset=True)
    for k in range(args.steps):
        step(t)
        t += 1
    torch.cuda.synchronize(dev)
    phases = ctx.timing(reset=True)
    ctx.set_timing(False)
    ctx.check()
    sampler.stop()
    clocks = sampler.summary(wall0, wall1)
    ms = comm.max(ms_rank)

    # e2e through the public API with host buffers (pinned), copies inside the
    # region: every step uploads its gradients and reads back its aggregate
    # bits.  Two device gradient buffers: step k+1's upload (copy stream)
    # overlaps step k's round (compute stream), as a training loop would.
    host_g = [torch.empty(D, dtype=dt, pin_memory=True) for _ in range(ml)]
    for i in range(ml):
        host_g[i].copy_(grads[i])
    nwords = (D + 63) // 64
    agg_dev = torch.empty(nwords, dtype=torch.int64, device=dev)
    agg_host = torch.empty(nwords, dtype=torch.int64, pin_memory=True)
    dev_g = [[torch.empty_like(x) for x in grads] for _ in range(2)]
    copy_stream = torch.cuda.Stream(dev)
    ev_copied = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    for e in ev_used:
        e.record(stream)

    def e2e_upload(k):
        bb = k % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(ev_used[bb])  # the round that read buffer bb is done
            for i in range(ml):
                dev_g[bb][i].copy_(host_g[i], non_blocking=True)
            ev_copied[bb].record(copy_stream)

    def e2e_round(k, t):
        bb = k % 2
        stream.wait_event(ev_copied[bb])
        ctx.sign_round(t, ETA, SEED, dev_g[bb], comp, agg_bits=agg_dev)
        ev_used[bb].record(stream)
        agg_host.copy_(agg_dev, non_blocking=True)

    e2e_upload(0)
    e2e_round(0, t)
    t += 1
    torch.cuda.synchronize(dev)
    comm.barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record(stream)
    ev_used[0].record(stream)
    ev_used[1].record(stream)  # no upload starts before x0
    e2e_upload(0)
    for k in range(args.e2e_steps):
        if k + 1 < args.e2e_steps:
            e2e_upload(k + 1)
        e2e_round(k, t)
        t += 1
    x1.record(stream)
    torch.cuda.synchronize(dev)
    comm.barrier()
    e2e_ms = comm.max(x0.elapsed_time(x1) / args.e2e_steps)
    ctx.check()

    # N > 1: parity self-check of the G-rank job against one context holding
    # all M workers (rank 0): the same round from c = 0 on every rank, hashes
    # of the aggregate bits and of every worker's compensation
    parity = None
    if world > 1:
        T0 = 1 << 20
        chk = [torch.zeros(D, device=dev, dtype=dt) for _ in range(ml)]
        agg_chk = torch.empty(nwords, dtype=torch.int64, device=dev)
        ctx.sign_round(T0, ETA, SEED, grads, chk, agg_bits=agg_chk)
        torch.cuda.synchronize(dev)
        ctx.check()
        mine = {"agg": _digest(agg_chk), "comp": {w0 + i: _digest(chk[i]) for i in range(ml)}}
        allh = comm.gather(mine)
        del chk, agg_chk
        if rank == 0:
            one = mb.Context(D, sched, dt, dev_index)
            g1 = [torch.empty(D, device=dev, dtype=dt) for _ in range(M)]
            for w in range(M):
                mb.fill_recipe(g1[w], args.recipe, SEED, w, 1)
            c1 = [torch.zeros(D, device=dev, dtype=dt) for _ in range(M)]
            a1 = torch.empty(nwords, dtype=torch.int64, device=dev)
            one.sign_round(T0, ETA, SEED, g1, c1, agg_bits=a1)
            torch.cuda.synchronize(dev)
            one.check()
            ok = all(h["agg"] == _digest(a1) for h in allh)
            for h in allh:
                for w, dg in h["comp"].items():
                    ok &= dg == _digest(c1[int(w)])
            parity = "bit-exact" if ok else "MISMATCH"
            del one, g1, c1, a1
        parity = comm.gather(parity)[0]

    # per-rank phase times (timing pass) and NVLink payload (N > 1)
    per_rank = comm.gather({k: v[0] / args.steps for k, v in phases.items() if v[1]})
    L = -(-D // S)
    seg_bytes = ((2 * -(-L // 64) + 3) // 4 * 4) * 4  # packed words of one segment (u32, x4)
    s_own = S // world
    nvl_in = ((M - ml) * s_own + (S - s_own)) * seg_bytes if world > 1 else 0

    # roofline: dominant kernel = decode+compensation (K3/K4), 8 + 4 B (fp32)
    # per worker-element + 1/8 B of aggregate bits
    hbm, hbm_kind = peaks()
    dec_ms_tot, dec_n = phases.get("decode_comp", (float("nan"), 0))
    ext_ms_tot, ext_n = phases.get("sign_extract", (float("nan"), 0))
    dec_unit = 3 * esize + 0.125
    dec_kernel = "decode_comp (K3+K4)"
    fused = not dec_n and phases.get("fused_round", (0.0, 0))[1] > 0
    spread = not dec_n and phases.get("spread_round", (0.0, 0))[1] > 0
    if fused:  # small rounds run as one launch (extract + merge + decode per cluster)
        dec_ms_tot, dec_n = phases["fused_round"]
        dec_unit = 5 * esize + 0.25
        dec_kernel = "fused_round (K1+K2+K3/K4, one cluster launch; the re-read of g, c hits L2)"
    elif spread:  # small rounds run as one launch over every SM (coins + K1 + K2 + K3/K4)
        dec_ms_tot, dec_n = phases["spread_round"]
        dec_unit = 5 * esize + 0.25
        dec_kernel = "spread_round (coins+K1+K2+K3/K4, one launch over every SM; the re-read of g, c hits L2)"
    dec_bytes = ml * D * dec_unit * args.steps   # read g, c; write c'; 1/8 B of bits
    ext_bytes = ml * D * (2 * esize + 0.125) * args.steps  # read g, c; write 1/8 B of bits
    dec_gbs = dec_bytes / (dec_ms_tot * 1e-3) / 1e9 if dec_ms_tot == dec_ms_tot and dec_ms_tot else 0.0
    dec_ms = dec_ms_tot / max(dec_n, 1)
    step_unit = 5 * esize + 0.25
    step_bytes = ml * D * step_unit
    step_gbs = step_bytes / (ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        traffic = tr.get(f"{args.config}_g{world}_decode_bytes" + ("_f64" if esize == 8 else ""))
    except Exception:
        pass
    launches = sum(nl for _, nl in phases.values())

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": D / (ms * 1e-3) / 1e9,
            "unit": "Gelem/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": n_warm,  # untimed steps actually run: >= max(W, 3) and >= --min-busy-s of work
            "warmup_requested": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": args.dtype,
            "data": "synthetic (SURVEY §8c dyadic recipe, on-device generation)"
                    if args.recipe == 0 else "synthetic (SURVEY §8d correlated recipe)",
            "config": {"workload": f"{args.config}: {topo} all-reduce M={M} workers "
                                   f"({ml} per GPU), D={D}, sign round + compensation",
                       "D": D, "workers": M, "topology": topo,
                       "parallelism": f"{world} rank(s) x {ml} workers",
                       "transport": (args.transport if world > 1 else "none (1 rank)"),
                       "l2": ("inputs (%.1f GB) > L2 (126 MB): no flush needed" % (in_bytes / 1e9))
                             if not flush_l2 else
                             ("inputs (%.0f MB) fit in L2 (126 MB): L2 flushed (512 MB write) before "
                              "every timed step, each step timed by its own events" % (in_bytes / 1e6))},
            "worker_gelem_s": M * D / (ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": dec_kernel,
                         "achieved": dec_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": dec_gbs / hbm, "traffic": traffic,
                         "peak_kind": hbm_kind,
                         "algorithmic_bytes_per_launch": dec_bytes / max(dec_n, 1),
                         "avg_launch_ms": dec_ms, "launches": int(dec_n)},
            "step_roofline": {"bytes_per_step": step_bytes, "achieved": step_gbs,
                              "frac": step_gbs / hbm,
                              "note": f"{step_unit} B per worker-element two-pass floor "
                                      f"(SURVEY §8d), this rank's {ml} workers"},
            "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items() if v[1]},
            "sign_extract_gbs": (ext_bytes / (ext_ms_tot * 1e-3) / 1e9) if ext_n else None,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "e2e": {"value": D / (e2e_ms * 1e-3) / 1e9, "unit": "Gelem/s",
                    "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": ml * D * esize * world,
                    "d2h_bytes_per_step": nwords * 8 * world,
                    "path": "Context.sign_round (C-ABI marsit_sign_round) with pinned host "
                            "gradients copied in and aggregate bits copied out every step on "
                            "every rank; double-buffered device gradients: step k+1's upload "
                            "(copy stream) overlaps step k's round",
                    "h2d_gbs_per_rank": ml * D * esize / (e2e_ms * 1e-3) / 1e9},
        }
        if world > 1:
            line["parity_vs_g1"] = parity
            line["per_rank_phases_ms"] = per_rank
            line["nvlink"] = {"bytes_in_per_rank_per_step": nvl_in,
                              "achieved_gbs": nvl_in / (ms * 1e-3) / 1e9,
                              "peak_gbs": 770.0, "peak_kind": "measured peer copy "
                              "(B200_PROFILING.md; 900 nominal)",
                              "frac": nvl_in / (ms * 1e-3) / 1e9 / 770.0,
                              "note": "owned segments' leaves from the other ranks + the other "
                                      "owners' aggregates, packed bits"}
            if shared:
                line["note"] = ("ranks shared one GPU (MARSIT_BENCH_DEVICE): functional run, "
                                "times are not a multi-GPU measurement")
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(args.config, D // 10)
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"value": None, "error": str(e)}
        print(json.dumps(line), flush=True)
    comm.barrier()
    del ctx
    for ptr in opened:
        mb._native.lib().marsit_ipc_close(ptr)
    comm.close()


def spawn(args):
    """`bench.py --gpus N` outside torchrun: re-launch this command as N ranks."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return 0
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        return spawn(args)
    if int(world or 1) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} does not match WORLD_SIZE={world}", file=sys.stderr)
        return 2
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
