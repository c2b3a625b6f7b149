"""B200-native Marsit sign-round synchronisation (drop-in for the reference's
``marsit::marsit_round`` / ``marsit::allreduce_sign`` path).

This module mirrors the reference's C++ operator API (sync.hpp, allreduce.hpp,
schedule.hpp, merge.hpp) over torch CUDA tensors: same names, same argument
meaning, same error taxonomy (errors.hpp:10-42 -> the exception classes below).
All compute runs in libmarsit_b200.so (hand-written sm_100a kernels) through
its C-ABI; torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _native as N

__all__ = [
    "ParameterError", "NonFiniteError", "ProtocolError", "UnsupportedError", "CudaError",
    "NcclError", "Schedule", "build_ring_schedule", "build_torus_schedule", "SyncConfig",
    "CompensationState", "BitsAccount", "MarsitRoundResult", "AggregateSign", "Context",
    "marsit_round", "allreduce_sign", "pack_signs", "merge_signs", "stream_key", "Driver",
    "write_params_checkpoint", "read_params_checkpoint",
]


# --------------------------------------------------------------------------
# errors.hpp:10-42
# --------------------------------------------------------------------------
class ParameterError(ValueError):
    """marsit::parameter_error"""


class NonFiniteError(ParameterError):
    """marsit::non_finite_error"""


class ProtocolError(RuntimeError):
    """marsit::protocol_error"""


class UnsupportedError(RuntimeError):
    """marsit::unsupported_error"""


class CudaError(RuntimeError):
    """CUDA failure (no device, launch error)."""


class NcclError(RuntimeError):
    """NCCL failure in a multi-rank context."""


_ERRORS = {N.EPARAM: ParameterError, N.ENONFINITE: NonFiniteError, N.EPROTOCOL: ProtocolError,
           N.EUNSUPPORTED: UnsupportedError, N.ECUDA: CudaError, N.ENCCL: NcclError}


def _check(status: int) -> None:
    if status != N.OK:
        msg = N.lib().marsit_last_error().decode(errors="replace")
        raise _ERRORS.get(status, RuntimeError)(msg)


# --------------------------------------------------------------------------
# Schedules (schedule.hpp:12-196)
# --------------------------------------------------------------------------
class Schedule:
    """A compiled marsit_schedule (ring, torus or explicit tables)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        w, s, k = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(N.lib().marsit_schedule_info(self._h, C.byref(w), C.byref(s), C.byref(k)))
        self.workers, self.segments, self.n_steps = w.value, s.value, k.value

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and N._lib is not None:
                N._lib.marsit_schedule_destroy(h)
        except Exception:  # interpreter shutdown
            pass
        self._h = None

    @staticmethod
    def from_tables(workers, segments, phase, send_to, recv_from, segment) -> "Schedule":
        import numpy as np
        ph = np.ascontiguousarray(phase, np.uint8)
        st = np.ascontiguousarray(send_to, np.uint32).ravel()
        rf = np.ascontiguousarray(recv_from, np.uint32).ravel()
        sg = np.ascontiguousarray(segment, np.uint32).ravel()
        out = C.c_void_p()
        _check(N.lib().marsit_schedule_from_tables(
            workers, segments, ph.size, ph.ctypes.data, st.ctypes.data, rf.ctypes.data,
            sg.ctypes.data, C.byref(out)))
        return Schedule(out.value)

    def tables(self):
        import numpy as np
        ph = np.zeros(max(self.n_steps, 1), np.uint8)
        n = max(self.n_steps * self.workers, 1)
        st, rf, sg = (np.zeros(n, np.uint32) for _ in range(3))
        _check(N.lib().marsit_schedule_tables(self._h, ph.ctypes.data, st.ctypes.data,
                                              rf.ctypes.data, sg.ctypes.data))
        k, W = self.n_steps, self.workers
        return (ph[:k], st[:k * W].reshape(k, W), rf[:k * W].reshape(k, W),
                sg[:k * W].reshape(k, W))

    def plan(self, segment: int):
        """The compiled merge DAG of one segment (list of dicts), final node, final count."""
        n, fn, fc = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(N.lib().marsit_schedule_plan(self._h, segment, 0, None, C.byref(n), C.byref(fn),
                                            C.byref(fc)))
        arr = (N.MergeInfo * max(n.value, 1))()
        _check(N.lib().marsit_schedule_plan(self._h, segment, n.value, arr, C.byref(n),
                                            C.byref(fn), C.byref(fc)))
        merges = [dict(recv_node=m.recv_node, local_node=m.local_node, receiver=m.receiver,
                       c_recv=m.c_recv, c_local=m.c_local, offset_src=m.offset_src,
                       stage=m.stage) for m in arr[:n.value]]
        return merges, fn.value, fc.value


def build_ring_schedule(m: int) -> Schedule:
    """schedule.hpp:61-94"""
    out = C.c_void_p()
    _check(N.lib().marsit_schedule_ring(m, C.byref(out)))
    return Schedule(out.value)


def build_torus_schedule(rows: int, cols: int) -> Schedule:
    """schedule.hpp:110-196"""
    out = C.c_void_p()
    _check(N.lib().marsit_schedule_torus(rows, cols, C.byref(out)))
    return Schedule(out.value)


# --------------------------------------------------------------------------
# sync.hpp:23-49
# --------------------------------------------------------------------------
@dataclass
class SyncConfig:
    """full_precision_period = K (None = never); eta_s > 0 (sync.hpp:23-35)."""
    full_precision_period: Optional[int] = None
    eta_s: float = 0.0

    def validate(self) -> None:
        if self.full_precision_period is not None and self.full_precision_period == 0:
            raise ParameterError("SyncConfig: full-precision period must be >= 1")
        if not (self.eta_s > 0.0):
            raise ParameterError("SyncConfig: eta_s must be > 0")


@dataclass
class CompensationState:
    c: "object"  # torch tensor [D]


@dataclass
class BitsAccount:
    per_worker: List[int] = field(default_factory=list)
    reduce_bits: int = 0
    gather_bits: int = 0
    total: int = 0


@dataclass
class MarsitRoundResult:
    global_update: "object"                 # tensor [D] (g_t, identical at every worker)
    compensation: List[CompensationState]
    bits: BitsAccount
    full_precision: bool = False
    aggregate_bits: "object" = None         # int64 tensor [ceil(D/64)] (u64 bit patterns)


@dataclass
class AggregateSign:
    """merge.hpp:16-19: packed bits (int64 tensor of u64 words) + contribution count."""
    bits: "object"
    count: int = 1
    length: int = 0


def stream_key(global_seed: int, purpose: int, worker: int, round_: int, segment: int) -> int:
    """RngStream constructor state (rng.hpp:30-38), computed on the host."""
    M64 = (1 << 64) - 1
    G = 0x9e3779b97f4a7c15

    def mix(z):
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M64
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M64
        return z ^ (z >> 31)

    h = mix((global_seed ^ 0x6a09e667f3bcc909) & M64)
    for v in (purpose, worker + 1, round_ + 1, segment + 1):
        h = mix(h ^ ((v * G) & M64))
    return h


# --------------------------------------------------------------------------
# Context: one marsit_ctx per (D, schedule, dtype, device, rank layout)
# --------------------------------------------------------------------------
def _dtype_code(t):
    import torch
    if t.dtype == torch.float32:
        return N.F32
    if t.dtype == torch.float64:
        return N.F64
    raise ParameterError(f"unsupported dtype {t.dtype} (float32 or float64)")


def _stream_ptr(device):
    import torch
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


@dataclass
class RoundMetrics:
    """Per-round figures of merit computed on the device:
    matching_rate as analysis.hpp:244-253 against the mean of u = g + c
    (trainer.hpp:241-251), the round's BitsAccount total, and the merge
    disagreement counters (coins drawn / bits compared)."""
    round: int
    valid: bool
    full_precision: bool
    has_matching: bool
    rank_local: bool
    dim: int
    matches: int
    matching_rate: Optional[float]
    merges: int
    compared_bits: int
    disagreements: int
    disagreement_rate: float
    round_bits: int

    @classmethod
    def from_c(cls, m) -> "RoundMetrics":
        return cls(int(m.round), bool(m.valid), bool(m.full_precision), bool(m.has_matching),
                   bool(m.rank_local), int(m.dim), int(m.matches),
                   float(m.matching_rate) if m.has_matching else None, int(m.merges),
                   int(m.compared_bits), int(m.disagreements), float(m.disagreement_rate),
                   int(m.round_bits))


class Context:
    """Owns a marsit_ctx (device scratch + compiled plan + optional NCCL comm)."""

    def __init__(self, dim: int, schedule: Schedule, dtype=None, device: int = 0,
                 nranks: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None,
                 external_transport: bool = False, transport: Optional[str] = None):
        """transport (nranks > 1): "p2p" (default: fused over peer memory; call
        set_peers / exchange_p2p_buffers before the first round), "nccl"
        (grouped send/recv + all-gather; needs nccl_id) or "external" (the
        caller moves blocks between marsit_round_phase calls)."""
        import torch
        dtype = dtype or torch.float32
        if transport is None:
            transport = "external" if external_transport else ("nccl" if nccl_id else "p2p")
        self.transport = transport
        self.dim, self.schedule, self.device = int(dim), schedule, int(device)
        self.dtype = dtype
        self.nranks, self.rank = nranks, rank
        desc = N.CtxDesc()
        desc.dim = self.dim
        desc.schedule = schedule._h
        desc.dtype = N.F32 if dtype == torch.float32 else N.F64
        desc.device = self.device
        desc.nranks = nranks
        desc.rank = rank
        desc.transport = {"p2p": 0, "external": 1, "nccl": 2}[transport]
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = C.create_string_buffer(bytes(nccl_id), 128)
            desc.nccl_id = C.cast(self._id_buf, C.c_void_p)
        out = C.c_void_p()
        _check(N.lib().marsit_ctx_create(C.byref(desc), C.byref(out)))
        self._h = out
        first, count = C.c_uint32(), C.c_uint32()
        _check(N.lib().marsit_ctx_local_workers(self._h, C.byref(first), C.byref(count)))
        self.first_worker, self.local_workers = first.value, count.value

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and N._lib is not None:
                N._lib.marsit_ctx_destroy(h)
        except Exception:  # interpreter shutdown
            pass
        self._h = None

    # P2P transport -----------------------------------------------------------
    def p2p_buffers(self) -> "N.P2PBuffers":
        """This rank's buffers to export to its peers (marsit_ctx_p2p_buffers)."""
        b = N.P2PBuffers()
        _check(N.lib().marsit_ctx_p2p_buffers(self._h, C.byref(b)))
        return b

    def set_peers(self, peers: Sequence["N.P2PBuffers"]):
        """All ranks' buffers as mapped in this process, indexed by rank."""
        arr = (N.P2PBuffers * len(peers))(*peers)
        _check(N.lib().marsit_ctx_set_peers(self._h, arr, len(peers)))

    # raw entry points ------------------------------------------------------
    def _ptrs(self, tensors):
        """ctypes pointer array of the tensors' device addresses, cached by
        address (the same buffers are passed every round; building the array
        is most of a small round's Python enqueue time)."""
        key = tuple([x.data_ptr() for x in tensors])
        cache = self.__dict__.setdefault("_ptr_cache", {})
        arr = cache.get(key)
        if arr is None:
            if len(cache) >= 64:
                cache.clear()
            arr = cache[key] = N.ptr_array(key)
        return arr

    def sign_round(self, t, eta_s, seed, grads, comp, comp_out=None, agg_bits=None,
                   update=None, stream=None):
        g = self._ptrs(grads)
        c = self._ptrs(comp)
        co = c if comp_out is None else self._ptrs(comp_out)
        _check(N.lib().marsit_sign_round(
            self._h, t, float(eta_s), seed, g, c, co,
            C.c_void_p(agg_bits.data_ptr() if agg_bits is not None else None),
            C.c_void_p(update.data_ptr() if update is not None else None),
            stream if stream is not None else _stream_ptr(self.device)))

    def dense_round(self, t, grads, comp, mean, comp_out=None, stream=None):
        g = N.ptr_array([x.data_ptr() for x in grads])
        c = N.ptr_array([x.data_ptr() for x in comp])
        co = N.ptr_array([x.data_ptr() for x in (comp_out if comp_out is not None else comp)])
        _check(N.lib().marsit_dense_round(self._h, t, g, c, co, C.c_void_p(mean.data_ptr()),
                                          stream if stream is not None
                                          else _stream_ptr(self.device)))

    def exchange_layout(self, dense: bool = False):
        lay = N.ExchangeLayout()
        _check(N.lib().marsit_ctx_exchange_layout(self._h, int(dense), C.byref(lay)))
        return lay

    def round_phase(self, phase, t, period, eta_s, seed, grads, comp, comp_out=None,
                    agg_bits=None, update=None, stream=None):
        g = N.ptr_array([x.data_ptr() for x in grads])
        c = N.ptr_array([x.data_ptr() for x in comp])
        co = N.ptr_array([x.data_ptr() for x in (comp_out if comp_out is not None else comp)])
        full = C.c_int()
        _check(N.lib().marsit_round_phase(
            self._h, phase, t, 0 if period is None else period, float(eta_s), seed, g, c, co,
            C.c_void_p(agg_bits.data_ptr() if agg_bits is not None else None),
            C.c_void_p(update.data_ptr() if update is not None else None), C.byref(full),
            stream if stream is not None else _stream_ptr(self.device)))
        return bool(full.value)

    def check(self, stream=None):
        _check(N.lib().marsit_ctx_check(self._h, stream if stream is not None
                                        else _stream_ptr(self.device)))

    def bits_account(self, dense: bool) -> BitsAccount:
        pw = (C.c_uint64 * self.schedule.workers)()
        rb, gb, tot = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(N.lib().marsit_bits_account(self._h, int(dense), pw, C.byref(rb), C.byref(gb),
                                           C.byref(tot)))
        return BitsAccount(list(pw), rb.value, gb.value, tot.value)

    def set_timing(self, on: bool):
        _check(N.lib().marsit_ctx_set_timing(self._h, int(on)))

    def set_wait_timeout(self, ms: int):
        """Bound on how long a round may wait for its peers / NCCL before the
        context fails with ProtocolError / NcclError (0 = unbounded)."""
        _check(N.lib().marsit_ctx_set_wait_timeout(self._h, int(ms)))

    def set_consensus(self, on: bool):
        """Opt-in data consensus (allreduce.hpp:32-43): every rank checks the
        aggregate it read against its owners' hashes; check() raises
        ProtocolError on a mismatch."""
        _check(N.lib().marsit_ctx_set_consensus(self._h, int(on)))

    def status(self):
        """Raise the latched failure of the context, if any (no synchronisation)."""
        _check(N.lib().marsit_ctx_status(self._h))

    def set_metrics(self, on: bool):
        """Fused on-device round metrics (matching count in the decode,
        per-merge disagreement totals from the merge)."""
        _check(N.lib().marsit_ctx_set_metrics(self._h, int(on)))

    def metrics(self, stream=None) -> RoundMetrics:
        """The last round's metrics (waits for the stream)."""
        m = N.RoundMetrics()
        _check(N.lib().marsit_ctx_metrics(self._h, C.byref(m), stream if stream is not None
                                          else _stream_ptr(self.device)))
        return RoundMetrics.from_c(m)

    def timing(self, reset: bool = False):
        ms = (C.c_float * N.N_PHASES)()
        ln = (C.c_uint64 * N.N_PHASES)()
        _check(N.lib().marsit_ctx_timing(self._h, ms, ln, int(reset)))
        return {name: (ms[i], ln[i]) for i, name in enumerate(N.PHASES)}

    def sign_extract(self, grads, comp, out, stream=None):
        g = N.ptr_array([x.data_ptr() for x in grads])
        c = N.ptr_array([x.data_ptr() for x in comp])
        _check(N.lib().marsit_sign_extract(self._h, g, c, C.c_void_p(out.data_ptr()),
                                           stream if stream is not None
                                           else _stream_ptr(self.device)))

    def allreduce_sign(self, round_, seed, signs, out, stream=None):
        counts = (C.c_uint32 * self.schedule.segments)()
        _check(N.lib().marsit_allreduce_sign(self._h, round_, seed, C.c_void_p(signs.data_ptr()),
                                             C.c_void_p(out.data_ptr()), counts,
                                             stream if stream is not None
                                             else _stream_ptr(self.device)))
        return list(counts)


_TLS = __import__("threading").local()


def _context_for(dim, sched, dtype, device) -> Context:
    """One cached context per (thread, D, schedule, dtype, device): a context's
    device scratch serves one round at a time, and ctypes releases the GIL
    during the calls, so threads never share one (like the C++ drop-in)."""
    cache = getattr(_TLS, "ctx_cache", None)
    if cache is None:
        cache = _TLS.ctx_cache = {}
    key = (dim, id(sched), dtype, device)
    ctx = cache.get(key)
    if ctx is None or ctx.schedule is not sched:
        ctx = Context(dim, sched, dtype, device)
        cache[key] = ctx
    return ctx


# --------------------------------------------------------------------------
# sync.hpp:60-120  marsit_round
# --------------------------------------------------------------------------
def marsit_round(t: int, cfg: SyncConfig, scaled_grads: Sequence, comp: Sequence,
                 sched: Schedule, global_seed: int, *, inplace: bool = False,
                 want_update: bool = True, check: bool = True) -> MarsitRoundResult:
    """One synchronisation round over M workers resident on this GPU.

    scaled_grads: M CUDA tensors [D] (float32 or float64); comp: M
    CompensationState (or tensors).  Value semantics like the reference:
    the returned compensation tensors are new unless ``inplace=True``.
    ``check`` synchronises and raises NonFiniteError like DenseVector does.
    """
    import torch
    cfg.validate()
    comps = [c.c if isinstance(c, CompensationState) else c for c in comp]
    if len(scaled_grads) != sched.workers or len(comps) != sched.workers:
        raise ParameterError("marsit_round: worker count mismatch")
    dim = scaled_grads[0].numel()
    dt = scaled_grads[0].dtype
    dev = scaled_grads[0].device
    for x in list(scaled_grads) + comps:
        if x.numel() != dim:
            raise ParameterError("marsit_round: dimension mismatch")
        if x.dtype != dt or x.device != dev or not x.is_cuda or not x.is_contiguous():
            raise ParameterError("marsit_round: tensors must be contiguous CUDA tensors of one "
                                 "dtype on one device")
    _dtype_code(scaled_grads[0])
    ctx = _context_for(dim, sched, dt, dev.index or 0)
    outs = comps if inplace else [torch.empty_like(c) for c in comps]
    dense = cfg.full_precision_period is not None and t % cfg.full_precision_period == 0
    update = torch.empty(dim, dtype=dt, device=dev) if (want_update or dense) else None
    if dense:
        ctx.dense_round(t, scaled_grads, comps, update, comp_out=outs)
        agg = None
    else:
        agg = torch.empty((dim + 63) // 64, dtype=torch.int64, device=dev)
        ctx.sign_round(t, cfg.eta_s, global_seed, scaled_grads, comps, comp_out=outs,
                       agg_bits=agg, update=update)
    if check:
        ctx.check()
    return MarsitRoundResult(update, [CompensationState(c) for c in outs],
                             ctx.bits_account(dense), dense, agg)


def allreduce_sign(signs, sched: Schedule, global_seed: int, round_: int, seg_len: int):
    """allreduce.hpp:148-189 on packed signs.

    signs: int64 CUDA tensor [M, S, ceil(L/64)] (u64 words, storage padding 0).
    Returns (aggregate tensor [S, ceil(L/64)], counts[S]) — the consensus that
    every worker holds after the round.
    """
    import torch
    M, S = sched.workers, sched.segments
    nw = (seg_len + 63) // 64
    if tuple(signs.shape) != (M, S, nw):
        raise ParameterError("allreduce_sign: signs must be [workers, segments, words]")
    dim = seg_len * S  # any D with ceil(D/M) == seg_len gives the same segments
    ctx = _context_for(dim, sched, torch.float32, signs.device.index or 0)
    out = torch.empty((S, nw), dtype=torch.int64, device=signs.device)
    counts = ctx.allreduce_sign(round_, global_seed, signs.contiguous(), out)
    return out, counts


def pack_signs(grads: Sequence, comp: Sequence, sched: Schedule):
    """u = g + c, segmented and packed (sync.hpp:71-76, 91-98): int64 [M, S, ceil(L/64)]."""
    import torch
    dim = grads[0].numel()
    ctx = _context_for(dim, sched, grads[0].dtype, grads[0].device.index or 0)
    L = -(-dim // sched.segments)
    out = torch.empty((sched.workers, sched.segments, (L + 63) // 64), dtype=torch.int64,
                      device=grads[0].device)
    ctx.sign_extract(grads, [c.c if isinstance(c, CompensationState) else c for c in comp], out)
    return out


# --------------------------------------------------------------------------
# SSDM baselines (ssdm.hpp:29-56, allreduce.hpp:198-339)
# --------------------------------------------------------------------------
@dataclass
class SsdmPacket:
    """ssdm.hpp:21-24: one sign bit per coordinate + the l2 norm."""
    norm: float
    bits: object  # int64 CUDA tensor, ceil(len/64) u64 words
    length: int


@dataclass
class CascadingAllreduceResult:
    per_worker: list  # the chain estimate of the mean (identical at every worker)
    bits: BitsAccount


@dataclass
class SumSsdmAllreduceResult:
    per_worker: list
    bits: BitsAccount
    max_abs_per_step: list


def ssdm_compress(v, global_seed: int, worker: int, round_: int, segment: int) -> SsdmPacket:
    """ssdm_compress (ssdm.hpp:29-40) with RngStream(seed, ssdm, worker, round, segment)."""
    import torch
    n = v.numel()
    bits = torch.zeros((n + 63) // 64, dtype=torch.int64, device=v.device)
    norm = C.c_double()
    dev = v.device.index or 0
    _check(N.lib().marsit_ssdm_compress(C.c_void_p(v.data_ptr()), n, _dtype_code(v),
                                        global_seed, worker, round_, segment,
                                        C.c_void_p(bits.data_ptr()), C.byref(norm),
                                        _stream_ptr(dev)))
    return SsdmPacket(norm.value, bits, n)


def ssdm_decompress(packet: SsdmPacket, dtype=None):
    """ssdm_decompress (ssdm.hpp:44-56): +-norm per coordinate (0 for norm 0)."""
    import torch
    dtype = dtype or torch.float64
    out = torch.empty(packet.length, dtype=dtype, device=packet.bits.device)
    dev = packet.bits.device.index or 0
    _check(N.lib().marsit_ssdm_decompress(C.c_void_p(packet.bits.data_ptr()), packet.length,
                                          packet.norm, _dtype_code(out),
                                          C.c_void_p(out.data_ptr()), _stream_ptr(dev)))
    return out


def _ssdm(mode: int, vectors: Sequence, sched: Schedule, global_seed: int, round_: int):
    import torch
    if len(vectors) != sched.workers:
        raise ParameterError("allreduce: vector count != schedule workers")
    dim = vectors[0].numel()
    if any(v.numel() != dim for v in vectors):
        raise ParameterError("allreduce: inconsistent dimensions")
    dev = vectors[0].device.index or 0
    ctx = _context_for(dim, sched, vectors[0].dtype, dev)
    out = torch.empty(dim, dtype=vectors[0].dtype, device=vectors[0].device)
    M = sched.workers
    pw = (C.c_uint64 * M)()
    rb, gb = C.c_uint64(), C.c_uint64()
    steps = max(sched.n_steps, 1)
    mx = (C.c_int64 * steps)()
    _check(N.lib().marsit_ssdm_allreduce(ctx._h, mode, round_, global_seed,
                                         N.ptr_array([v.data_ptr() for v in vectors]),
                                         C.c_void_p(out.data_ptr()), pw, C.byref(rb),
                                         C.byref(gb), mx, _stream_ptr(dev)))
    ctx.check()
    bits = BitsAccount(list(pw), rb.value, gb.value, rb.value + gb.value)
    return out, bits, list(mx)[:sched.n_steps]


def cascading_allreduce(vectors: Sequence, sched: Schedule, global_seed: int,
                        round_: int) -> CascadingAllreduceResult:
    """cascading_allreduce (allreduce.hpp:205-262): every hop decompresses,
    adds its own segment and recompresses; ring schedules only."""
    out, bits, _ = _ssdm(0, vectors, sched, global_seed, round_)
    return CascadingAllreduceResult([out] * sched.workers, bits)


def sum_ssdm_allreduce(vectors: Sequence, sched: Schedule, global_seed: int,
                       round_: int) -> SumSsdmAllreduceResult:
    """sum_ssdm_allreduce (allreduce.hpp:275-339): integer sums of the signs on
    the wire (Elias-gamma accounting), estimate = mean of the packets."""
    out, bits, mx = _ssdm(1, vectors, sched, global_seed, round_)
    return SumSsdmAllreduceResult([out] * sched.workers, bits, mx)


def ipc_handle(ptr: int) -> bytes:
    """64-byte CUDA IPC handle of a device allocation (marsit_ipc_handle)."""
    buf = C.create_string_buffer(64)
    _check(N.lib().marsit_ipc_handle(C.c_void_p(ptr), buf))
    return buf.raw


def ipc_open(handle: bytes, device: int) -> int:
    """Map a peer allocation into this process (marsit_ipc_open)."""
    out = C.c_void_p()
    _check(N.lib().marsit_ipc_open(C.create_string_buffer(bytes(handle), 64), device,
                                   C.byref(out)))
    return out.value


def _exchange_tables(mine, rank: int, device: int, set_peers, group=None):
    import torch.distributed as dist
    names = ("bits", "agg", "dense_send", "dense_mean", "flags")
    handles = {k: ipc_handle(getattr(mine, k)) for k in names}
    world = [None] * dist.get_world_size(group)
    dist.all_gather_object(world, handles, group=group)
    table, opened = [], []
    for q, h in enumerate(world):
        b = N.P2PBuffers()
        for k in names:
            if q == rank:
                setattr(b, k, getattr(mine, k))
            else:
                ptr = ipc_open(h[k], device)
                opened.append(ptr)
                setattr(b, k, ptr)
        table.append(b)
    set_peers(table)
    return opened


def exchange_p2p_buffers(ctx: "Context", group=None):
    """Multi-process setup of a P2P-transport context over torch.distributed:
    every rank exports its buffers as IPC handles, maps the others' and hands
    the full table to ctx.set_peers.  Returns the mapped pointers (close them
    with marsit_ipc_close when the context is gone)."""
    return _exchange_tables(ctx.p2p_buffers(), ctx.rank, ctx.device, ctx.set_peers, group)


def merge_signs(received: AggregateSign, local: AggregateSign, key: int, used: int = 0):
    """merge.hpp:34-58 on the device: returns (AggregateSign, draws consumed)."""
    import torch
    if received.length != local.length:
        raise ProtocolError("merge_signs: bit length mismatch")
    L = received.length
    out = torch.zeros_like(received.bits)
    consumed = C.c_uint64()
    dev = received.bits.device.index or 0
    _check(N.lib().marsit_merge_signs(
        C.c_void_p(received.bits.data_ptr()), received.count, C.c_void_p(local.bits.data_ptr()),
        local.count, L, key, used, C.c_void_p(out.data_ptr()), C.byref(consumed), dev,
        _stream_ptr(dev)))
    torch.cuda.synchronize(dev)
    return AggregateSign(out, received.count + local.count, L), consumed.value


def fill_recipe(out, recipe: int, seed: int, worker: int, round_: int) -> None:
    """Synthetic inputs on the device (SURVEY §8c dyadic = 0, §8d correlated = 1)."""
    _check(N.lib().marsit_fill_recipe(recipe, seed, worker, round_, out.numel(),
                                      _dtype_code(out), C.c_void_p(out.data_ptr()),
                                      _stream_ptr(out.device.index or 0)))


class Driver:
    """Multi-step sync driver (marsit_driver_*): the per-round sync part of the
    reference trainer (trainer.hpp:184-307) — device-resident compensation
    carried across rounds, dense cadence K, fused replica update x -= g_t,
    cumulative bits, buckets (seed_b = mix(seed ^ (b+1)*gamma) when > 1), and
    checkpoint/resume of (t, cum_bits, compensation)."""

    def __init__(self, dim: int, schedule: Schedule, *, eta_s: float, global_seed: int,
                 period: Optional[int] = None, bucket_elems: int = 0, dtype=None,
                 device: int = 0, first_round: int = 0, nranks: int = 1, rank: int = 0,
                 nccl_id: Optional[bytes] = None, transport: str = "p2p"):
        """transport (nranks > 1): "p2p" (default; exchange every bucket's
        buffers with set_peers / exchange_p2p_buffers first) or "nccl"."""
        import torch
        dtype = dtype or torch.float32
        if period == 0:
            raise ParameterError("SyncConfig: full-precision period must be >= 1")
        self.dim, self.schedule, self.device, self.dtype = int(dim), schedule, device, dtype
        d = N.DriverDesc()
        d.dim = self.dim
        d.schedule = schedule._h
        d.dtype = N.F32 if dtype == torch.float32 else N.F64
        d.device = device
        d.nranks = nranks
        d.rank = rank
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = C.create_string_buffer(bytes(nccl_id), 128)
            d.nccl_id = C.cast(self._id_buf, C.c_void_p)
        d.bucket_elems = bucket_elems
        d.period = 0 if period is None else int(period)
        d.eta_s = float(eta_s)
        d.global_seed = global_seed
        d.first_round = first_round
        d.transport = {"p2p": 0, "nccl": 2}[transport]
        out = C.c_void_p()
        _check(N.lib().marsit_driver_create(C.byref(d), C.byref(out)))
        self._h = out
        self.local_workers = schedule.workers // nranks
        self.rank, self.nranks, self.transport = rank, nranks, transport

    def p2p_buffers(self, bucket: int) -> "N.P2PBuffers":
        b = N.P2PBuffers()
        _check(N.lib().marsit_driver_p2p_buffers(self._h, bucket, C.byref(b)))
        return b

    def set_peers(self, bucket: int, peers: Sequence["N.P2PBuffers"]):
        arr = (N.P2PBuffers * len(peers))(*peers)
        _check(N.lib().marsit_driver_set_peers(self._h, bucket, arr, len(peers)))

    def exchange_p2p_buffers(self, group=None):
        """CUDA IPC exchange of every bucket's buffers over torch.distributed."""
        opened = []
        for b in range(self.state()["buckets"]):
            opened += _exchange_tables(self.p2p_buffers(b), self.rank, self.device,
                                       lambda tab, b=b: self.set_peers(b, tab), group)
        return opened

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value and N._lib is not None:
                N._lib.marsit_driver_destroy(h)
        except Exception:
            pass
        self._h = None

    def step(self, grads, params=None, update=None, stream=None):
        g = N.ptr_array([x.data_ptr() for x in grads])
        pp = N.ptr_array([x.data_ptr() for x in params]) if params is not None else None
        full = C.c_int()
        _check(N.lib().marsit_driver_step(
            self._h, g, pp, C.c_void_p(update.data_ptr() if update is not None else None),
            C.byref(full), stream if stream is not None else _stream_ptr(self.device)))
        return bool(full.value)

    def compensation(self, i: int):
        """A torch view of local worker i's device compensation (D elements)."""
        import torch
        ptr = C.c_void_p()
        _check(N.lib().marsit_driver_compensation(self._h, i, C.byref(ptr)))
        esize = 4 if self.dtype == torch.float32 else 8
        return _device_view(ptr.value, self.dim, self.dtype, self.device, esize)

    def state(self):
        t, bits, nb = C.c_uint64(), C.c_uint64(), C.c_uint32()
        _check(N.lib().marsit_driver_state(self._h, C.byref(t), C.byref(bits), C.byref(nb)))
        return {"next_round": t.value, "cum_bits": bits.value, "buckets": nb.value}

    def set_metrics(self, on: bool):
        _check(N.lib().marsit_driver_set_metrics(self._h, int(on)))

    def set_wait_timeout(self, ms: int):
        _check(N.lib().marsit_driver_set_wait_timeout(self._h, int(ms)))

    def set_consensus(self, on: bool):
        _check(N.lib().marsit_driver_set_consensus(self._h, int(on)))

    def metrics(self) -> "RoundMetrics":
        """Last step's metrics summed over the buckets (trainer.hpp:278-281)."""
        m = N.RoundMetrics()
        _check(N.lib().marsit_driver_metrics(self._h, C.byref(m), _stream_ptr(self.device)))
        return RoundMetrics.from_c(m)

    def save(self, path: str):
        _check(N.lib().marsit_driver_save(self._h, path.encode(), _stream_ptr(self.device)))

    def load(self, path: str):
        _check(N.lib().marsit_driver_load(self._h, path.encode(), _stream_ptr(self.device)))


def _device_view(ptr: int, n: int, dtype, device: int, esize: int):
    """Zero-copy torch tensor over device memory owned by the library."""
    import torch

    class _Holder:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": "<f4" if esize == 4 else "<f8",
            "data": (ptr, False), "version": 3, "strides": None}
    return torch.as_tensor(_Holder(), device=f"cuda:{device}")


def write_params_checkpoint(path: str, params) -> None:
    """Reference checkpoint format (checkpoint.hpp:18-91) from a device vector."""
    _check(N.lib().marsit_write_params_checkpoint(path.encode(), C.c_void_p(params.data_ptr()),
                                                  params.numel(), _dtype_code(params),
                                                  _stream_ptr(params.device.index or 0)))


def read_params_checkpoint(path: str, params) -> None:
    _check(N.lib().marsit_read_params_checkpoint(path.encode(), C.c_void_p(params.data_ptr()),
                                                 params.numel(), _dtype_code(params),
                                                 _stream_ptr(params.device.index or 0)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(N.lib().marsit_nccl_unique_id(buf))
    return buf.raw


# fail loudly at import if the native library is absent
N.lib()
