"""ctypes binding of libmarsit_b200.so (include/marsit_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the library is missing, importing the package fails
loudly, and without a CUDA device every compute entry point raises CudaError.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("MARSIT_SO") or os.path.join(HERE, "libmarsit_b200.so")

# status codes (include/marsit_b200.h)
OK, EPARAM, ENONFINITE, EPROTOCOL, EUNSUPPORTED, ECUDA, ENCCL = range(7)
N_PHASES = 10
PHASES = ("sign_extract", "exchange", "merge", "allgather", "decode_comp", "export", "dense",
          "coins", "fused_round", "spread_round")

F32, F64 = 0, 1


class MergeInfo(C.Structure):
    _fields_ = [("recv_node", C.c_uint32), ("local_node", C.c_uint32), ("receiver", C.c_uint32),
                ("c_recv", C.c_uint32), ("c_local", C.c_uint32), ("offset_src", C.c_int32),
                ("stage", C.c_uint32)]


class DriverDesc(C.Structure):
    _fields_ = [("dim", C.c_uint64), ("schedule", C.c_void_p), ("dtype", C.c_int),
                ("device", C.c_int), ("nranks", C.c_uint32), ("rank", C.c_uint32),
                ("nccl_id", C.c_void_p), ("bucket_elems", C.c_uint64), ("period", C.c_uint64),
                ("eta_s", C.c_double), ("global_seed", C.c_uint64), ("first_round", C.c_uint64),
                ("transport", C.c_int)]


class CtxDesc(C.Structure):
    _fields_ = [("dim", C.c_uint64), ("schedule", C.c_void_p), ("dtype", C.c_int),
                ("device", C.c_int), ("nranks", C.c_uint32), ("rank", C.c_uint32),
                ("nccl_id", C.c_void_p), ("transport", C.c_int)]


class P2PBuffers(C.Structure):
    """marsit_p2p_buffers (include/marsit_b200.h)."""
    _fields_ = [("bits", C.c_void_p), ("agg", C.c_void_p), ("dense_send", C.c_void_p),
                ("dense_mean", C.c_void_p), ("flags", C.c_void_p)]


class ExchangeLayout(C.Structure):
    _fields_ = [("send", C.c_void_p), ("recv", C.c_void_p), ("block_bytes", C.c_uint64),
                ("gather", C.c_void_p), ("gather_block_bytes", C.c_uint64)]


# Every symbol include/marsit_b200.h declares: name -> (restype, argtypes)
_vp, _u32, _u64, _i32, _dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
_pvp = C.POINTER(C.c_void_p)
class RoundMetrics(C.Structure):
    """marsit_round_metrics (include/marsit_b200.h)."""
    _fields_ = [("round", C.c_uint64), ("valid", C.c_int32), ("full_precision", C.c_int32),
                ("has_matching", C.c_int32), ("rank_local", C.c_int32), ("dim", C.c_uint64),
                ("matches", C.c_uint64), ("matching_rate", C.c_double),
                ("merges", C.c_uint64), ("compared_bits", C.c_uint64),
                ("disagreements", C.c_uint64), ("disagreement_rate", C.c_double),
                ("round_bits", C.c_uint64)]


SIGNATURES = {
    "marsit_schedule_ring": (_i32, [_u32, _pvp]),
    "marsit_schedule_torus": (_i32, [_u32, _u32, _pvp]),
    "marsit_schedule_from_tables": (_i32, [_u32, _u32, _u32, _vp, _vp, _vp, _vp, _pvp]),
    "marsit_schedule_info": (_i32, [_vp, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u32)]),
    "marsit_schedule_tables": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "marsit_schedule_destroy": (None, [_vp]),
    "marsit_schedule_plan": (_i32, [_vp, _u32, _u32, C.POINTER(MergeInfo), C.POINTER(_u32),
                                    C.POINTER(_u32), C.POINTER(_u32)]),
    "marsit_ctx_create": (_i32, [C.POINTER(CtxDesc), _pvp]),
    "marsit_ctx_destroy": (None, [_vp]),
    "marsit_ctx_local_workers": (_i32, [_vp, C.POINTER(_u32), C.POINTER(_u32)]),
    "marsit_sign_round": (_i32, [_vp, _u64, _dbl, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "marsit_dense_round": (_i32, [_vp, _u64, _vp, _vp, _vp, _vp, _vp]),
    "marsit_round": (_i32, [_vp, _u64, _u64, _dbl, _u64, _vp, _vp, _vp, _vp, _vp,
                            C.POINTER(_i32), _vp]),
    "marsit_allreduce_sign": (_i32, [_vp, _u64, _u64, _vp, _vp, _vp, _vp]),
    "marsit_sign_extract": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "marsit_ctx_exchange_layout": (_i32, [_vp, _i32, C.POINTER(ExchangeLayout)]),
    "marsit_round_phase": (_i32, [_vp, _i32, _u64, _u64, _dbl, _u64, _vp, _vp, _vp, _vp, _vp,
                                  C.POINTER(_i32), _vp]),
    "marsit_merge_signs": (_i32, [_vp, _u32, _vp, _u32, _u64, _u64, _u64, _vp,
                                  C.POINTER(_u64), _i32, _vp]),
    "marsit_bits_account": (_i32, [_vp, _i32, _vp, C.POINTER(_u64), C.POINTER(_u64),
                                   C.POINTER(_u64)]),
    "marsit_ctx_check": (_i32, [_vp, _vp]),
    "marsit_ctx_set_timing": (_i32, [_vp, _i32]),
    "marsit_ctx_set_wait_timeout": (_i32, [_vp, _u64]),
    "marsit_ctx_set_consensus": (_i32, [_vp, _i32]),
    "marsit_ctx_status": (_i32, [_vp]),
    "marsit_driver_set_wait_timeout": (_i32, [_vp, _u64]),
    "marsit_driver_set_consensus": (_i32, [_vp, _i32]),
    "marsit_ctx_set_metrics": (_i32, [_vp, _i32]),
    "marsit_ctx_p2p_buffers": (_i32, [_vp, C.POINTER(P2PBuffers)]),
    "marsit_ctx_set_peers": (_i32, [_vp, C.POINTER(P2PBuffers), _u32]),
    "marsit_driver_p2p_buffers": (_i32, [_vp, _u32, C.POINTER(P2PBuffers)]),
    "marsit_driver_set_peers": (_i32, [_vp, _u32, C.POINTER(P2PBuffers), _u32]),
    "marsit_ipc_handle": (_i32, [_vp, _vp]),
    "marsit_ipc_open": (_i32, [_vp, _i32, C.POINTER(_vp)]),
    "marsit_ipc_close": (_i32, [_vp]),
    "marsit_ssdm_compress": (_i32, [_vp, _u64, _i32, _u64, _u64, _u64, _u64, _vp,
                                    C.POINTER(_dbl), _vp]),
    "marsit_ssdm_decompress": (_i32, [_vp, _u64, _dbl, _i32, _vp, _vp]),
    "marsit_ssdm_allreduce": (_i32, [_vp, _i32, _u64, _u64, _vp, _vp, _vp,
                                     C.POINTER(_u64), C.POINTER(_u64), _vp, _vp]),
    "marsit_ctx_metrics": (_i32, [_vp, C.POINTER(RoundMetrics), _vp]),
    "marsit_driver_set_metrics": (_i32, [_vp, _i32]),
    "marsit_driver_metrics": (_i32, [_vp, C.POINTER(RoundMetrics), _vp]),
    "marsit_ctx_timing": (_i32, [_vp, _vp, _vp, _i32]),
    "marsit_fill_recipe": (_i32, [_i32, _u64, _u64, _u64, _u64, _i32, _vp, _vp]),
    "marsit_nccl_unique_id": (_i32, [_vp]),
    "marsit_driver_create": (_i32, [C.POINTER(DriverDesc), _pvp]),
    "marsit_driver_destroy": (None, [_vp]),
    "marsit_driver_step": (_i32, [_vp, _vp, _vp, _vp, C.POINTER(_i32), _vp]),
    "marsit_driver_compensation": (_i32, [_vp, _u32, _pvp]),
    "marsit_driver_state": (_i32, [_vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u32)]),
    "marsit_driver_save": (_i32, [_vp, C.c_char_p, _vp]),
    "marsit_driver_load": (_i32, [_vp, C.c_char_p, _vp]),
    "marsit_write_params_checkpoint": (_i32, [C.c_char_p, _vp, _u64, _i32, _vp]),
    "marsit_read_params_checkpoint": (_i32, [C.c_char_p, _vp, _u64, _i32, _vp]),
    "marsit_last_error": (C.c_char_p, []),
    "marsit_abi_version": (_i32, []),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(
                f"{SO_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
        L = C.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr_array(ptrs):
    arr = (C.c_void_p * max(len(ptrs), 1))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
