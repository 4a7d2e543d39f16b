"""ctypes binding of libsv (include/sv.h).  Argument marshalling only: every step of the
hot path runs in the CUDA kernels behind the C ABI.  There is no CPU fallback -- if the
library is missing or no CUDA device is present, every compute call raises."""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsv.so")

SV_OK, SV_ERR_INVALID_ARG, SV_ERR_UNSUPPORTED, SV_ERR_CUDA, SV_ERR_WORKSPACE = 0, 1, 2, 3, 4
SV_F32, SV_BF16 = 0, 1
SV_SCHED_PER_ROW, SV_SCHED_BATCH_GREEDY = 0, 1
ROW_NAN, ROW_ALL_NEG_INF, ROW_BAD_TOKEN, ROW_DRAFT_ZERO = 1, 2, 4, 8
ROW_PHAT_BAD, ROW_RESID_ZERO, ROW_BAD_GAMMA, ROW_BAD_LATENCY = 16, 32, 64, 128
ROW_FILTER_UNSUPPORTED = 256

EXPORTS = ("sv_workspace_bytes", "sv_status_string", "sv_score", "sv_schedule", "sd_verify",
           "sv_shard_xch_bytes", "sv_shard_score_p1", "sv_shard_score_p2", "sv_shard_score_finish",
           "sv_shard_verify_p1", "sv_shard_verify_p2", "sv_shard_verify_finish", "sd_verify_ragged",
           "sv_profile_workspace_bytes", "sv_profile_build", "sv_filter_workspace_bytes", "sv_score_filtered",
           "sd_verify_filtered", "sv_score_schedule")


class SvLogits(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("stride_b", ctypes.c_int64), ("stride_i", ctypes.c_int64)]


class SvProfile(ctypes.Structure):
    _fields_ = [("s_edges", ctypes.c_void_p), ("n_s", ctypes.c_int32), ("n_a", ctypes.c_int32),
                ("a_edges", ctypes.c_void_p), ("cells", ctypes.c_void_p)]


class SvFilter(ctypes.Structure):
    _fields_ = [("top_k", ctypes.c_int32), ("top_p", ctypes.c_float)]


class SvError(RuntimeError):
    pass


_lib = None


def load(path: str = LIB_PATH):
    """Load libsv.so and declare the C signatures (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libsv.so not built at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, i32, i64, u64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
    sz = ctypes.c_size_t
    lib.sv_workspace_bytes.argtypes = [i32, i32, i32, i32]
    lib.sv_workspace_bytes.restype = sz
    lib.sv_status_string.argtypes = [i32]
    lib.sv_status_string.restype = ctypes.c_char_p
    LP = ctypes.POINTER(SvLogits)
    lib.sv_score.argtypes = [LP, LP, P, i32, i32, i32, f32, f32, ctypes.POINTER(SvProfile),
                             P, P, P, P, P, P, P, P, P, sz, P]
    lib.sv_score.restype = i32
    lib.sv_score_schedule.argtypes = [LP, LP, P, i32, i32, i32, f32, f32, ctypes.POINTER(SvProfile),
                                      P, P, P, P, P, P, P, P, P, i32, i32, P, P, P, P, P, sz, P]
    lib.sv_score_schedule.restype = i32
    lib.sv_schedule.argtypes = [P, i32, i32, P, i32, i32, i32, P, P, P, P, P, sz, P]
    lib.sv_schedule.restype = i32
    lib.sd_verify.argtypes = [LP, LP, P, P, P, P, P, i32, i32, i32, f32, f32, u64, u64, i64,
                              P, P, P, P, P, P, sz, P]
    lib.sd_verify.restype = i32
    lib.sd_verify_ragged.argtypes = [LP, P, i64, P, P, P, P, P, P, i32, i32, i32, f32, f32, u64, u64, P, i64,
                                     P, P, P, P, P, P, sz, P]
    lib.sd_verify_ragged.restype = i32
    FP = ctypes.POINTER(SvFilter)
    lib.sv_filter_workspace_bytes.argtypes = [i32, i32]
    lib.sv_filter_workspace_bytes.restype = sz
    lib.sv_score_filtered.argtypes = [LP, LP, P, i32, i32, i32, f32, f32, FP, ctypes.POINTER(SvProfile), P, P, P, P,
                                      P, P, P, sz, P]
    lib.sv_score_filtered.restype = i32
    lib.sd_verify_filtered.argtypes = [LP, LP, P, P, i32, i32, i32, f32, FP, u64, u64, i64, P, P, P, P, P, P, sz, P]
    lib.sd_verify_filtered.restype = i32
    lib.sv_profile_workspace_bytes.argtypes = [i32, i32, i32, i32]
    lib.sv_profile_workspace_bytes.restype = sz
    lib.sv_profile_build.argtypes = [P, P, P, i32, i32, i32, i32, P, P, P, P, P, P, P, sz, P]
    lib.sv_profile_build.restype = i32
    lib.sv_shard_xch_bytes.argtypes = [i32, i32, i32, i32, i32]
    lib.sv_shard_xch_bytes.restype = sz
    lib.sv_shard_score_p1.argtypes = [LP, LP, P, i32, i32, i32, i64, f32, f32, P, P]
    lib.sv_shard_score_p2.argtypes = [LP, LP, P, i32, i32, i32, f32, f32, P, i32, P, P]
    lib.sv_shard_score_finish.argtypes = [P, i32, i32, i32, i32, i32, f32, f32, ctypes.POINTER(SvProfile), P, P, i32,
                                          P, P, P, P, P, P, P, P, P]
    lib.sv_shard_verify_p1.argtypes = [LP, P, P, i32, i32, i32, i64, f32, P, P]
    lib.sv_shard_verify_p2.argtypes = [LP, LP, P, P, P, P, P, i32, i32, i32, i32, f32, f32, u64, u64, i64, P, i32,
                                       P, P, P, P, sz, P]
    lib.sv_shard_verify_finish.argtypes = [LP, LP, i32, i32, i32, i64, f32, f32, P, i32, i32, P, P, P, P, sz, P]
    for name in ("sv_shard_score_p1", "sv_shard_score_p2", "sv_shard_score_finish", "sv_shard_verify_p1",
                 "sv_shard_verify_p2", "sv_shard_verify_finish"):
        getattr(lib, name).restype = i32
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != SV_OK:
        msg = load().sv_status_string(status).decode()
        raise SvError(f"{what}: {msg} (status {status})")
