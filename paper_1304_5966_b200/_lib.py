"""ctypes binding of libswb.so (include/swb.h).

The library is built in-tree (paper_1304_5966_b200/libswb.so) by
__graft_entry__.build() / `make -C paper_1304_5966_b200/csrc`.  Loading fails
loudly (DeviceUnavailable) when the library is missing or no sm_100 device is
visible: there is no CPU fallback on the product path.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import DeviceUnavailable, ScoreMismatch, WorkerPanic

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SWB_LIB", _HERE / "libswb.so"))

SWB_OK, SWB_EINVAL, SWB_ECUDA, SWB_ERANGE, SWB_EUNSUPPORTED, SWB_EMISMATCH = 0, -1, -2, -3, -4, -5
BORDER_LOCAL, BORDER_RESTRICTED, BORDER_FREE, BORDER_CONTINUE, BORDER_CHARGE = range(5)
TRACK_NONE, TRACK_MIN, TRACK_MAX = 0, 1, 2
NEG_INF_REF = -(2 ** 61)
NEG_REPORT = -(2 ** 29)

c_i32, c_i64, c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p


class Scheme(ctypes.Structure):
    _fields_ = [("k", c_i32), ("sub", c_i32 * 1024), ("gap_open", c_i32), ("gap_extend", c_i32),
                ("max_sub", c_i32)]


class PassDesc(ctypes.Structure):
    _fields_ = [("seq1", c_i32), ("seq2", c_i32), ("off1", c_i64), ("len1", c_i64),
                ("off2", c_i64), ("len2", c_i64), ("rev1", c_i32), ("rev2", c_i32),
                ("border", c_i32), ("clamp_zero", c_i32), ("track", c_i32), ("has_band", c_i32),
                ("band_lo", c_i64), ("band_hi", c_i64), ("prune", c_i32),
                ("want_final_rows", c_i32), ("final_row_h", c_p), ("final_row_f", c_p),
                ("row_offset", c_i64), ("prune_target", c_i64), ("corner_i", c_i64),
                ("corner_j", c_i64), ("ext_in_buf", ctypes.c_uint64),
                ("ext_in_progress", ctypes.c_uint64), ("ext_out_buf", ctypes.c_uint64),
                ("ext_out_progress", ctypes.c_uint64), ("rows_after", c_i64),
                ("bound_write", c_i32), ("bound_read", c_i32), ("bound_offset", c_i64),
                ("shared_best", ctypes.c_uint64)]


class PassOut(ctypes.Structure):
    _fields_ = [("best_score", c_i64), ("best_i", c_i64), ("best_j", c_i64),
                ("cells_executed", c_i64), ("tiles_total", c_i64), ("tiles_executed", c_i64),
                ("tiles_pruned", c_i64), ("tiles_banded_out", c_i64), ("kernel_ms", ctypes.c_double),
                ("kernel", c_i32), ("rows_per_lane", c_i32)]


class Subproblem(ctypes.Structure):
    _fields_ = [("si", c_i64), ("sj", c_i64), ("ei", c_i64), ("ej", c_i64), ("expected", c_i64),
                ("start_vgap", c_i32), ("end_vgap", c_i32), ("use_bounds", c_i32), ("pad", c_i32),
                ("prefix", c_i64), ("suffix", c_i64)]


class Crossing(ctypes.Structure):
    _fields_ = [("mid_i", c_i64), ("mid_j", c_i64), ("upper", c_i64), ("lower", c_i64),
                ("gap_join", c_i32), ("status", c_i32)]


class IntPeak(ctypes.Structure):
    _fields_ = [("viaddmnmx", ctypes.c_double), ("vimnmx3", ctypes.c_double),
                ("viaddmnmx_relu", ctypes.c_double), ("iadd", ctypes.c_double),
                ("prmt", ctypes.c_double), ("imad", ctypes.c_double),
                ("ms_last", ctypes.c_double), ("sms", c_i32)]


# every symbol include/swb.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "swb_ctx_create", "swb_ctx_destroy", "swb_last_error", "swb_version", "swb_seq_upload",
    "swb_seq_release", "swb_pass", "swb_crossings", "swb_leaves", "swb_measure_int_peak",
    "swb_last_kernel_ms", "swb_launch_count", "swb_set_option", "swb_get_option", "swb_debug_stats",
    "swb_debug_times", "swb_debug_strips", "swb_debug_claims",
    "swb_timer_start", "swb_timer_stop", "swb_flush_l2",
    "swb_boundary_alloc", "swb_boundary_reset", "swb_boundary_free", "swb_ipc_export",
    "swb_ipc_import", "swb_ipc_close", "swb_bounds_reset", "swb_bounds_read", "swb_bounds_device",
)

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libswb.so and declare prototypes (no device is touched)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise DeviceUnavailable(
                f"{LIB_PATH} not found; build it with __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.POINTER
        lib.swb_ctx_create.argtypes = [c_i32]
        lib.swb_ctx_create.restype = c_p
        lib.swb_ctx_destroy.argtypes = [c_p]
        lib.swb_ctx_destroy.restype = None
        lib.swb_last_error.restype = ctypes.c_char_p
        lib.swb_version.restype = c_i32
        lib.swb_seq_upload.argtypes = [c_p, c_p, c_i64, P(c_i32)]
        lib.swb_seq_upload.restype = c_i32
        lib.swb_seq_release.argtypes = [c_p, c_i32]
        lib.swb_seq_release.restype = c_i32
        lib.swb_pass.argtypes = [c_p, P(Scheme), P(PassDesc), c_i32, P(PassOut)]
        lib.swb_pass.restype = c_i32
        lib.swb_crossings.argtypes = [c_p, P(Scheme), c_i32, c_i32, P(Subproblem), c_i32, c_i32,
                                      P(Crossing), P(c_i64)]
        lib.swb_crossings.restype = c_i32
        lib.swb_bounds_reset.argtypes = [c_p, c_i32, c_i32]
        lib.swb_bounds_reset.restype = c_i32
        lib.swb_bounds_read.argtypes = [c_p, c_i32, c_p, c_i64]
        lib.swb_bounds_read.restype = c_i64
        lib.swb_bounds_device.argtypes = [c_p, c_i32, P(ctypes.c_uint64), P(c_i64), P(c_i64)]
        lib.swb_bounds_device.restype = c_i32
        lib.swb_leaves.argtypes = [c_p, P(Scheme), c_i32, c_i32, P(Subproblem), c_i32, c_i32,
                                   c_p, c_p, c_p, c_p]
        lib.swb_leaves.restype = c_i32
        lib.swb_measure_int_peak.argtypes = [c_p, P(IntPeak)]
        lib.swb_measure_int_peak.restype = c_i32
        lib.swb_last_kernel_ms.argtypes = [c_p]
        lib.swb_last_kernel_ms.restype = ctypes.c_double
        lib.swb_launch_count.argtypes = [c_p]
        lib.swb_launch_count.restype = c_i64
        lib.swb_set_option.argtypes = [c_p, ctypes.c_char_p, c_i64]
        lib.swb_set_option.restype = c_i32
        lib.swb_get_option.argtypes = [c_p, ctypes.c_char_p]
        lib.swb_get_option.restype = c_i64
        lib.swb_debug_stats.argtypes = [c_p, c_p, c_i32]
        lib.swb_debug_stats.restype = c_i32
        lib.swb_debug_times.argtypes = [c_p, c_p, c_i32]
        lib.swb_debug_times.restype = c_i32
        lib.swb_debug_strips.argtypes = [c_p, c_p, c_i32]
        lib.swb_debug_strips.restype = c_i32
        lib.swb_debug_claims.argtypes = [c_p, c_p, c_i32]
        lib.swb_debug_claims.restype = c_i32
        lib.swb_timer_start.argtypes = [c_p]
        lib.swb_timer_start.restype = c_i32
        lib.swb_timer_stop.argtypes = [c_p, ctypes.POINTER(ctypes.c_double)]
        lib.swb_timer_stop.restype = c_i32
        lib.swb_flush_l2.argtypes = [c_p, c_i64]
        lib.swb_flush_l2.restype = c_i32
        u64, P64 = ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)
        lib.swb_boundary_alloc.argtypes = [c_p, c_i64, P64, P64]
        lib.swb_boundary_alloc.restype = c_i32
        lib.swb_boundary_reset.argtypes = [c_p, u64]
        lib.swb_boundary_reset.restype = c_i32
        lib.swb_boundary_free.argtypes = [c_p, u64, u64]
        lib.swb_boundary_free.restype = c_i32
        lib.swb_ipc_export.argtypes = [c_p, u64, c_p]
        lib.swb_ipc_export.restype = c_i32
        lib.swb_ipc_import.argtypes = [c_p, c_p, P64]
        lib.swb_ipc_import.restype = c_i32
        lib.swb_ipc_close.argtypes = [c_p, u64]
        lib.swb_ipc_close.restype = c_i32
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().swb_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code onto the reference exception classes."""
    if rc == SWB_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == SWB_ECUDA:
        raise WorkerPanic(msg)
    if rc == SWB_EMISMATCH:
        raise ScoreMismatch(msg)
    raise ValueError(msg)
