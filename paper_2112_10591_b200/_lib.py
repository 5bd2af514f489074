"""ctypes loader for libieds.so (the C ABI in include/ieds.h).  Argument marshalling only.

The library is built in-tree (paper_2112_10591_b200/lib/libieds.so) by
`paper_2112_10591_b200.build.build_library()` / `__graft_entry__.build()`.  There is no
fallback: if the library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libieds.so")

IEDS_OK = 0
IEDS_EINVAL = -1
IEDS_ERANGE = -2
IEDS_ECAPACITY = -3
IEDS_EORDER = -4
IEDS_ECUDA = -5
IEDS_ENOMEM = -6
IEDS_NO_EDGE = 0xFFFFFFFF

# every symbol include/ieds.h declares
EXPORTS = (
    "ieds_create", "ieds_destroy", "ieds_build_batch", "ieds_build_batch_host", "ieds_sync",
    "ieds_window_offsets", "ieds_window_count", "ieds_stream_create", "ieds_stream_closing", "ieds_stream_push",
    "ieds_stream_flush", "ieds_stream_destroy", "ieds_pipeline_create", "ieds_pipeline_closing", "ieds_pipeline_push",
    "ieds_pipeline_flush", "ieds_pipeline_destroy", "ieds_fwl_batch", "ieds_flow_create", "ieds_flow_destroy", "ieds_flow_reset",
    "ieds_flow_step", "ieds_flow_launches_per_step", "ieds_launches_per_batch", "ieds_profile_enable", "ieds_profile_read", "ieds_strerror", "ieds_alpha_from_dsat", "ieds_version",
)


class IedsFlowConfig(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("levels", ctypes.c_int32),
        ("iterations", ctypes.c_int32 * 8),
        ("lambda_", ctypes.c_double * 8),
        ("gamma", ctypes.c_double),
        ("scale", ctypes.c_double),
        ("device", ctypes.c_int32),
    ]


class IedsConfig(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("n_d", ctypes.c_int32),
        ("n_f", ctypes.c_int32),
        ("alpha", ctypes.c_double),
        ("chunk_windows", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("transfer", ctypes.c_int32),
        ("bound", ctypes.c_double),
        ("out_format", ctypes.c_int32),
    ]


IEDS_FLAG_EXACT_EDT = 1
IEDS_FLAG_TEST_BANDS = 2   # testing aid: 64-row frame bands even when the frame fits one CTA
TRANSFERS = {"invexp": 0, "linear": 1, "bounded": 2, "log": 3}   # IEDS_TRANSFER_*
OUT_FORMATS = {"f32": 0, "u8": 1, "f16": 2}                         # IEDS_OUT_*


class IedsError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        msg = load().ieds_strerror(code).decode()
        super().__init__(f"{what}: {msg} ({code})" if what else f"{msg} ({code})")


class IedsRangeError(IedsError):
    """An event lies outside the frame (device-detected, latched)."""


class IedsOrderError(IedsError):
    """Window offsets not non-decreasing or out of [0, n_events]."""


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.ieds_create.argtypes = [ctypes.POINTER(IedsConfig), ctypes.POINTER(P)]
    lib.ieds_create.restype = ctypes.c_int
    lib.ieds_destroy.argtypes = [P]
    lib.ieds_destroy.restype = None
    lib.ieds_build_batch.argtypes = [P, P, P, i64, i32, P, P, P, P, P, P]
    lib.ieds_build_batch.restype = ctypes.c_int
    lib.ieds_build_batch_host.argtypes = [P, P, P, i32, P]
    lib.ieds_build_batch_host.restype = ctypes.c_int
    lib.ieds_window_offsets.argtypes = [P, P, i64, i64, i64, i32, P, P]
    lib.ieds_window_offsets.restype = ctypes.c_int
    lib.ieds_window_count.argtypes = [P, P, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i32), P]
    lib.ieds_window_count.restype = ctypes.c_int
    lib.ieds_stream_create.argtypes = [P, i64, ctypes.POINTER(P)]
    lib.ieds_stream_create.restype = ctypes.c_int
    lib.ieds_stream_closing.argtypes = [P, i64, i64]
    lib.ieds_stream_closing.restype = i64
    lib.ieds_stream_push.argtypes = [P, P, P, i64, P, i32, ctypes.POINTER(i32)]
    lib.ieds_stream_push.restype = ctypes.c_int
    lib.ieds_stream_flush.argtypes = [P, P, i32, ctypes.POINTER(i32)]
    lib.ieds_stream_flush.restype = ctypes.c_int
    lib.ieds_stream_destroy.argtypes = [P]
    lib.ieds_stream_destroy.restype = None
    lib.ieds_pipeline_create.argtypes = [P, P, i64, ctypes.POINTER(P)]
    lib.ieds_pipeline_create.restype = ctypes.c_int
    lib.ieds_pipeline_closing.argtypes = [P, i64, i64]
    lib.ieds_pipeline_closing.restype = i64
    lib.ieds_pipeline_push.argtypes = [P, P, P, i64, P, P, P, i32, ctypes.POINTER(i32)]
    lib.ieds_pipeline_push.restype = ctypes.c_int
    lib.ieds_pipeline_flush.argtypes = [P, P, P, P, i32, ctypes.POINTER(i32)]
    lib.ieds_pipeline_flush.restype = ctypes.c_int
    lib.ieds_pipeline_destroy.argtypes = [P]
    lib.ieds_pipeline_destroy.restype = None
    lib.ieds_fwl_batch.argtypes = [P, P, P, P, P, i64, i32, P, P, i64, P, P, P, P, P]
    lib.ieds_fwl_batch.restype = ctypes.c_int
    lib.ieds_flow_create.argtypes = [P, P]
    lib.ieds_flow_create.restype = ctypes.c_int
    lib.ieds_flow_destroy.argtypes = [P]
    lib.ieds_flow_destroy.restype = None
    lib.ieds_flow_reset.argtypes = [P]
    lib.ieds_flow_reset.restype = ctypes.c_int
    lib.ieds_flow_step.argtypes = [P, P, P, P, P, P]
    lib.ieds_flow_step.restype = ctypes.c_int
    lib.ieds_flow_launches_per_step.argtypes = [P]
    lib.ieds_flow_launches_per_step.restype = i64
    lib.ieds_sync.argtypes = [P, P]
    lib.ieds_sync.restype = ctypes.c_int
    lib.ieds_launches_per_batch.argtypes = [P, i32]
    lib.ieds_launches_per_batch.restype = i64
    lib.ieds_profile_enable.argtypes = [P, ctypes.c_int]
    lib.ieds_profile_enable.restype = ctypes.c_int
    lib.ieds_profile_read.argtypes = [P, ctypes.POINTER(f64), ctypes.POINTER(i64), ctypes.POINTER(f64),
                                      ctypes.POINTER(i64)]
    lib.ieds_profile_read.restype = ctypes.c_int
    lib.ieds_strerror.argtypes = [ctypes.c_int]
    lib.ieds_strerror.restype = ctypes.c_char_p
    lib.ieds_alpha_from_dsat.argtypes = [f64]
    lib.ieds_alpha_from_dsat.restype = f64
    lib.ieds_version.argtypes = []
    lib.ieds_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(code: int, what: str = "") -> None:
    if code == IEDS_OK:
        return
    if code == IEDS_ERANGE:
        raise IedsRangeError(code, what)
    if code == IEDS_EORDER:
        raise IedsOrderError(code, what)
    raise IedsError(code, what)
