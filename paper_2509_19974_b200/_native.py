"""ctypes binding of libqxcorr_b200.so (the C ABI in include/qxcorr_b200.h).

The shared library is built in-tree by ``make -C paper_2509_19974_b200/csrc``
(or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing, every GPU entry point raises ImportError -- the product path never
silently degrades to a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QX_NATIVE_LIB: an alternative build of the same library (A/B and
# -DQX_TC_TIMING instrumentation builds under tools/ab/)
LIB_PATH = os.environ.get("QX_NATIVE_LIB") or os.path.join(_HERE, "_native", "libqxcorr_b200.so")

# qx_status (include/qxcorr_b200.h)
QX_OK = 0
QX_ERR_INVALID = 1
QX_DEGENERATE_QUANTIZATION = 2
QX_DEGENERATE_INPUT = 3
QX_BOUND_EXCEEDED = 4
QX_INTERNAL_OVERFLOW = 5
QX_ERR_CUDA = 6
QX_ERR_UNSUPPORTED = 7
QX_ERR_NOMEM = 8
QX_ERR_NONFINITE = 9

QX_F32, QX_F64, QX_I64 = 0, 1, 2
QX_Q_SIGN, QX_Q_UNIFORM, QX_Q_CUSTOM, QX_Q_CODES = 0, 1, 2, 3
PATHS = {"auto": 0, "ntt": 1, "direct": 2, "tc": 2, "popc": 3}
PROFILE_KINDS = 10  # qxcorr_b200.h QX_PROFILE_KINDS
ABI_VERSION = 4  # qxcorr_b200.h QX_ABI_VERSION

RF_DEGENERATE_X = 1
RF_DEGENERATE_Y = 2
RF_NONFINITE = 4
RF_CODE_RANGE = 8

INT64_MIN = -(1 << 63)
INT64_MAX = (1 << 63) - 1


class QxQuantizer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32), ("k", ctypes.c_int64),
                ("step", ctypes.c_double), ("thresholds", ctypes.c_void_p)]


class QxSignals(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("n", ctypes.c_int64), ("ld", ctypes.c_int64), ("start", ctypes.c_int64)]


class QxResult(ctypes.Structure):
    _fields_ = [("value", ctypes.c_int64), ("lag", ctypes.c_int64), ("ties", ctypes.c_int64),
                ("sumsq_x", ctypes.c_int64), ("sumsq_y", ctypes.c_int64), ("nnz_x", ctypes.c_int64),
                ("nnz_y", ctypes.c_int64), ("flags", ctypes.c_int32), ("status", ctypes.c_int32)]


class QxProfile(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("count", ctypes.c_int64 * PROFILE_KINDS),
                ("ms", ctypes.c_double * PROFILE_KINDS)]


RESULT_DTYPE = np.dtype([("value", "<i8"), ("lag", "<i8"), ("ties", "<i8"), ("sumsq_x", "<i8"),
                         ("sumsq_y", "<i8"), ("nnz_x", "<i8"), ("nnz_y", "<i8"), ("flags", "<i4"),
                         ("status", "<i4")])
assert RESULT_DTYPE.itemsize == ctypes.sizeof(QxResult) == 64

# every symbol include/qxcorr_b200.h declares
EXPORTS = (
    "qx_abi_version", "qx_status_string", "qx_context_create", "qx_context_destroy",
    "qx_context_last_error", "qx_context_set_option", "qx_quantizer_thresholds", "qx_quantize", "qx_xcorr_full",
    "qx_estimate_batch", "qx_estimate_batch_host", "qx_estimate_sweep", "qx_estimate_sweep_host", "qx_template_search", "qx_decode_pcm16",
    "qx_profile_begin",
    "qx_profile_end",
    "qx_profile_kind_name", "qx_summary_reduce_nccl", "qx_template_search_nccl", "qx_estimate_batch_nccl",
    "qx_comm_rank_size", "qx_plan_create", "qx_plan_run", "qx_plan_run_host", "qx_plan_path", "qx_plan_destroy",
    "qx_quantize_packed", "qx_packed_words",
)

_lib = None
_lib_lock = threading.Lock()
_contexts: dict[int, ctypes.c_void_p] = {}


def load():
    """Load (once) and prototype the native library; ImportError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2509_19974_b200/csrc` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.qx_abi_version.restype = ctypes.c_int
        L.qx_status_string.argtypes = [st]
        L.qx_status_string.restype = ctypes.c_char_p
        L.qx_context_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
        L.qx_context_create.restype = st
        L.qx_context_destroy.argtypes = [vp]
        L.qx_context_destroy.restype = None
        L.qx_context_last_error.argtypes = [vp]
        L.qx_context_last_error.restype = ctypes.c_char_p
        L.qx_context_set_option.argtypes = [vp, ctypes.c_char_p, i64]
        L.qx_context_set_option.restype = st
        qp, sp = ctypes.POINTER(QxQuantizer), ctypes.POINTER(QxSignals)
        L.qx_quantizer_thresholds.argtypes = [qp, ctypes.c_int, vp]
        L.qx_quantizer_thresholds.restype = st
        L.qx_quantize_packed.argtypes = [vp, qp, sp, i64, ctypes.c_int, vp, vp, vp, vp, vp]
        L.qx_quantize_packed.restype = st
        L.qx_packed_words.argtypes = [i64, ctypes.c_int]
        L.qx_packed_words.restype = i64
        L.qx_quantize.argtypes = [vp, qp, sp, i64, vp, vp, vp, vp]
        L.qx_quantize.restype = st
        L.qx_xcorr_full.argtypes = [vp, sp, sp, i64, qp, qp, vp, vp, st, vp]
        L.qx_xcorr_full.restype = st
        L.qx_estimate_batch.argtypes = [vp, sp, sp, i64, qp, qp, i64, i64, st, vp, vp]
        L.qx_estimate_batch.restype = st
        L.qx_estimate_batch_host.argtypes = [vp, sp, sp, i64, qp, qp, i64, i64, st, vp]
        L.qx_estimate_batch_host.restype = st
        L.qx_estimate_sweep_host.argtypes = [vp, sp, sp, i64, i64, qp, qp, i64, i64, st, vp]
        L.qx_estimate_sweep_host.restype = st
        L.qx_estimate_sweep.argtypes = [vp, sp, sp, i64, i64, qp, qp, i64, i64, st, vp, vp]
        L.qx_estimate_sweep.restype = st
        L.qx_template_search.argtypes = [vp, sp, sp, qp, qp, i64, st, vp, vp]
        L.qx_template_search.restype = st
        L.qx_summary_reduce_nccl.argtypes = [vp, vp, vp, vp]
        L.qx_summary_reduce_nccl.restype = st
        L.qx_template_search_nccl.argtypes = [vp, sp, sp, qp, qp, i64, st, vp, vp, vp]
        L.qx_template_search_nccl.restype = st
        L.qx_estimate_batch_nccl.argtypes = [vp, sp, sp, i64, qp, qp, i64, i64, st, vp, vp, vp, vp]
        L.qx_estimate_batch_nccl.restype = st
        L.qx_comm_rank_size.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.qx_comm_rank_size.restype = st
        L.qx_plan_create.argtypes = [vp, sp, sp, i64, qp, qp, i64, i64, st, ctypes.POINTER(vp)]
        L.qx_plan_create.restype = st
        L.qx_plan_run.argtypes = [vp, vp, vp, vp, vp]
        L.qx_plan_run.restype = st
        L.qx_plan_run_host.argtypes = [vp, vp, vp, vp]
        L.qx_plan_run_host.restype = st
        L.qx_plan_path.argtypes = [vp]
        L.qx_plan_path.restype = ctypes.c_int
        L.qx_plan_destroy.argtypes = [vp]
        L.qx_plan_destroy.restype = None
        L.qx_decode_pcm16.argtypes = [vp, vp, i64, vp, vp]
        L.qx_decode_pcm16.restype = st
        L.qx_profile_begin.argtypes = [vp, ctypes.c_int]
        L.qx_profile_begin.restype = st
        L.qx_profile_end.argtypes = [vp, ctypes.POINTER(QxProfile)]
        L.qx_profile_end.restype = st
        L.qx_profile_kind_name.argtypes = [ctypes.c_int]
        L.qx_profile_kind_name.restype = ctypes.c_char_p
        # (an A/B build named by QX_NATIVE_LIB may predate the current ABI)
        assert L.qx_abi_version() == ABI_VERSION or os.environ.get("QX_NATIVE_LIB")
        _lib = L
    return _lib


def context(device: int | None = None) -> ctypes.c_void_p:
    """Per-device native context (created on first use)."""
    import torch

    if device is None:
        device = torch.cuda.current_device()
    ctx = _contexts.get(device)
    if ctx is None:
        L = load()
        with _lib_lock:
            ctx = _contexts.get(device)
            if ctx is None:
                torch.cuda.init()
                ctx = ctypes.c_void_p()
                check(L.qx_context_create(device, ctypes.byref(ctx)), None)
                _contexts[device] = ctx
    return ctx


def set_option(name: str, value: int, device: int | None = None) -> None:
    """qx_context_set_option on the device's context (tuning / measurement
    knobs; defaults come from the QX_* environment at context creation)."""
    ctx = context(device)
    check(load().qx_context_set_option(ctx, name.encode(), int(value)), ctx)


class option:
    """Context manager: set a context option, restore it on exit."""

    DEFAULTS = {"sweep_restage": 1, "sweep_compute": 1, "popc": 1, "popc_timing": 0, "tc_f4": 1, "sweep_lanes": 0,
                "sweep_chunks": 0, "sweep_taper": 2, "sweep_even": 0, "chunk_pairs": 0, "zero_copy": 1}

    def __init__(self, name: str, value: int, device: int | None = None, restore: int | None = None):
        self.name, self.value, self.device = name, value, device
        self.restore = self.DEFAULTS[name] if restore is None else restore

    def __enter__(self):
        set_option(self.name, self.value, self.device)
        return self

    def __exit__(self, *exc):
        set_option(self.name, self.restore, self.device)
        return False


class NativeError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def check(status: int, ctx) -> None:
    if status == QX_OK:
        return
    L = load()
    msg = L.qx_context_last_error(ctx).decode() if ctx is not None else ""
    if not msg:
        msg = L.qx_status_string(status).decode()
    raise NativeError(status, msg)


def thresholds(q: QxQuantizer, dtype: int, k: int) -> np.ndarray:
    out = np.empty(2 * k, dtype=np.float64)
    check(load().qx_quantizer_thresholds(ctypes.byref(q), dtype, out.ctypes.data), None)
    return out


class profile:
    """Context manager: count (and optionally event-time) every library
    kernel launched inside the block; ``.result`` = {kind: (count, ms)}."""

    def __init__(self, timed: bool = True, device=None):
        self.timed = timed
        self.device = device
        self.result = None
        self.launches = 0

    def __enter__(self):
        self.ctx = context(self.device)
        check(load().qx_profile_begin(self.ctx, int(self.timed)), self.ctx)
        return self

    def __exit__(self, *exc):
        out = QxProfile()
        check(load().qx_profile_end(self.ctx, ctypes.byref(out)), self.ctx)
        L = load()
        self.launches = int(out.launches)
        self.result = {L.qx_profile_kind_name(i).decode(): (int(out.count[i]), float(out.ms[i]))
                       for i in range(PROFILE_KINDS) if out.count[i]}
        return False
