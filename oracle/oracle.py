"""ctypes wrapper around the C oracle (oracle/qx_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.  It restates the
reference `qxcorr` hot path on the CPU:

* ``quantize``   -- Quantizer.__call__          (quantize.py:53-65)
* ``xcorr_bf``   -- xcorr_int_bf               (intxcorr.py:96-100)
* ``xcorr_ks``   -- xcorr_int_ks with GMP mpn  (intxcorr.py:103-265)
* ``argmax``     -- argmax_set summary          (estimator.py:50-57)
* ``estimate_batch_f32`` -- estimate() lines 1-5 per pair, threaded over pairs

Parity of this restatement is pinned by tests/test_oracle_golden.py against
vectors produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libqxoracle.so")
_lib = None

KIND = {"sign": 0, "uniform": 1, "custom": 2}

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64


def build() -> str:
    """Compile the oracle (gcc + system libgmp.so.10); idempotent."""
    src = os.path.join(_HERE, "qx_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.qxo_quantize_f64.argtypes = [_f64p, _i64, ctypes.c_int, _i64, ctypes.c_double,
                                       ctypes.c_void_p, _i64p]
        L.qxo_quantize_f32.argtypes = [_f32p, _i64, ctypes.c_int, _i64, ctypes.c_double,
                                       ctypes.c_void_p, _i64p]
        L.qxo_xcorr_bf_window.argtypes = [_i64p, _i64, _i64p, _i64, _i64, _i64, _i64p]
        L.qxo_xcorr_ks.argtypes = [_i64p, _i64, _i64, _i64p, _i64, _i64, _i64p]
        L.qxo_argmax.argtypes = [_i64p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                 ctypes.POINTER(_i64)]
        L.qxo_sumsq.argtypes = [_i64p, _i64]
        L.qxo_sumsq.restype = _i64
        L.qxo_plan_slot_bits.argtypes = [_i64, _i64, _i64]
        L.qxo_estimate_batch_f32.argtypes = [
            _f32p, _i64, _i64, _f32p, _i64, _i64, _i64,
            ctypes.c_int, _i64, ctypes.c_double, ctypes.c_void_p,
            ctypes.c_int, _i64, ctypes.c_double, ctypes.c_void_p,
            _i64, _i64, ctypes.c_int, ctypes.c_int, _i64p]
        _lib = L
    return _lib


def _qparams(q):
    """(kind, k, step, thresholds-array-or-None) from any Quantizer-like object."""
    kind = KIND[q.kind]
    thr = None
    if q.kind == "custom":
        thr = np.ascontiguousarray(np.asarray(q.thresholds, dtype=np.float64))
    step = float(getattr(q, "step", 1.0))
    return kind, int(q.k), step, thr


def quantize(q, values) -> np.ndarray:
    v = np.asarray(values)
    kind, k, step, thr = _qparams(q)
    out = np.empty(v.size, dtype=np.int64)
    tp = thr.ctypes.data if thr is not None else None
    if v.dtype == np.float32:
        rc = lib().qxo_quantize_f32(np.ascontiguousarray(v.ravel()), v.size, kind, k, step, tp, out)
    else:
        rc = lib().qxo_quantize_f64(np.ascontiguousarray(v.ravel(), dtype=np.float64), v.size,
                                    kind, k, step, tp, out)
    if rc:
        raise ValueError(f"oracle quantize failed rc={rc}")
    return out.reshape(v.shape)


def xcorr_bf(u, v, t_lo: int | None = None, t_hi: int | None = None) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    t_lo = 0 if t_lo is None else t_lo
    t_hi = u.size + v.size - 2 if t_hi is None else t_hi
    out = np.empty(t_hi - t_lo + 1, dtype=np.int64)
    rc = lib().qxo_xcorr_bf_window(u, u.size, v, v.size, t_lo, t_hi, out)
    if rc:
        raise ValueError(f"oracle xcorr_bf failed rc={rc}")
    return out


def xcorr_ks(u, v, ku: int, kv: int) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    out = np.empty(u.size + v.size - 1, dtype=np.int64)
    rc = lib().qxo_xcorr_ks(u, u.size, ku, v, v.size, kv, out)
    if rc:
        raise ValueError(f"oracle xcorr_ks failed rc={rc}")
    return out


def argmax(c) -> tuple[int, int, int]:
    """(max value, first index, tie count)."""
    c = np.ascontiguousarray(c, dtype=np.int64)
    m, f, n = _i64(), _i64(), _i64()
    lib().qxo_argmax(c, c.size, ctypes.byref(m), ctypes.byref(f), ctypes.byref(n))
    return m.value, f.value, n.value


def sumsq(c) -> int:
    c = np.ascontiguousarray(c, dtype=np.int64)
    return int(lib().qxo_sumsq(c, c.size))


def slot_bits(n_min: int, ku: int, kv: int) -> int:
    return int(lib().qxo_plan_slot_bits(n_min, ku, kv))


def estimate_batch_f32(x, y, qx, qy, t_lo=None, t_hi=None, *, use_bf=False, threads=1):
    """Per-pair (value, t_first, ties, status) of estimate() lines 1-5.

    x: (B, Nx) float32, y: (B, Ny) float32.  t is the index into the full
    correlogram (lag = first_lag + t).  status 0 ok, 1/2 degenerate x/y.
    """
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    B, nx = x.shape
    _, ny = y.shape
    t_lo = 0 if t_lo is None else t_lo
    t_hi = nx + ny - 2 if t_hi is None else t_hi
    kx, Kx, sx, tx = _qparams(qx)
    ky, Ky, sy, ty = _qparams(qy)
    rec = np.zeros((B, 5), dtype=np.int64)
    rc = lib().qxo_estimate_batch_f32(
        x, nx, nx, y, ny, ny, B, kx, Kx, sx, tx.ctypes.data if tx is not None else None,
        ky, Ky, sy, ty.ctypes.data if ty is not None else None, t_lo, t_hi, int(use_bf),
        int(threads), rec)
    if rc:
        raise ValueError(f"oracle estimate_batch failed rc={rc}")
    return rec[:, :4]
