"""Exact integer cross-correlation on the GPU (full correlogram).

Drop-in for /root/reference/pkg/src/qxcorr/intxcorr.py's ``xcorr_int_bf``
(96-100) and ``xcorr_int_ks`` (259-265): both names return the same
bit-identical int64 ``Correlogram`` (with ``norm_x``/``norm_y``) computed by
the NTT kernels through ``qx_xcorr_full``.  ``_check_coeff_bound`` (89-93)
and ``plan_ks``'s all-zero check (109-110) keep their exceptions.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _device as D
from . import _native as N
from ._call import call
from .errors import DegenerateInput
from .quantize import native_quantizer
from .signals import Correlogram

__all__ = ["xcorr_int_gpu", "xcorr_int_bf", "xcorr_int_ks", "MAX_COEFF_BOUND", "xcorr_full_device"]

MAX_COEFF_BOUND = 1 << 59  # intxcorr.py:50


def _check_coeff_bound(n_min: int, k_u: int, k_v: int) -> None:
    if n_min * k_u * k_v > MAX_COEFF_BOUND:
        raise ValueError("coefficient bound N_min*K_u*K_v exceeds the supported int64 range")


def xcorr_full_device(x, y, qx, qy, x_start=0, y_start=0, path="auto"):
    """values (batch, nx+ny-1) int64 CUDA tensor and per-pair stats records.

    x, y: CUDA tensors (n,) or (batch, n); float rows are quantised with
    qx/qy, int64 rows are codes and qx/qy are then their integer bounds.
    """
    t = D.torch()
    xb = x if x.dim() == 2 else x.unsqueeze(0)
    yb = y if y.dim() == 2 else y.unsqueeze(0)
    batch = xb.shape[0]
    nout = xb.shape[1] + yb.shape[1] - 1
    values = t.empty((batch, nout), dtype=t.int64, device=x.device)
    stats = t.empty((batch, 8), dtype=t.int64, device=x.device)
    nqx, kx = native_quantizer(qx)
    nqy, ky = native_quantizer(qy)
    sx, sy = D.signals(xb, x_start), D.signals(yb, y_start)
    ctx = N.context(x.device.index)
    call(N.load().qx_xcorr_full, ctx, ctypes.byref(sx), ctypes.byref(sy), batch, ctypes.byref(nqx),
         ctypes.byref(nqy), values.data_ptr(), stats.data_ptr(), N.PATHS[path], D.stream_handle())
    return values, stats


def xcorr_int_gpu(u, v) -> Correlogram:
    """sum_m u[m] * v[m+n] over every overlap lag, exact int64 (GPU)."""
    _check_coeff_bound(min(len(u.samples), len(v.samples)), max(u.bound, 1), max(v.bound, 1))
    du = D.as_device(np.asarray(u.samples, dtype=np.int64))
    dv = D.as_device(np.asarray(v.samples, dtype=np.int64))
    values, stats = xcorr_full_device(du, dv, int(u.bound), int(v.bound), int(u.start), int(v.start))
    st = stats[0].cpu().numpy()
    vals = values[0].cpu().numpy()
    first_lag = int(v.start) - (int(u.start) + len(u.samples) - 1)
    return Correlogram(first_lag, vals, norm_x=math.sqrt(int(st[3])), norm_y=math.sqrt(int(st[4])))


def xcorr_int_bf(u, v) -> Correlogram:
    """Reference name (intxcorr.py:96); same exact values as every path."""
    return xcorr_int_gpu(u, v)


def xcorr_int_ks(u, v, mul_backend: str = "auto") -> Correlogram:
    """Reference name (intxcorr.py:259); rejects all-zero input like plan_ks."""
    if not np.asarray(u.samples).any() or not np.asarray(v.samples).any():
        raise DegenerateInput("cannot plan a Kronecker correlation for an all-zero signal")
    return xcorr_int_gpu(u, v)
