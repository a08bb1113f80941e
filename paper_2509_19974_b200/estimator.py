"""Time-difference estimation (Alg. 1) on the GPU -- drop-in ``estimate``.

Mirrors /root/reference/pkg/src/qxcorr/estimator.py: ``EstimationResult``
(27-47), ``argmax_set`` (50-57) and ``estimate`` (60-101) with the same
signature, exceptions and tie handling.  Lines 1-5 (quantise both signals,
exact integer correlation, argmax) run in the kernels; when the integer peak
ties, the tied lags come from the GPU correlogram and line 6 refines them
with the float64 correlation at those lags on the host, as the reference
does (realxcorr.py:135-150).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .batch import estimate_batch
from .errors import DegenerateQuantization
from .intxcorr import xcorr_full_device
from .errors import DegenerateInput
from .realxcorr import xcorr_real_at, xcorr_real_bf, xcorr_real_fft

__all__ = ["EstimationResult", "argmax_set", "estimate", "estimate_real", "METHODS"]

METHODS = ("ks", "bf", "gpu")


@dataclass(frozen=True)
class EstimationResult:
    lags: tuple[int, ...]
    peak_value_int: int | float
    tie_broken: bool = False
    tie_break_values: tuple[tuple[int, float], ...] = ()
    method: str = "ks"

    def __post_init__(self):
        if not self.lags:
            raise ValueError("an estimate must contain at least one lag")


def argmax_set(c) -> list[int]:
    """All lags attaining the exact maximum, ascending (estimator.py:50-57)."""
    top = np.flatnonzero(c.values == c.values.max())
    return [int(i) + c.first_lag for i in top]


def _samples(s):
    return np.asarray(s.samples, dtype=np.float64)


def estimate(x, y, qx, qy, method: str = "ks", *, refine_ties: bool = True,
             mul_backend: str = "auto", lag_lo=None, lag_hi=None) -> EstimationResult:
    """Estimate the time difference(s) between x and y from quantised data.

    ``method`` "ks" / "bf" (the reference's names; both are exact, so both
    run the GPU engine and give the reference's bit-identical answer) or
    "gpu".  ``lag_lo``/``lag_hi`` optionally restrict the lag search.
    """
    xd = D.as_device(_samples(x))
    yd = D.as_device(_samples(y))
    res = estimate_batch(xd, yd, qx, qy, lag_lo=lag_lo, lag_hi=lag_hi, x_start=int(x.start),
                         y_start=int(y.start)).numpy()[0]
    flags, status = int(res["flags"]), int(res["status"])
    if flags & N.RF_NONFINITE:
        raise ValueError("input contains NaN")
    if flags & N.RF_DEGENERATE_X:
        raise DegenerateQuantization("x quantizes to all zeros")
    if flags & N.RF_DEGENERATE_Y:
        raise DegenerateQuantization("y quantizes to all zeros")
    if status:
        raise RuntimeError(f"estimate failed with status {status}")
    if method not in METHODS:
        raise ValueError(f"unknown integer correlation method {method!r}")
    peak = int(res["value"])
    if int(res["ties"]) == 1:
        return EstimationResult((int(res["lag"]),), peak, False, (), method)
    # several lags tie: recover the whole tie set from the GPU correlogram
    values, _ = xcorr_full_device(xd, yd, qx, qy, int(x.start), int(y.start))
    first_lag = int(y.start) - (int(x.start) + len(x.samples) - 1)
    t = D.torch()
    idx = t.nonzero(values[0] == peak).flatten().cpu().numpy()
    lags = [int(i) + first_lag for i in idx]
    if lag_lo is not None:
        lags = [l for l in lags if l >= lag_lo]
    if lag_hi is not None:
        lags = [l for l in lags if l <= lag_hi]
    if len(lags) > 1 and refine_ties:
        real_values = xcorr_real_at(x, y, lags)
        best = real_values.max()
        pairs = tuple((lag, float(val)) for lag, val in zip(lags, real_values))
        survivors = tuple(lag for lag, val in zip(lags, real_values) if val == best)
        return EstimationResult(survivors, peak, True, pairs, method)
    return EstimationResult(tuple(lags), peak, False, (), method)


def estimate_real(x, y, method: str = "fft") -> EstimationResult:
    """The unquantised baseline: argmax set of the real correlation
    (estimator.py:104-117), same exceptions and result fields."""
    if not np.asarray(x.samples).any():
        raise DegenerateInput("x is all-zero")
    if not np.asarray(y.samples).any():
        raise DegenerateInput("y is all-zero")
    if method == "fft":
        c = xcorr_real_fft(x, y)
    elif method == "bf":
        c = xcorr_real_bf(x, y)
    else:
        raise ValueError(f"unknown real correlation method {method!r}")
    return EstimationResult(tuple(argmax_set(c)), float(c.values.max()), False, (), f"real_{method}")
