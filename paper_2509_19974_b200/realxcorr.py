"""Real-valued correlation at selected lags: the tie refinement of Alg. 1
line 6.  Restates /root/reference/pkg/src/qxcorr/realxcorr.py:135-150 on the
host with the same float64 ``np.dot`` so refined values are bit-identical;
it touches O(#ties * N) samples and runs only when the integer peak ties."""

from __future__ import annotations

import numpy as np

__all__ = ["xcorr_real_at"]


def xcorr_real_at(x, y, lags) -> np.ndarray:
    out = np.empty(len(lags), dtype=np.float64)
    xs = np.asarray(x.samples, dtype=np.float64)
    ys = np.asarray(y.samples, dtype=np.float64)
    for pos, lag in enumerate(lags):
        d = x.start + int(lag) - y.start
        i_lo = max(0, -d)
        i_hi = min(len(xs), len(ys) - d)
        if i_lo >= i_hi:
            raise ValueError(f"lag {lag} has no overlap between the signals")
        out[pos] = float(np.dot(xs[i_lo:i_hi], ys[i_lo + d : i_hi + d]))
    return out
