"""CPU baselines of the reference's own two paths, timed on this host
(measurement infrastructure; bench.py's `cpu_baseline` legs and the
`--impl reference` arm).  Never imported by the product package.

* integer leg -- the reference's Integer-KS estimate (float64 quantise,
  Kronecker substitution with the GMP multiply, argmax;
  /root/reference/pkg/src/qxcorr/estimator.py:60-94, intxcorr.py:259-265) as
  the pinned C oracle (oracle/qx_oracle.c), threaded over pairs / blocks;
* float leg -- the reference's Real-FFT correlation ``ccf_fft_array``
  (realxcorr.py:99-116, timed on float32 as harness.py:148-150 does) + the
  argmax, as restated in oracle/refport.py (bit-identical to the reference on
  the same numpy), in a process pool with one worker per core (the reference
  calls are single-threaded numpy).

Every leg runs a bounded sample (about 5-15 s of CPU work) and says what it
was; rates are per unit of the config's metric.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

_G: dict = {}  # arrays shared with forked FFT workers


def cpu_info() -> dict:
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count()}


def _oracle():
    import oracle as O

    O.build()
    return O


# -------------------------------------------------------------- float leg
def _fft_pair(i):
    import refport as R

    x, y = _G["x"][i], _G["y"][i]
    c = R.ccf_fft_array(x, y)
    return int(np.argmax(c))


def _fft_block(s0):
    import refport as R

    t, st, B = _G["t"], _G["st"], _G["B"]
    c = R.ccf_fft_array(t, st[s0:s0 + B + t.size - 1])
    return int(np.argmax(c[t.size - 1:t.size - 1 + B]))


def _pool_rate(fn, tasks, procs, min_seconds):
    """Run fn over tasks (repeating) in a fork pool until min_seconds; units/s."""
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        t0 = time.perf_counter()
        n = 0
        while True:
            pool.map(fn, tasks, chunksize=1)
            n += len(tasks)
            if time.perf_counter() - t0 >= min_seconds:
                break
        dt = time.perf_counter() - t0
    return n / dt, dt, n


def fft_pairs(xs, ys, procs, min_seconds=5.0, max_pairs=None):
    """Real-FFT estimates/s over pairs (rows of xs, ys: float32)."""
    n = xs.shape[0] if max_pairs is None else min(max_pairs, xs.shape[0])
    _G["x"], _G["y"] = xs[:n], ys[:n]
    rate, dt, done = _pool_rate(_fft_pair, list(range(n)), procs, min_seconds)
    return {"value": rate, "cores": procs, "seconds": dt,
            "sample": f"{done} pair correlations ({xs.shape[1]} x {ys.shape[1]} float32) with ccf_fft_array + argmax"}


def fft_single(x, y, scale_to: int | None = None):
    """One Real-FFT correlation (1 core).  With `scale_to`, x/y are a shorter
    sample and the time is extrapolated by P log P to `scale_to` samples."""
    import refport as R

    t0 = time.perf_counter()
    c = R.ccf_fft_array(x, y)
    int(np.argmax(c))
    dt = time.perf_counter() - t0
    n = x.size
    if scale_to:
        P0 = 1 << (2 * n - 2).bit_length()
        P1 = 1 << (2 * scale_to - 2).bit_length()
        dt *= (P1 * math.log2(P1)) / (P0 * math.log2(P0))
    return dt


def fft_stream(t, st, procs, min_seconds=5.0, B=1 << 18, nblocks=None):
    """Real-FFT template search: valid-lag blocks of B lags (+ halo), a
    sample of blocks spread over the stream; stream samples/s."""
    nvalid = st.size - t.size + 1
    starts = list(range(0, nvalid - B + 1, B))
    if nblocks:
        starts = starts[::max(1, len(starts) // nblocks)][:nblocks]
    _G["t"], _G["st"], _G["B"] = t, st, B
    rate, dt, done = _pool_rate(_fft_block, starts, procs, min_seconds)
    return {"blocks_per_s": rate, "samples_per_s": rate * B, "cores": procs, "seconds": dt,
            "sample": f"{done} blocks of {B} valid lags (+{t.size - 1}-sample halo) with ccf_fft_array + argmax"}


# ------------------------------------------------------------ integer leg
def int_pairs(xs, ys, qx, qy, threads, min_seconds=5.0, t_lo=None, t_hi=None, max_pairs=None):
    """Integer-KS estimates/s over pairs (oracle, threaded)."""
    O = _oracle()
    n = xs.shape[0] if max_pairs is None else min(max_pairs, xs.shape[0])
    t0 = time.perf_counter()
    done = 0
    while True:
        O.estimate_batch_f32(xs[:n], ys[:n], qx, qy, t_lo, t_hi, threads=threads)
        done += n
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "cores": threads, "seconds": dt,
            "sample": f"{done} pair estimates ({xs.shape[1]} x {ys.shape[1]}): float64 quantise, KS + GMP mpn_mul, "
                      "argmax"}


def int_single(x, y, qx, qy):
    """One Integer-KS estimate (1 core); seconds."""
    O = _oracle()
    t0 = time.perf_counter()
    O.estimate_batch_f32(np.ascontiguousarray(x[None], np.float32), np.ascontiguousarray(y[None], np.float32), qx, qy,
                         threads=1)
    return time.perf_counter() - t0


def int_stream(t, st, qx, qy, threads, B=1 << 18, nblocks=64):
    """Integer-KS template search on a sample of valid-lag blocks; stream samples/s."""
    O = _oracle()
    nvalid = st.size - t.size + 1
    starts = list(range(0, nvalid - B + 1, B))
    starts = starts[::max(1, len(starts) // nblocks)][:nblocks]
    rows = np.stack([st[s0:s0 + B + t.size - 1] for s0 in starts])
    tt = np.broadcast_to(t, (len(starts), t.size)).copy()
    t0 = time.perf_counter()
    O.estimate_batch_f32(tt, rows, qx, qy, t.size - 1, t.size - 1 + B - 1, threads=threads)
    dt = time.perf_counter() - t0
    return {"samples_per_s": len(starts) * B / dt, "cores": threads, "seconds": dt,
            "sample": f"{len(starts)} blocks of {B} valid lags (+{t.size - 1}-sample halo) spread over the stream: "
                      "float64 quantise, KS + GMP mpn_mul, argmax"}
