"""Seeded synthetic workloads for the five BASELINE.json configurations.

No public dataset is involved (the paper's Speech Commands / ESC-50 are not
used); these generators ARE the benchmark inputs, with the shapes, value
distributions, delays and SNRs BASELINE.json states.  They
run on the host with numpy so the oracle sees identical bits.

Lag convention (reference, signals.py:100-105): estimate(x, y) returns the
lag n maximising sum_m x[m] y[m+n]; with x = g[a:], y = g[a+d:] that is -d.

Quantisers per bit depth b: b=1 sign(); b>=2 the mid-tread
uniform(K = 2^(b-1)-1, step = 6 sigma / 2^b) -- the reference cannot express
a mid-rise quantiser (it violates q(0)=0), so this is the b-bit analogue
with parity.  sigma is the analytic standard deviation of the noisy input.
"""

from __future__ import annotations

import math

import numpy as np

from .quantize import Quantizer, sign, uniform

__all__ = ["bit_quantizer", "c1", "c2", "c3", "c4", "c5", "C2_N", "C3_N", "C3_PAIRS", "C4_N", "C4_DELAY"]

C2_N = 1 << 18
C2_PAIRS = 64
C2_MAXD = 4096
C3_N = 4096
C3_PAIRS = 65536
C3_MAXD = 512
C4_N = 1 << 24
C4_DELAY = 731_205
C5_STREAM = 1 << 28
C5_TEMPLATE = 1 << 12
C5_OFFSET = 123_456_789


def bit_quantizer(b: int, sigma: float) -> Quantizer:
    if b == 1:
        return sign()
    k = (1 << (b - 1)) - 1
    return uniform(k, 6.0 * sigma / (1 << b))


def c1(seed: int = 0):
    """Single 2^14 float64 pair, delay 137, N(0, 0.1^2) noise on each; the
    reference returns lags (-137,), peak 14839."""
    n = 1 << 14
    rng = np.random.default_rng(seed)
    s = rng.standard_normal(n + 512)
    x = s[0:n] + rng.normal(0, 0.1, n)
    y = s[137:137 + n] + rng.normal(0, 0.1, n)
    return x, y


def c2(pairs: int = C2_PAIRS, n: int = C2_N, seed: int = 2, first: int = 0):
    """Bit-depth sweep: per pair a N(0,1) float32 source, integer delay
    d ~ U{-4096..4096}, x = g[4096:4096+n], y = g[4096+d:...], white
    N(0, 0.1^2) noise on each (20 dB).  Pair p is seeded by (seed, p), so any
    sub-range [first, first+pairs) reproduces the full workload's pairs.
    Returns x (pairs, n) f32, y (pairs, n) f32, expected lags (-d)."""
    x = np.empty((pairs, n), np.float32)
    y = np.empty((pairs, n), np.float32)
    lag = np.empty(pairs, np.int64)
    for i in range(pairs):
        rng = np.random.default_rng([seed, first + i])
        g = rng.standard_normal(n + 2 * C2_MAXD, dtype=np.float32)
        d = int(rng.integers(-C2_MAXD, C2_MAXD + 1))
        x[i] = g[C2_MAXD:C2_MAXD + n] + np.float32(0.1) * rng.standard_normal(n, dtype=np.float32)
        y[i] = g[C2_MAXD + d:C2_MAXD + d + n] + np.float32(0.1) * rng.standard_normal(n, dtype=np.float32)
        lag[i] = -d
    return x, y, lag


C2_SIGMA = math.sqrt(1.0 + 0.01)


def c3(pairs: int = C3_PAIRS, n: int = C3_N, seed: int = 3, first: int = 0, block: int = 1024):
    """Many short pairs: N(0,1) float32 sources of n+1024, delay
    d ~ U{-512..512}, noise sigma 10^(-10/20) (10 dB).  Blocks of `block`
    pairs share one generator seeded by (seed, block index)."""
    assert first % block == 0
    sn = np.float32(10 ** (-10 / 20))
    x = np.empty((pairs, n), np.float32)
    y = np.empty((pairs, n), np.float32)
    lag = np.empty(pairs, np.int64)
    done = 0
    while done < pairs:
        blk = (first + done) // block
        rng = np.random.default_rng([seed, blk])
        g = rng.standard_normal((block, n + 2 * C3_MAXD), dtype=np.float32)
        d = rng.integers(-C3_MAXD, C3_MAXD + 1, size=block)
        nx = rng.standard_normal((block, n), dtype=np.float32) * sn
        ny = rng.standard_normal((block, n), dtype=np.float32) * sn
        take = min(block, pairs - done)
        idx = np.arange(n)
        x[done:done + take] = g[:take, C3_MAXD:C3_MAXD + n] + nx[:take]
        y[done:done + take] = g[np.arange(take)[:, None], C3_MAXD + d[:take, None] + idx[None]] + ny[:take]
        lag[done:done + take] = -d[:take]
        done += take
    return x, y, lag


C3_SIGMA = math.sqrt(1.0 + 0.1)


def c4(n: int = C4_N, delay: int = C4_DELAY, seed: int = 4):
    """Long pair: Laplace(0,1) float32 source (sigma_s^2 = 2), x = g[0:n],
    y = g[delay:delay+n], independent N(0, 2) noise on each (0 dB)."""
    rng = np.random.default_rng(seed)
    g = rng.laplace(0.0, 1.0, n + delay).astype(np.float32)
    x = g[:n] + rng.normal(0.0, math.sqrt(2.0), n).astype(np.float32)
    y = g[delay:delay + n] + rng.normal(0.0, math.sqrt(2.0), n).astype(np.float32)
    return x, y, -delay


C4_SIGMA = 2.0


def c5(stream: int = C5_STREAM, template: int = C5_TEMPLATE, offset: int = C5_OFFSET, seed: int = 5):
    """Template search: Laplace(0,1) float32 stream, template = clean
    stream[offset:offset+template]; the stream gets N(0, sigma_n^2) noise with
    sigma_n^2 = 2*10^(-0.5) (5 dB).  estimate(x=template, y=stream) peaks at
    lag +offset over the valid lags 0..stream-template."""
    rng = np.random.default_rng(seed)
    clean = rng.laplace(0.0, 1.0, stream).astype(np.float32)
    t = clean[offset:offset + template].copy()
    sn2 = 2.0 * 10 ** (-0.5)
    y = clean + rng.normal(0.0, math.sqrt(sn2), stream).astype(np.float32)
    return t, y, offset, sn2
