"""CPU restatement of the reference's signal generation and float FFT
correlation (test / baseline infrastructure; NOT product code).

TEST INFRASTRUCTURE ONLY -- imported by tests/ (the accuracy experiment's
trial generator and its "ccf_wo_quant" float baseline, checked per trial
against the reference's own outcomes in tests/golden/accuracy.json) and by
bench.py's CPU-baseline legs (the reference's float-FFT cross-correlation
timed beside the GPU, north_star / BASELINE.md section 3).  The product
package never imports it.

Restated from /root/reference/pkg/src/qxcorr:
- ``gen_target`` / ``_bandlimited`` / ``_unit_rms``  (signalgen.py:52-97)
- ``_sinc_shift`` (100-116), ``_mix_at_snr`` (119-127), ``make_trial`` (130-147)
- ``accuracy_trial_inputs``: the per-trial seeding of _accuracy_trial
  (harness.py:238-257)
- ``_fft`` (realxcorr.py:46-88) and ``ccf_fft_array`` (realxcorr.py:99-116),
  ``baseline_lags`` = estimate_real(x, y, "fft").lags (estimator.py:104-117)
Bit-identical to the reference on the same numpy (tests/test_accuracy.py).
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_19974_b200.errors import DegenerateInput  # noqa: E402
from paper_2509_19974_b200.estimator import argmax_set  # noqa: E402
from paper_2509_19974_b200.signals import Correlogram, Signal  # noqa: E402

# ------------------------------------------------------- trial generation


def _bandlimited(rng: np.random.Generator, length: int, band) -> np.ndarray:
    freqs = np.fft.rfftfreq(length)
    mask = (freqs >= band[0]) & (freqs <= band[1])
    if not mask.any():
        raise ValueError(f"length {length} has no DFT bins inside band {band}")
    spectrum = np.fft.rfft(rng.standard_normal(length)) * mask
    return np.fft.irfft(spectrum, length)


def _unit_rms(samples: np.ndarray) -> np.ndarray:
    return samples / math.sqrt(np.mean(samples * samples))


def gen_target(seed: int, length: int, kind: str = "white", *, band=(0.02, 0.2)) -> Signal:
    """Deterministic unit-RMS test signal anchored at 0 (signalgen.py:65-97)."""
    if length < 1:
        raise ValueError("length must be >= 1")
    rng = np.random.default_rng(seed)
    if kind == "white":
        samples = rng.standard_normal(length)
    elif kind == "bandlimited":
        samples = _bandlimited(rng, length, band)
    elif kind == "am_bursts":
        carrier = _bandlimited(rng, length, band)
        envelope = np.zeros(length)
        for _ in range(max(1, length // 512)):
            width = max(3, int(round(rng.uniform(length / 16, length / 4))))
            center = rng.uniform(0, length)
            amp = rng.uniform(0.3, 1.0)
            lo = int(round(center - width / 2))
            bump = amp * np.hanning(width)
            a, b = max(0, lo), min(length, lo + width)
            if a < b:
                envelope[a:b] += bump[a - lo:b - lo]
        samples = carrier * envelope
        if not samples.any():
            samples = carrier
    else:
        raise ValueError(f"unknown target kind {kind!r}")
    return Signal(0, _unit_rms(samples))


def _window(s: Signal, start: int, length: int) -> np.ndarray:
    out = np.zeros(length, dtype=s.samples.dtype)
    lo, hi = max(start, s.start), min(start + length, s.start + len(s.samples))
    if lo < hi:
        out[lo - start:hi - start] = s.samples[lo - s.start:hi - s.start]
    return out


def _sinc_shift(s: Signal, d: float, half_width: int = 64) -> Signal:
    """result[n] ~= s[n + d], Hann-windowed sinc (signalgen.py:100-116)."""
    whole = math.floor(d)
    frac = float(d) - whole
    if frac == 0.0:
        return Signal(s.start - int(whole), s.samples)
    w = half_width
    u = frac - np.arange(-w + 1, w + 1)
    taps = np.sinc(u) * (0.5 + 0.5 * np.cos(np.pi * u / w))
    return Signal(s.start - whole - w, np.convolve(s.samples, taps[::-1]))


def _l2(s: Signal) -> float:
    return math.sqrt(math.fsum(v * v for v in s.samples.tolist()))


def _mix_at_snr(target: Signal, background: Signal, snr_db: float) -> Signal:
    """target + g*background at the requested energy ratio (signalgen.py:119-127)."""
    e_t, e_b = _l2(target) ** 2, _l2(background) ** 2
    if e_t == 0.0 or e_b == 0.0:
        raise DegenerateInput("cannot set an SNR against an all-zero signal")
    g = math.sqrt((e_t / len(target.samples)) / (e_b / len(background.samples))) * 10.0 ** (-snr_db / 20.0)
    lo = min(target.start, background.start)
    hi = max(target.start + len(target.samples), background.start + len(background.samples)) - 1
    out = np.zeros(hi - lo + 1, dtype=np.float64)
    out[target.start - lo:target.start - lo + len(target.samples)] += target.samples
    out[background.start - lo:background.start - lo + len(background.samples)] += background.samples * g
    return Signal(lo, out)


def make_trial(target: Signal, background: Signal, true_delay: float, snr_db: float, scene_len: int):
    """(x = scene, y = target, true lag) (signalgen.py:130-147)."""
    if len(background.samples) < scene_len:
        raise DegenerateInput("background is shorter than the scene")
    placed = _sinc_shift(target, -true_delay)
    scene_bg = Signal(0, _window(background, 0, scene_len))
    mixed = _mix_at_snr(placed, scene_bg, snr_db)
    return Signal(0, _window(mixed, 0, scene_len)), target, -float(true_delay)


def accuracy_trial_inputs(config, snr_idx: int, trial_idx: int):
    """The seeded draws of _accuracy_trial (harness.py:238-257)."""
    rng = np.random.default_rng(np.random.SeedSequence([config.seed, snr_idx, trial_idx]))
    delay = float(rng.uniform(0.0, config.scene_len - config.target_len))
    target_seed = int(rng.integers(0, 2**63))
    background_seed = int(rng.integers(0, 2**63))
    background = gen_target(background_seed, config.scene_len, config.background_kind)
    target = gen_target(target_seed, config.target_len, config.target_kind)
    return make_trial(target, background, delay, config.snr_db_list[snr_idx], config.scene_len)


# ------------------------------------------------------------ float CCF


def _bit_reverse_indices(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros(n, dtype=np.int64)
    for _ in range(bits):
        rev = (rev << 1) | (idx & 1)
        idx >>= 1
    return rev


def _fft(values: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Iterative radix-2 DFT (realxcorr.py:46-88)."""
    a = np.asarray(values)
    n = a.shape[0]
    cdtype = np.complex64 if a.dtype in (np.float32, np.complex64) else np.complex128
    out = a.astype(cdtype)[_bit_reverse_indices(n)]
    m = 2
    while m <= n:
        half = m // 2
        ang = (2j if inverse else -2j) * np.pi / m
        twiddle = np.exp(ang * np.arange(half)).astype(cdtype)
        blocks = out.reshape(-1, m)
        lo = blocks[:, :half].copy()
        hi = blocks[:, half:] * twiddle
        blocks[:, :half] = lo + hi
        blocks[:, half:] = lo - hi
        m *= 2
    if inverse:
        out /= n
    return out


def ccf_fft_array(xs: np.ndarray, ys: np.ndarray) -> np.ndarray:
    """Full-overlap float CCF via zero-padded spectra (realxcorr.py:99-116)."""
    n_x, n_y = len(xs), len(ys)
    count = n_x + n_y - 1
    padded = 1 << (count - 1).bit_length()
    dtype = xs.dtype if xs.dtype == np.float32 else np.float64
    x_pad = np.zeros(padded, dtype=dtype)
    y_pad = np.zeros(padded, dtype=dtype)
    x_pad[:n_x] = xs
    y_pad[:n_y] = ys
    circ = _fft(np.conj(_fft(x_pad)) * _fft(y_pad), inverse=True).real
    return circ[(np.arange(count) - (n_x - 1)) % padded].astype(dtype)


def baseline_lags(x: Signal, y: Signal) -> list[int]:
    """estimate_real(x, y, "fft").lags (estimator.py:104-117)."""
    if not x.samples.any() or not y.samples.any():
        raise DegenerateInput("all-zero signal")
    first = y.start - (x.start + len(x.samples) - 1)
    return argmax_set(Correlogram(first, ccf_fft_array(x.samples, y.samples)))
