"""Batched accuracy experiment on the GPU engine.

The reference's ``run_accuracy`` (/root/reference/pkg/src/qxcorr/harness.py:
283-327) scores three modes per (SNR, trial):
- "proposed": the quantised estimate with tie refinement;
- "proposed_until_line4": the quantised estimate without it;
- "ccf_wo_quant": the float FFT correlation.

The reference runs one ``estimate`` per trial. Here the caller supplies the
trials (``trial_fn(config, snr_idx, trial_idx) -> (x, y, true_lag)``, e.g.
the restated reference generator in oracle/refport.py) and the float
baseline (``baseline_fn(x, y) -> lags``); every quantised estimate of the
whole SNR grid then runs as ONE ``estimate_batch`` launch on the device.
Only the (rare) pairs whose peak ties take the exact per-pair path (GPU
correlogram + float64 refinement at the tied lags, ``estimator.estimate``).
Without a baseline_fn the "ccf_wo_quant" row is not scored (None).

Parity: tests/golden/accuracy.json holds the reference's per-trial outcomes,
rows and diagnostics for small configurations (tests/golden/make_golden_accuracy.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _device as D
from .batch import estimate_batch
from .errors import DegenerateQuantization
from .estimator import estimate
from .quantize import from_spec

__all__ = ["AccuracyConfig", "AccuracyRow", "ACCURACY_MODES", "run_accuracy", "accuracy_trials"]

ACCURACY_MODES = ("proposed", "proposed_until_line4", "ccf_wo_quant")  # harness.py:56


@dataclass(frozen=True)
class AccuracyConfig:
    """harness.py:175-202 (synthetic targets; ``threads`` has no meaning here)."""

    snr_db_list: tuple[float, ...] = (-10.0, -5.0, 0.0, 5.0, 10.0)
    trials: int = 200
    seed: int = 0
    quantizer_spec: str = "sign"
    target_len: int = 2048
    scene_len: int = 8192
    target_kind: str = "am_bursts"
    background_kind: str = "bandlimited"
    method: str = "ks"
    sample_rate: float = 16000.0

    def __post_init__(self):
        if not self.snr_db_list:
            raise ValueError("at least one SNR value is required")
        if self.trials < 1:
            raise ValueError("trial count must be positive")
        if self.target_len < 1 or self.scene_len < self.target_len:
            raise ValueError("need scene_len >= target_len >= 1")
        if self.method not in ("ks", "bf"):
            raise ValueError(f"unknown integer correlation method {self.method!r}")
        from_spec(self.quantizer_spec)


@dataclass(frozen=True)
class AccuracyRow:
    snr_db: float
    quantizer: str
    mode: str
    trials: int
    correct: int
    accuracy: float


# ---------------------------------------------------------------- driver


def accuracy_trials(config: AccuracyConfig, trial_fn, baseline_fn=None, *, device=None):
    """Per (snr_idx, trial_idx): (ok_proposed, ok_raw, ok_baseline,
    tie_changed, errored), as _accuracy_trial returns (harness.py:238-280).
    ``trial_fn(config, snr_idx, trial_idx) -> (x, y, true_lag)`` supplies the
    trials; ``baseline_fn(x, y) -> lags`` the float baseline (ok_baseline is
    None without it).  All quantised estimates of the grid run as one GPU
    batch."""
    t = D.torch()
    q = from_spec(config.quantizer_spec)
    keys, xs, ys, truths, out = [], [], [], [], {}
    for si in range(len(config.snr_db_list)):
        for ti in range(config.trials):
            try:
                x, y, nu = trial_fn(config, si, ti)
            except Exception:
                out[(si, ti)] = (False, False, False, False, True)
                continue
            keys.append((si, ti))
            xs.append(x)
            ys.append(y)
            truths.append(nu)
    if keys:
        dev = t.device("cuda", device if device is not None else t.cuda.current_device())
        xb = t.from_numpy(np.stack([s.samples for s in xs])).to(dev)
        yb = t.from_numpy(np.stack([s.samples for s in ys])).to(dev)
        res = estimate_batch(xb, yb, q, q).numpy()
    for i, key in enumerate(keys):
        x, y, nu = xs[i], ys[i], truths[i]
        r = res[i]
        try:
            if r["flags"] & 3:  # DegenerateQuantization (estimator.py:83-86)
                raise DegenerateQuantization("quantizes to all zeros")
            if int(r["ties"]) == 1:
                lags = raw = (int(r["lag"]),)
            else:  # the whole tie set and its refinement, exactly as estimate()
                e = estimate(x, y, q, q, config.method)
                lags = e.lags
                raw = tuple(lag for lag, _ in e.tie_break_values) if e.tie_broken else e.lags
            base = baseline_fn(x, y) if baseline_fn is not None else None
        except Exception:
            out[key] = (False, False, False, False, True)
            continue

        def close(ls):
            return all(abs(lag - nu) < 1.0 for lag in ls)

        out[key] = (close(lags), close(raw), close(base) if base is not None else None, tuple(lags) != tuple(raw),
                    False)
    return out


def run_accuracy(config: AccuracyConfig, trial_fn, baseline_fn=None, *,
                 device=None) -> tuple[list[AccuracyRow], dict]:
    """The reference's run_accuracy rows and diagnostics (harness.py:283-327)
    over caller-supplied trials (see accuracy_trials)."""
    trials = accuracy_trials(config, trial_fn, baseline_fn, device=device)
    rows: list[AccuracyRow] = []
    tie_changed_fraction: dict[float, float] = {}
    trial_errors = 0
    for si, snr in enumerate(config.snr_db_list):
        correct = [0, 0, 0]
        changed = 0
        for ti in range(config.trials):
            okp, okr, okb, tie_changed, errored = trials[(si, ti)]
            correct[0] += okp
            correct[1] += okr
            correct[2] += bool(okb)
            changed += tie_changed
            trial_errors += errored
        for mode, n in zip(ACCURACY_MODES, correct):
            if mode == "ccf_wo_quant" and baseline_fn is None:
                continue
            rows.append(AccuracyRow(float(snr), config.quantizer_spec, mode, config.trials, int(n),
                                    n / config.trials))
        tie_changed_fraction[float(snr)] = changed / config.trials
    return rows, {"tie_changed_fraction": tie_changed_fraction, "trial_errors": trial_errors}
