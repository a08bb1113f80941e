"""Batched accuracy experiment against the reference's
own outcomes (tests/golden/accuracy.json, tests/golden/make_golden_accuracy.py)."""
import hashlib
import json
import os

import numpy as np
import pytest

import refport as R  # oracle/refport.py: the reference's generator and float FFT, restated (test infrastructure)

from paper_2509_19974_b200 import accuracy as A

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "accuracy.json")))


def _cfg(kw):
    kw = dict(kw)
    kw["snr_db_list"] = tuple(kw["snr_db_list"])
    return A.AccuracyConfig(**kw)


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", range(len(GOLD)))
def test_trial_generation_matches_reference(case):
    """make_trial / gen_target / seeding restated: bit-identical samples."""
    g = GOLD[case]
    cfg = _cfg(g["config"])
    for rec in g["inputs"]:
        x, y, nu = R.accuracy_trial_inputs(cfg, rec["snr_idx"], rec["trial"])
        assert (x.start, _digest(x.samples)) == (rec["x_start"], rec["x"])
        assert (y.start, _digest(y.samples)) == (rec["y_start"], rec["y"])
        assert nu == rec["truth"]


@pytest.mark.parametrize("case", range(len(GOLD)))
def test_float_baseline_matches_reference(case):
    """The ccf_wo_quant mode (radix-2 FFT correlation, realxcorr.py) per trial."""
    g = GOLD[case]
    cfg = _cfg(g["config"])
    for si in range(len(cfg.snr_db_list)):
        for ti in range(cfg.trials):
            x, y, nu = R.accuracy_trial_inputs(cfg, si, ti)
            ok = all(abs(lag - nu) < 1.0 for lag in R.baseline_lags(x, y))
            assert ok == g["trials"][si][ti][2], (si, ti)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(GOLD)))
def test_batched_accuracy_matches_reference(case):
    """All trials' integer estimates in one GPU batch (+ exact tie refinement):
    per-trial outcomes, rows and diagnostics equal run_accuracy's."""
    g = GOLD[case]
    cfg = _cfg(g["config"])
    trials = A.accuracy_trials(cfg, R.accuracy_trial_inputs, R.baseline_lags)
    for si in range(len(cfg.snr_db_list)):
        for ti in range(cfg.trials):
            assert list(trials[(si, ti)]) == g["trials"][si][ti], (si, ti)
    rows, diag = A.run_accuracy(cfg, R.accuracy_trial_inputs, R.baseline_lags)
    assert [[r.snr_db, r.quantizer, r.mode, r.trials, r.correct, r.accuracy] for r in rows] == g["rows"]
    assert {str(k): v for k, v in diag["tie_changed_fraction"].items()} == g["diagnostics"]["tie_changed_fraction"]
    assert diag["trial_errors"] == g["diagnostics"]["trial_errors"]
