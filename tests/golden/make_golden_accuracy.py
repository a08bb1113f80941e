"""Golden outcomes of the reference's accuracy experiment (harness.py:238-327)
for small configurations, from the UNMODIFIED reference package.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_accuracy.py

Writes tests/golden/accuracy.json: per configuration, the per-trial tuples
of _accuracy_trial, the rows/diagnostics of run_accuracy, and sha256 digests
of the first trials' (x, y) samples (make_trial) for the generator tests.
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from qxcorr import harness as H  # noqa: E402  (reference)
from qxcorr.quantize import from_spec  # noqa: E402
from qxcorr.signalgen import TrialSpec, gen_target, make_trial  # noqa: E402

CONFIGS = [
    dict(snr_db_list=(-20.0, -10.0, 0.0), trials=24, seed=7, quantizer_spec="sign", target_len=256,
         scene_len=1024),
    dict(snr_db_list=(-25.0, -5.0), trials=20, seed=3, quantizer_spec="uniform:1:0.6", target_len=512,
         scene_len=1536, target_kind="bandlimited", background_kind="white"),
    dict(snr_db_list=(-15.0, 5.0), trials=6, seed=11, quantizer_spec="uniform:7:0.4"),  # default shapes
]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


out = []
for kw in CONFIGS:
    cfg = H.AccuracyConfig(threads=1, **kw)
    q = from_spec(cfg.quantizer_spec)
    trials = [[list(map(bool, H._accuracy_trial(cfg, q, si, ti, None))) for ti in range(cfg.trials)]
              for si in range(len(cfg.snr_db_list))]
    rows, diag = H.run_accuracy(cfg)
    inputs = []
    for si in range(len(cfg.snr_db_list)):
        for ti in range(min(3, cfg.trials)):
            rng = np.random.default_rng(np.random.SeedSequence([cfg.seed, si, ti]))
            delay = float(rng.uniform(0.0, cfg.scene_len - cfg.target_len))
            tseed, bseed = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**63))
            bg = gen_target(bseed, cfg.scene_len, cfg.background_kind)
            spec = TrialSpec(seed=tseed, target_len=cfg.target_len, scene_len=cfg.scene_len, true_delay=delay,
                             snr_db=cfg.snr_db_list[si], quantizer_spec=cfg.quantizer_spec,
                             target_kind=cfg.target_kind)
            x, y, nu = make_trial(spec, bg)
            inputs.append({"snr_idx": si, "trial": ti, "x_start": x.start, "x": digest(x.samples),
                           "y_start": y.start, "y": digest(y.samples), "truth": nu})
    out.append({"config": kw, "trials": trials, "inputs": inputs,
                "rows": [[r.snr_db, r.quantizer, r.mode, r.trials, r.correct, r.accuracy] for r in rows],
                "diagnostics": {"tie_changed_fraction": {str(k): v for k, v in diag["tie_changed_fraction"].items()},
                                "trial_errors": diag["trial_errors"]}})
    print(kw["quantizer_spec"], [[r.mode, r.correct] for r in rows][:6], diag)
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "accuracy.json"), "w") as fh:
    json.dump(out, fh, indent=1)
