"""Golden vectors for the drop-in API surface beyond the hot path kernels,
from the UNMODIFIED reference (/root/reference/pkg/src/qxcorr):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_api_golden.py

random_monotone thresholds, the KS plumbing (plan_ks / pack / big_mul /
unpack_and_correct) on seeded pairs, the signal helpers (window, trim, scale,
add, crop) and estimate_real on seeded pairs.  Writes tests/golden/api.json;
tests/test_api_surface.py reads only that file.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import qxcorr as R  # noqa: E402  (reference)
from qxcorr.intxcorr import pack, plan_ks, unpack_and_correct  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "api.json")


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    g = {"reference_all": list(R.__all__)}
    g["random_monotone"] = []
    for seed in (0, 1, 7, 42, 12345, 2**31 - 1):
        for k, levels, scale in ((1, None, 1.0), (3, None, 1.0), (16, None, 2.5), (16, 7, 0.3), (5, 99, 1.0)):
            q = R.random_monotone(seed, k, levels, scale)
            g["random_monotone"].append({"args": [seed, k, levels, scale], "k": q.k,
                                         "thresholds": [float(t) for t in q.thresholds]})
    rng = np.random.default_rng(5)
    ks = []
    for _ in range(40):
        ku, kv = int(rng.integers(1, 130)), int(rng.integers(1, 17))
        u = R.IntSignal(int(rng.integers(-50, 50)), rng.integers(-ku, ku + 1, int(rng.integers(1, 400))), bound=ku)
        v = R.IntSignal(int(rng.integers(-50, 50)), rng.integers(-kv, kv + 1, int(rng.integers(1, 400))), bound=kv)
        if not (u.samples.any() and v.samples.any()):
            continue
        plan = plan_ks(u, v)
        a = pack(R.reverse(u), plan, bias=plan.bias_u)
        b = pack(v, plan, bias=plan.bias_v)
        c = unpack_and_correct(a * b, plan, u, v)
        ks.append({"u": [int(u.start), u.samples.tolist(), int(u.bound)], "v": [int(v.start), v.samples.tolist(), int(v.bound)],
                   "slot_bits": plan.slot_bits, "a": hex(a), "b": hex(b), "first_lag": c.first_lag,
                   "values": c.values.tolist(), "norms": [c.norm_x, c.norm_y]})
    g["ks"] = ks
    s = R.Signal(-3, [0.0, 0.0, 1.5, -2.0, 0.0, 3.25, 0.0])
    t = R.Signal(2, [1.0, 2.0, -1.0])
    iz = R.IntSignal(5, [0, 0, 0], bound=2)
    ii = R.IntSignal(-4, [0, 2, -1, 0, 1, 0], bound=2)
    g["signals"] = {
        "window": [s.window(-5, 12).tolist(), s.window(10, 3).tolist(), ii.window(-6, 5).tolist()],
        "trim": [[R.trim(s).start, R.trim(s).samples.tolist()], [R.trim(iz).start, R.trim(iz).samples.tolist()],
                 [R.trim(ii).start, R.trim(ii).samples.tolist(), R.trim(ii).bound]],
        "scale": [R.scale(s, -0.5).start, R.scale(s, -0.5).samples.tolist()],
        "add": [R.add(s, t).start, R.add(s, t).samples.tolist()],
        "crop": [[R.crop(s, -1, 6).start, R.crop(s, -1, 6).samples.tolist()],
                 [R.crop(ii, -10, 8).start, R.crop(ii, -10, 8).samples.tolist(), R.crop(ii, -10, 8).bound]],
    }
    er = []
    rng = np.random.default_rng(9)
    for trial in range(12):
        n = int(rng.integers(50, 3000))
        x = R.Signal(int(rng.integers(-20, 20)), rng.standard_normal(n))
        d = int(rng.integers(-n // 2, n // 2))
        y = R.Signal(x.start + d, x.samples * 1.7 + rng.normal(0, 0.3, n))
        for method in ("bf", "fft"):
            r = R.estimate_real(x, y, method)
            er.append({"x": [x.start, h(x.samples)], "seed_trial": trial, "n": n, "d": d, "method": method,
                       "lags": list(r.lags), "peak": r.peak_value_int, "result_method": r.method})
    g["estimate_real"] = er
    json.dump(g, open(OUT, "w"), indent=0)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
