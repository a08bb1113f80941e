"""Generate golden vectors from the REFERENCE implementation itself.

Run in the development container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package (/root/reference/pkg/src/qxcorr)
and its acceptance-test helpers, evaluates them on the reference's own
known-answer inputs, on seeded sweeps and on reduced BASELINE-config inputs,
and writes tests/golden/golden.npz + golden.json.  The tests (CPU: oracle vs
golden; GPU: kernels vs golden and oracle) read only these files, so nothing
at test time touches /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import qxcorr  # noqa: E402  (reference)
from qxcorr import IntSignal, Signal  # noqa: E402
from qxcorr.estimator import argmax_set, estimate  # noqa: E402
from qxcorr.intxcorr import xcorr_int_bf, xcorr_int_ks  # noqa: E402
from qxcorr.quantize import custom, random_monotone, sign, uniform  # noqa: E402

from paper_2509_19974_b200 import workloads as W  # noqa: E402  (seeded generators only)

OUT = os.path.dirname(os.path.abspath(__file__))
arrays: dict[str, np.ndarray] = {}
meta: dict = {"reference": "qxcorr " + getattr(qxcorr, "__version__", "?"), "numpy": np.__version__}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()[:16]


def refq(q):
    """the reference's own Quantizer with q's parameters"""
    return qxcorr.Quantizer(kind=q.kind, k=int(q.k), step=float(q.step), thresholds=tuple(q.thresholds))


def qdesc(q):
    return {"kind": q.kind, "k": int(q.k), "step": float(q.step), "thresholds": [float(t) for t in q.thresholds]}


# ------------------------------------------------------------ quantisers
def quant_cases():
    cases = []
    # known-answer inputs of pkg/tests/test_quantize.py:8-30
    kats = [
        (sign(), [-3.5, -0.0, 0.0, 1e-12, 2.0]),
        (uniform(4, 1.0), [0.49, 0.5, 1.49, 1.5, -0.5, -1.5, 100.0, -100.0, 0.0]),
        (uniform(8, 0.25), [0.12, 0.13, 0.375]),
        (custom([-1.0, 0.5]), [-2.0, -1.0, 0.0, 0.4, 0.5, 3.0]),
    ]
    rng = np.random.default_rng(1234)
    s2 = W.C2_SIGMA
    quants = [sign(), uniform(1, 1.5 * s2), uniform(7, 0.375 * s2), uniform(127, 6 * s2 / 256),
              uniform(3, 0.4), uniform(16, 1.0), uniform(2, 1e-30), custom([-1.0, 0.5])]
    quants += [random_monotone(int(s), k=16) for s in rng.integers(0, 2**31, size=6)]
    for dt in (np.float32, np.float64):
        fi = np.finfo(dt)
        edge = np.array([0.0, -0.0, fi.tiny, -fi.tiny, fi.smallest_subnormal, -fi.smallest_subnormal,
                         np.inf, -np.inf, fi.max, -fi.max, 1.0, -1.0], dtype=dt)
        for qi, q in enumerate(quants):
            base = np.concatenate([rng.standard_normal(3000) * sc for sc in (1.0, 10.0, 1e-3)]).astype(dt)
            if q.kind == "uniform":  # exact half-steps and their float neighbours
                hs = (np.arange(-q.k - 2, q.k + 3) + 0.5) * q.step
                hs = hs.astype(dt)
                base = np.concatenate([base, hs, np.nextafter(hs, dt(np.inf)), np.nextafter(hs, dt(-np.inf))])
            if q.kind == "custom":
                t = np.asarray(q.thresholds).astype(dt)
                base = np.concatenate([base, t, np.nextafter(t, dt(np.inf)), np.nextafter(t, dt(-np.inf))])
            vals = np.concatenate([base, edge]).astype(dt)
            cases.append((q, vals))
    for q, vals in kats:
        cases.append((q, np.asarray(vals, dtype=np.float64)))
    out = []
    for i, (q, vals) in enumerate(cases):
        codes = q(vals.astype(np.float64))  # the reference upcasts (signals.py:46)
        arrays[f"q{i}_in"] = vals
        arrays[f"q{i}_out"] = codes.astype(np.int64)
        out.append(qdesc(q))
    meta["quant"] = out


# ----------------------------------------------------------- correlation
def random_int_signal(rng, max_len=64, max_k=16):
    # generator of pkg/tests/test_intxcorr.py:41-45
    n = int(rng.integers(1, max_len + 1))
    k = int(rng.integers(1, max_k + 1))
    start = int(rng.integers(-100, 100))
    return IntSignal(start, rng.integers(-k, k + 1, size=n), bound=k)


def xcorr_cases():
    pairs = [
        (IntSignal(0, [1, 2], bound=2), IntSignal(0, [1, 2], bound=2)),
        (IntSignal(0, [1], bound=1), IntSignal(2, [1], bound=1)),
        (IntSignal(0, [1, -1], bound=1), IntSignal(0, [1, -1], bound=1)),
        (IntSignal(0, [1, 1, 1], bound=1), IntSignal(0, [1, 1, 1], bound=1)),
        (IntSignal(0, [16], bound=16), IntSignal(0, [16], bound=16)),
        (IntSignal(0, [-5] * 9, bound=5), IntSignal(-3, [-5] * 4, bound=5)),
        (IntSignal(0, [3, -3] * 8, bound=3), IntSignal(0, [-3, 3] * 5, bound=3)),
        (IntSignal(2, [1, -1, 1, -1, 1], bound=1), IntSignal(-2, [-1] * 7, bound=1)),
        (IntSignal(0, [16] * 4, bound=16), IntSignal(0, [-16] * 4, bound=16)),
        (IntSignal(0, [1], bound=1), IntSignal(5, [-1], bound=1)),
        (IntSignal(0, [3, 4], bound=4), IntSignal(0, [3, 4], bound=4)),
    ]
    rng = np.random.default_rng(101)
    pairs += [(random_int_signal(rng), random_int_signal(rng)) for _ in range(150)]
    rng = np.random.default_rng(202)
    pairs += [(random_int_signal(rng, max_len=96), random_int_signal(rng, max_len=96)) for _ in range(200)]
    import test_acceptance as TA  # reference acceptance helpers (imported, not copied)

    pairs += TA._edge_pairs()
    out = []
    for i, (u, v) in enumerate(pairs):
        c = xcorr_int_bf(u, v)
        if u.samples.any() and v.samples.any():
            assert xcorr_int_ks(u, v) == c
        arrays[f"x{i}_u"] = u.samples
        arrays[f"x{i}_v"] = v.samples
        arrays[f"x{i}_c"] = c.values.astype(np.int64)
        out.append({"u_start": u.start, "v_start": v.start, "ku": int(u.bound), "kv": int(v.bound),
                    "first_lag": int(c.first_lag), "norm_x": c.norm_x, "norm_y": c.norm_y,
                    "argmax": argmax_set(c)})
    meta["xcorr"] = out
    # acceptance criterion 2 (pkg/tests/test_acceptance.py:103-151): record
    # digests of the brute-force correlograms of its 1000 seeded pairs
    ok, blob, failures = TA._run_ks_bf_equivalence(TA.SEED_PAIRS)
    assert ok and failures == 0
    meta["acceptance_c2"] = {"seed": TA.SEED_PAIRS, "records": json.loads(blob)}


# -------------------------------------------------------------- estimate
def estimate_cases():
    out = []

    def add(x, y, qx, qy, **kw):
        i = len(out)
        try:
            r = estimate(x, y, qx, qy, **kw)
            res = {"lags": list(r.lags), "peak": int(r.peak_value_int), "tie_broken": r.tie_broken,
                   "tie_break_values": [[int(a), float(b)] for a, b in r.tie_break_values], "method": r.method}
        except Exception as exc:  # noqa: BLE001 -- recorded as the expected exception
            res = {"raises": type(exc).__name__, "message": str(exc)}
        arrays[f"e{i}_x"] = np.asarray(x.samples)
        arrays[f"e{i}_y"] = np.asarray(y.samples)
        out.append({"x_start": x.start, "y_start": y.start, "qx": qdesc(qx), "qy": qdesc(qy), "kw": kw,
                    "result": res})

    # pkg/tests/test_estimator.py KAT inputs
    add(Signal(0, [1.0]), Signal(0, [1.0, 0.5]), sign(), sign())
    add(Signal(0, [1.0]), Signal(0, [1.0, 0.5]), sign(), sign(), refine_ties=False)
    rng = np.random.default_rng(3)
    x = Signal(0, rng.uniform(0.5, 1.0, size=50))
    y = Signal(0, rng.uniform(0.5, 1.0, size=80))
    add(x, y, sign(), sign())
    rng = np.random.default_rng(0)
    x = Signal(0, rng.standard_normal(256))
    for d in (-37, 0, 64):
        add(x, Signal(x.start + d, x.samples * 2.5), sign(), sign())
    rng = np.random.default_rng(5)
    for _ in range(20):
        x = Signal(0, rng.standard_normal(100))
        y = Signal(int(rng.integers(-30, 30)), rng.standard_normal(130))
        add(x, y, uniform(4, 0.5), uniform(4, 0.5))
        add(x, y, uniform(4, 0.5), uniform(4, 0.5), method="bf")
    add(Signal(0, [0.01, -0.02, 0.03]), Signal(0, [1.0, -1.0, 1.0]), uniform(4, 1.0), uniform(4, 1.0))
    add(Signal(0, [1.0, -1.0, 1.0]), Signal(0, [0.01, -0.02, 0.03]), uniform(4, 1.0), uniform(4, 1.0))
    add(Signal(0, [1.0, -1.0]), Signal(0, [1.0, -1.0]), sign(), sign(), method="phat")
    # random monotone quantizers, shifted/scaled pairs (test_estimator.py:35-53 style)
    rng = np.random.default_rng(11)
    for _ in range(40):
        n = int(rng.integers(4, 257))
        yv = Signal(int(rng.integers(-20, 20)), rng.standard_normal(n))
        a = float(rng.uniform(0.05, 10.0))
        v = int(rng.integers(-128, 129))
        xv = Signal(yv.start - v, yv.samples * a)
        qx = random_monotone(int(rng.integers(2**31)), k=16, scale=a)
        qy = random_monotone(int(rng.integers(2**31)), k=16, scale=1.0)
        add(xv, yv, qx, qy)
    meta["estimate"] = out


# ----------------------------------------------------- BASELINE configs
def config_cases():
    cfg = {}
    t0 = time.time()
    x, y = W.c1(0)
    r = estimate(Signal(0, x), Signal(0, y), sign(), sign())
    cfg["c1"] = {"lags": list(r.lags), "peak": int(r.peak_value_int), "tie_broken": r.tie_broken}
    # C2: first 3 pairs at every bit depth, full correlograms (reference KS)
    xs, ys, lag = W.c2(pairs=3)
    c2 = []
    for b in (1, 2, 4, 8):
        q = refq(W.bit_quantizer(b, W.C2_SIGMA))
        for p in range(3):
            from qxcorr.quantize import apply

            u = apply(q, Signal(0, xs[p]))
            v = apply(q, Signal(0, ys[p]))
            c = xcorr_int_ks(u, v)
            top = argmax_set(c)
            c2.append({"b": b, "pair": p, "peak": int(c.values.max()), "lags": top, "sha": sha(c.values),
                       "expected": int(lag[p]), "sumsq_u": int(np.sum(u.samples ** 2)),
                       "sumsq_v": int(np.sum(v.samples ** 2))})
    cfg["c2"] = c2
    # C3: first 256 pairs, window -512..512 of the reference correlogram
    xs, ys, lag = W.c3(pairs=256)
    c3 = []
    for b in (2, 4):
        q = refq(W.bit_quantizer(b, W.C3_SIGMA))
        for p in range(256):
            u = qxcorr.apply(q, Signal(0, xs[p]))
            v = qxcorr.apply(q, Signal(0, ys[p]))
            c = xcorr_int_bf(u, v)
            lo = -512 - c.first_lag
            win = c.values[lo:lo + 1025]
            m = int(win.max())
            c3.append({"b": b, "pair": p, "peak": m, "lags": [int(i) - 512 for i in np.flatnonzero(win == m)],
                       "sha": sha(win), "expected": int(lag[p])})
    cfg["c3"] = c3
    # C4-shaped at reduced length (the full 2^24 KS takes ~1 h in the reference)
    x4, y4, l4 = W.c4(n=1 << 17, delay=73_120)
    q4 = refq(W.bit_quantizer(4, W.C4_SIGMA))
    c = xcorr_int_ks(qxcorr.apply(q4, Signal(0, x4)), qxcorr.apply(q4, Signal(0, y4)))
    cfg["c4_small"] = {"n": 1 << 17, "delay": 73_120, "peak": int(c.values.max()), "lags": argmax_set(c),
                       "sha": sha(c.values), "expected": int(l4)}
    # C5-shaped at reduced length: valid lags of template vs stream
    t5, s5, off, sn2 = W.c5(stream=1 << 16, template=1 << 12, offset=12_345)
    c5 = []
    for b in (1, 2):
        if b == 1:
            qx = qy = sign()
        else:
            qx = uniform(1, 1.5 * np.sqrt(2.0))
            qy = uniform(1, 1.5 * np.sqrt(2.0 + sn2))
        c = xcorr_int_bf(qxcorr.apply(qx, Signal(0, t5)), qxcorr.apply(qy, Signal(0, s5)))
        lo = 0 - c.first_lag
        valid = c.values[lo:lo + (1 << 16) - (1 << 12) + 1]
        m = int(valid.max())
        c5.append({"b": b, "peak": m, "lags": [int(i) for i in np.flatnonzero(valid == m)], "sha": sha(valid),
                   "qx": qdesc(qx), "qy": qdesc(qy)})
    cfg["c5_small"] = {"stream": 1 << 16, "template": 1 << 12, "offset": 12_345, "cases": c5}
    cfg["seconds"] = time.time() - t0
    meta["configs"] = cfg


if __name__ == "__main__":
    quant_cases()
    xcorr_cases()
    estimate_cases()
    config_cases()
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays;", meta["configs"]["c1"])
