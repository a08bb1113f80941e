"""Pin the CPU oracle (oracle/qx_oracle.c) to vectors produced by the
reference itself (tests/golden/, made by tests/golden/make_golden.py)."""

import hashlib
import math

import numpy as np


def test_quantizer_matches_reference(golden, oracle, qrec):
    meta, arr = golden
    for i, qd in enumerate(meta["quant"]):
        vals, want = arr[f"q{i}_in"], arr[f"q{i}_out"]
        got = oracle.quantize(qrec(qd), vals)
        assert np.array_equal(got, want), (i, qd)


def test_xcorr_bf_and_ks_match_reference(golden, oracle):
    meta, arr = golden
    for i, d in enumerate(meta["xcorr"]):
        u, v, c = arr[f"x{i}_u"], arr[f"x{i}_v"], arr[f"x{i}_c"]
        assert np.array_equal(oracle.xcorr_bf(u, v), c), i
        if u.any() and v.any():
            assert np.array_equal(oracle.xcorr_ks(u, v, max(d["ku"], 1), max(d["kv"], 1)), c), i
        assert math.sqrt(oracle.sumsq(u)) == d["norm_x"]
        m, f, n = oracle.argmax(c)
        lags = [d["first_lag"] + j for j in np.flatnonzero(c == m)]
        assert lags == d["argmax"] and d["first_lag"] + f == lags[0] and n == len(lags)


def _acceptance_pair(seed, case, fixed):
    # restatement of the seeded draw in pkg/tests/test_acceptance.py:103-130
    if case < len(fixed):
        return fixed[case]
    rng = np.random.default_rng(np.random.SeedSequence([seed, case]))
    k_u = int(rng.integers(1, 17))
    k_v = int(rng.integers(1, 17))
    su = int(rng.integers(-99, 100))
    u = rng.integers(-k_u, k_u + 1, size=int(rng.integers(1, 1025)))
    sv = int(rng.integers(-99, 100))
    v = rng.integers(-k_v, k_v + 1, size=int(rng.integers(1, 1025)))
    return (su, u, k_u), (sv, v, k_v)


def _edge_pairs():
    # restatement of pkg/tests/test_acceptance.py:85-100 as (start, samples, k)
    pairs = []
    for n in (1, 2, 3, 17, 256, 1024):
        for k in (1, 16):
            neg = (0, np.array([-k] * n), k)
            pairs.append((neg, neg))
            alt_a = (-5, np.array([k if i % 2 else -k for i in range(n)]), k)
            alt_b = (9, np.array([-k if i % 2 else k for i in range(max(1, n // 2))]), k)
            pairs.append((alt_a, alt_b))
    for n in (1, 4, 333, 1024):
        rng = np.random.default_rng(n)
        ones = (0, 2 * rng.integers(0, 2, size=n) - 1, 1)
        pairs.append((ones, (3, np.array([1]), 1)))
        pairs.append((ones, ones))
    return pairs


def test_acceptance_criterion2_digests(golden, oracle):
    """All 1000 pairs of the reference's acceptance criterion 2: the oracle's
    brute-force and KS correlograms hash to the reference's digests."""
    meta, _ = golden
    acc = meta["acceptance_c2"]
    fixed = _edge_pairs()
    checked = 0
    for rec in acc["records"]:
        if "skipped" in rec:
            continue
        (su, u, ku), (sv, v, kv) = _acceptance_pair(acc["seed"], rec["case"], fixed)
        c = oracle.xcorr_bf(u, v)
        assert hashlib.sha256(c.tobytes()).hexdigest()[:16] == rec["sha"], rec
        assert sv - (su + len(u) - 1) == rec["first_lag"]
        assert np.array_equal(oracle.xcorr_ks(u, v, ku, kv), c)
        checked += 1
    assert checked > 900


def test_c1_golden(golden, oracle):
    from paper_2509_19974_b200 import workloads as W

    meta, _ = golden
    x, y = W.c1(0)

    class S:
        kind, k, step, thresholds = "sign", 1, 1.0, ()

    u, v = oracle.quantize(S, x), oracle.quantize(S, y)
    c = oracle.xcorr_ks(u, v, 1, 1)
    m, f, n = oracle.argmax(c)
    first_lag = 0 - (len(u) - 1)
    assert (m, first_lag + f, n) == (meta["configs"]["c1"]["peak"], meta["configs"]["c1"]["lags"][0], 1)


def test_slot_bits_match_plan_ks(oracle):
    # plan_ks KATs (pkg/tests/test_intxcorr.py:82-90) and SURVEY 8(a) a8 widths
    assert oracle.slot_bits(2, 4, 4) == 8
    assert oracle.slot_bits(4, 1, 1) == 5
    assert oracle.slot_bits(1, 1, 1) == 3
    assert oracle.slot_bits(1 << 18, 127, 127) == 34
    assert oracle.slot_bits(1 << 24, 7, 7) == 32
