"""Full-size golden records (tests/golden/fullsize.*) for bench.py and
tools/bench_configs.py: each benchmarked estimate is checked against the
pinned oracle's exact (peak, smallest lag, ties), not the planted delay.
Test/measurement infrastructure only (the records come from
tests/golden/make_fullsize.py)."""

from __future__ import annotations

import json
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
_cache = None


def load():
    global _cache
    if _cache is None:
        meta = json.load(open(os.path.join(GOLD, "fullsize.json")))
        with np.load(os.path.join(GOLD, "fullsize.npz")) as z:
            arrays = {k: z[k] for k in z.files}
        c1 = json.load(open(os.path.join(GOLD, "golden.json")))["configs"]["c1"]
        _cache = (meta, arrays, c1)
    return _cache


def records(res) -> np.ndarray:
    """(B, 3) int64 (value, lag, ties) from a structured qx_result array."""
    return np.stack([res["value"], res["lag"], res["ties"]], axis=1).astype(np.int64)


def check_c2(bits_index: int, first: int, res) -> None:
    meta, arr, _ = load()
    want = arr["c2_rec"][bits_index, first:first + len(res)]
    if first + len(res) > arr["c2_rec"].shape[1]:
        raise AssertionError(f"no C2 goldens for pairs {first}..{first + len(res) - 1}")
    got = records(res)
    bad = np.flatnonzero((got != want).any(axis=1))
    if bad.size:
        raise AssertionError(f"C2 b-index {bits_index}: {bad.size} pairs differ from the oracle, first "
                             f"pair {first + int(bad[0])}: {got[bad[0]].tolist()} != {want[bad[0]].tolist()}")
    ss = arr["c2_sumsq"][bits_index, first:first + len(res)]
    if not (np.array_equal(res["sumsq_x"], ss[:, 0]) and np.array_equal(res["sumsq_y"], ss[:, 1])):
        raise AssertionError("C2 code sums of squares differ from the oracle")


def check_c3(bits_index: int, first: int, res) -> None:
    _, arr, _ = load()
    want = arr["c3_rec"][bits_index, first:first + len(res)].astype(np.int64)
    got = records(res)
    bad = np.flatnonzero((got != want).any(axis=1))
    if bad.size:
        raise AssertionError(f"C3 b-index {bits_index}: {bad.size} pairs differ from the oracle, first "
                             f"pair {first + int(bad[0])}: {got[bad[0]].tolist()} != {want[bad[0]].tolist()}")


def check_c1(lag: int, peak: int) -> None:
    c1 = load()[2]
    assert (lag, peak) == (c1["lags"][0], c1["peak"]), ((lag, peak), c1)


def check_c4(res) -> None:
    g = load()[0]["c4"]
    got = (int(res["value"]), int(res["lag"]), int(res["ties"]))
    assert got == (g["peak"], g["lag"], g["ties"]), (got, g)


def check_c5(b: int, summary) -> None:
    case = [c for c in load()[0]["c5"]["cases"] if c["b"] == b][0]
    assert tuple(summary) == (case["peak"], case["lag"], case["ties"]), (summary, case)
