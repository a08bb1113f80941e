"""The exact-arithmetic model of the NTT kernels' index math (tools/
ntt_model.py) reproduces np.correlate for every transform size class."""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tools"))
import ntt_model as M  # noqa: E402


@pytest.mark.parametrize("lp", [10, 11, 12, 13])
def test_fourstep_matches_correlate(lp):
    rng = np.random.default_rng(lp)
    p = 1012924417
    for _ in range(2):
        nu = int(rng.integers(1, (1 << lp) - 1))
        nv = int(rng.integers(1, (1 << lp) - nu + 2))
        u = rng.integers(-7, 8, nu).tolist()
        v = rng.integers(-7, 8, nv).tolist()
        assert M.correlate_fourstep(u, v, p, lp) == np.correlate(v, u, "full").tolist()


def test_schedule_sums():
    for l in range(5, 14):
        s = M.schedule(l)
        assert sum(s) == l and max(s) <= 4
