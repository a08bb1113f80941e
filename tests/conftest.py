import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the kernels")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle():
    import oracle as O  # oracle/oracle.py (test infrastructure)

    O.build()
    return O


class Q:
    """Quantizer-like record built from golden metadata."""

    def __init__(self, d):
        self.kind = d["kind"]
        self.k = d["k"]
        self.step = d["step"]
        self.thresholds = tuple(d["thresholds"])


@pytest.fixture(scope="session")
def qrec():
    return Q
