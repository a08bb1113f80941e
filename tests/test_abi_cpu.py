"""C ABI checks that need no GPU: the library loads, exports every symbol
include/qxcorr_b200.h declares, and its host-side exact threshold tables
reproduce the reference quantisers on the golden vectors."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    from paper_2509_19974_b200 import _native as N

    L = N.load()
    header = open(os.path.join(ROOT, "include", "qxcorr_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(qx_[a-z_0-9]+)\s*\(", header, re.M))
    assert declared == set(N.EXPORTS), declared ^ set(N.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.qx_abi_version() == N.ABI_VERSION == int(re.search(r"#define QX_ABI_VERSION (\d+)", header).group(1))
    assert L.qx_status_string(2) == b"quantizes to all zeros"


def test_header_constants_match_the_python_mirror():
    """The ctypes mirror agrees with include/qxcorr_b200.h on the ABI version,
    the profile-kind count (qx_profile's array sizes), the path enum and the
    profile kind names the C library reports."""
    from paper_2509_19974_b200 import _native as N

    header = open(os.path.join(ROOT, "include", "qxcorr_b200.h")).read()
    kinds = int(re.search(r"#define QX_PROFILE_KINDS (\d+)", header).group(1))
    assert kinds == N.PROFILE_KINDS == len(N.QxProfile._fields_[1][1]()) and \
        ctypes.sizeof(N.QxProfile) == 8 + 16 * kinds
    paths = dict(re.findall(r"QX_PATH_([A-Z]+) = (\d)", header))
    assert {k.lower(): int(v) for k, v in paths.items()} == {k: v for k, v in N.PATHS.items() if k != "tc"}
    assert N.PATHS["tc"] == N.PATHS["direct"]
    L = N.load()
    names = [L.qx_profile_kind_name(i).decode() for i in range(kinds)]
    assert {"ntt_pass1", "ntt_pass2", "ntt_pass3", "direct", "direct_f4", "popc"} <= set(names)


def _levels(thr, vals, k):
    # level(v) = -k + #{i : v >= T[i]}
    return np.searchsorted(thr, vals, side="right") - k


def test_thresholds_reproduce_reference(golden, qrec):
    from paper_2509_19974_b200 import quantize

    meta, arr = golden
    for i, qd in enumerate(meta["quant"]):
        q = qrec(qd)
        vals, want = arr[f"q{i}_in"], arr[f"q{i}_out"]
        dt = "float32" if vals.dtype == np.float32 else "float64"
        thr = quantize.thresholds(q, dt)
        assert thr.size == 2 * q.k and np.all(np.diff(thr) >= 0)
        got = _levels(thr.astype(vals.dtype), vals, q.k)
        assert np.array_equal(got, want), (i, qd)


def test_thresholds_exhaustive_float32_sample():
    """Dense sweep over float32 bit patterns for the C2 b=4 quantiser: the
    threshold map equals the reference formula in float64 on every sample."""
    from paper_2509_19974_b200 import quantize, workloads as W

    q = W.bit_quantizer(4, W.C2_SIGMA)
    thr = quantize.thresholds(q, "float32").astype(np.float32)
    bits = np.arange(0, 1 << 32, 4099, dtype=np.uint64).astype(np.uint32)
    v = bits.view(np.float32)
    v = v[~np.isnan(v)]
    ref = np.clip(np.sign(v.astype(np.float64)) * np.floor(np.abs(v.astype(np.float64)) / q.step + 0.5),
                  -q.k, q.k).astype(np.int64)
    assert np.array_equal(_levels(thr, v, q.k), ref)


def test_quantizer_validation_errors():
    from paper_2509_19974_b200 import _native as N
    from paper_2509_19974_b200 import quantize

    import pytest

    with pytest.raises(ValueError):
        quantize.custom([0.5, 1.0])
    with pytest.raises(ValueError):
        quantize.custom([1.0, -1.0])
    with pytest.raises(ValueError):
        quantize.Quantizer(kind="uniform", k=0)
    bad = N.QxQuantizer(N.QX_Q_UNIFORM, 0, 3, -1.0, None)
    out = np.empty(6)
    assert N.load().qx_quantizer_thresholds(ctypes.byref(bad), N.QX_F32, out.ctypes.data) == N.QX_ERR_INVALID


def test_big_mul_host_backends_and_errors():
    """big_mul's plugin-slot contract (intxcorr.py:183-205, pkg/tests/test_intxcorr.py:139-149)
    for the host backends; the "cuda" backend is covered by the GPU tests."""
    import paper_2509_19974_b200 as qx

    assert qx.big_mul(257, 515) == 132355
    for backend in ("native", "karatsuba", "schoolbook", "auto"):
        assert qx.big_mul(123456789, 0, backend) == 0
        assert qx.big_mul(123456789, 1, backend) == 123456789
        assert qx.big_mul(-7, 9, backend) == -63
        assert qx.big_mul(-7, -9, backend) == 63
    with pytest.raises(ValueError):
        qx.big_mul(1, 1, "fft")
    with pytest.raises(ValueError):
        qx.big_mul(1, 1, "gmp")  # gmpy2 is not installed here, as in the reference
