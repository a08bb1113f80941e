"""Full-size bit-exact parity for BASELINE configs 2-5 (GPU).

Every record and digest in tests/golden/fullsize.{npz,json} was produced by
the pinned CPU oracle (tests/golden/make_fullsize.py: float64 quantise,
Kronecker substitution with GMP, argmax; pinned to the reference's own
vectors).  Here the kernels reproduce all of them at BASELINE's full sizes:

* C2: 512 pairs x 4 bit depths of (peak, smallest lag, ties) and both code
  sums of squares (the norms), and the sha256 digest of every one of the 256
  full correlograms of bench.py's rank-0 batch (2^19 - 1 lags each);
* C3: all 65,536 pairs x 2 bit depths of (peak, smallest lag, ties) on the
  tensor-core window path, and a digest over every pair's 1025-lag window on
  the NTT path;
* C4: the sha256 of the full 2^25 - 1 lag correlogram and its summary;
* C5: the 2^28-sample template search summary at b = 1, 2 (tensor-core
  path), 4096 per-65,536-lag block records (NTT path) and the sha256 of all
  268,431,361 valid-lag values.

The digest format is the reference's acceptance pattern
(pkg/tests/test_acceptance.py:131-134): sha256 over int64 LE values.
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def full():
    meta = json.load(open(os.path.join(GOLD, "fullsize.json")))
    with np.load(os.path.join(GOLD, "fullsize.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    return meta, arrays


@pytest.fixture(scope="module")
def P():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2509_19974_b200 as P

    return P


def sha16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()[:16]


def recs(res):
    return np.stack([res["value"], res["lag"], res["ties"]], axis=1)


def test_c2_full_size(P, full):
    import torch

    from paper_2509_19974_b200 import workloads as W
    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    meta, arr = full
    want_rec, want_ss = arr["c2_rec"], arr["c2_sumsq"]
    npairs = want_rec.shape[1]
    qs = [W.bit_quantizer(b, W.C2_SIGMA) for b in (1, 2, 4, 8)]
    for first in range(0, npairs, 64):
        xs, ys, _ = W.c2(pairs=64, first=first)
        xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
        sw = P.estimate_sweep(xd, yd, [(q, q) for q in qs])
        for bi in range(4):
            r = sw[bi].numpy()
            assert (r["status"] == 0).all()
            np.testing.assert_array_equal(recs(r), want_rec[bi, first:first + 64], err_msg=f"b{bi} @{first}")
            np.testing.assert_array_equal(np.stack([r["sumsq_x"], r["sumsq_y"]], 1), want_ss[bi, first:first + 64])
        if first == 0:  # every full correlogram of the rank-0 batch, digest-exact
            for bi, q in enumerate(qs):
                vals, _ = xcorr_full_device(xd, yd, q, q)
                host = vals.cpu().numpy()
                got = [sha16(host[p]) for p in range(64)]
                assert got == meta["c2"]["sha16"][bi][:64], bi
                del vals


def test_c3_full_size(P, full):
    import torch

    from paper_2509_19974_b200 import workloads as W
    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    meta, arr = full
    want = arr["c3_rec"]
    n, half = W.C3_N, W.C3_MAXD
    xs, ys, _ = W.c3()
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    del xs, ys
    t_lo = n - 1 - half
    for bi, b in enumerate((2, 4)):
        q = W.bit_quantizer(b, W.C3_SIGMA)
        # tensor-core window path, all 65,536 pairs in one call
        r = P.estimate_batch(xd, yd, q, q, lag_lo=-half, lag_hi=half).numpy()
        assert (r["status"] == 0).all()
        np.testing.assert_array_equal(recs(r), want[bi].astype(np.int64), err_msg=f"b={b}")
        # every window value, via the full NTT correlograms (4096 pairs per call)
        h = hashlib.sha256()
        for c0 in range(0, W.C3_PAIRS, 4096):
            vals, _ = xcorr_full_device(xd[c0:c0 + 4096], yd[c0:c0 + 4096], q, q)
            h.update(vals[:, t_lo:t_lo + 2 * half + 1].contiguous().cpu().numpy().tobytes())
            del vals
        assert h.hexdigest() == meta["c3"]["window_sha256"][bi], b


def test_c4_full_size_digest(P, full):
    import torch

    from paper_2509_19974_b200 import workloads as W
    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    g = full[0]["c4"]
    x, y, _ = W.c4()
    q = W.bit_quantizer(4, W.C4_SIGMA)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    r = P.estimate_batch(xd, yd, q, q).numpy()[0]
    assert (int(r["value"]), int(r["lag"]), int(r["ties"])) == (g["peak"], g["lag"], g["ties"])
    assert [int(r["sumsq_x"]), int(r["sumsq_y"])] == g["sumsq"]
    vals, _ = xcorr_full_device(xd, yd, q, q)
    assert hashlib.sha256(vals[0].cpu().numpy().tobytes()).hexdigest() == g["sha256"]


def _c5_q(P, b, sn2):
    if b == 1:
        return P.sign(), P.sign()
    return P.uniform(1, 1.5 * math.sqrt(2.0)), P.uniform(1, 1.5 * math.sqrt(2.0 + sn2))


def test_c5_full_size(P, full):
    import torch

    from paper_2509_19974_b200 import workloads as W
    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    meta, arr = full
    g = meta["c5"]
    tpl, st, off, sn2 = W.c5()
    assert (len(st), len(tpl), off) == (g["stream"], g["template"], g["offset"])
    td, sd = torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda()
    del st
    nt, ns = td.shape[0], sd.shape[0]
    nvalid = ns - nt + 1
    B = g["block"]
    for case in g["cases"]:
        b = case["b"]
        qa, qb = _c5_q(P, b, sn2)
        # 1) the product call (tensor-core template search, device merge)
        assert P.template_search(td, sd, qa, qb) == (case["peak"], case["lag"], case["ties"]), b
        # 2) per-65,536-lag block records on the NTT path: stride-0 template
        #    rows against overlapping stream rows (no copies)
        want = arr[f"c5_b{b}_blocks"]
        nfull = nvalid // B
        xr = td.expand(nfull, nt)
        yr = torch.as_strided(sd, (nfull, B + nt - 1), (B, 1))
        r = P.estimate_batch(xr, yr, qa, qb, lag_lo=0, lag_hi=B - 1, path="ntt").numpy()
        got = recs(r)
        got[:, 1] += np.arange(nfull, dtype=np.int64) * B
        np.testing.assert_array_equal(got, want[:nfull], err_msg=f"b={b}")
        rl = P.estimate_batch(td[None], sd[nfull * B:][None], qa, qb, lag_lo=0, lag_hi=nvalid - nfull * B - 1,
                              path="ntt").numpy()
        assert (int(rl["value"][0]), int(rl["lag"][0]) + nfull * B, int(rl["ties"][0])) == tuple(want[nfull])
        # 3) every valid-lag value: full correlograms of 2^18-lag blocks
        h = hashlib.sha256()
        B2 = 1 << 18
        n2 = nvalid // B2
        for c0 in range(0, n2, 128):
            c1 = min(n2, c0 + 128)
            yr = torch.as_strided(sd[c0 * B2:], (c1 - c0, B2 + nt - 1), (B2, 1))
            vals, _ = xcorr_full_device(td.expand(c1 - c0, nt), yr, qa, qb)
            h.update(vals[:, nt - 1:nt - 1 + B2].contiguous().cpu().numpy().tobytes())
            del vals
        if n2 * B2 < nvalid:
            vals, _ = xcorr_full_device(td[None], sd[n2 * B2:][None], qa, qb)
            h.update(vals[0, nt - 1:nt - 1 + nvalid - n2 * B2].contiguous().cpu().numpy().tobytes())
        assert h.hexdigest() == case["valid_sha256"], b
