"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Integer results must be bit-exact."""

import hashlib
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()[:16]


@pytest.fixture(scope="module")
def qx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2509_19974_b200 as P

    return P


def test_native_library_loaded(qx):
    from paper_2509_19974_b200 import _native as N

    N.context()
    import os

    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert "libqxcorr_b200.so" in maps


def test_quantize_kernel_matches_reference(qx, golden, qrec):
    import torch

    from paper_2509_19974_b200.quantize import quantize_device

    meta, arr = golden
    for i, qd in enumerate(meta["quant"]):
        vals, want = arr[f"q{i}_in"], arr[f"q{i}_out"]
        x = torch.from_numpy(vals).cuda()
        codes, sums = quantize_device(qrec(qd), x, with_stats=True)
        assert np.array_equal(codes.cpu().numpy(), want), (i, qd)
        assert int(sums[0, 0]) == int(np.sum(want * want))
        assert int(sums[1, 0]) == int(np.count_nonzero(want))


def test_packed_quantizer_matches_reference(qx, golden, qrec, oracle):
    """qx_quantize_packed (bit-packed b-bit codes, 16-byte vector loads) gives
    the reference's codes: every golden quantiser sweep (+-0, subnormals,
    +-inf, half-steps +-1 ulp) at every field width that holds it, then random
    rows of both float types with misaligned row strides (the scalar-load
    path), lengths not multiple of 4 or 32, and per-row statistics."""
    import torch

    from paper_2509_19974_b200.quantize import packed_bits, quantize_packed, unpack_codes

    meta, arr = golden
    for i, qd in enumerate(meta["quant"]):
        q = qrec(qd)
        vals, want = arr[f"q{i}_in"], arr[f"q{i}_out"]
        x = torch.from_numpy(vals).cuda()
        for bits in (1, 2, 4, 8):
            if (bits == 1 and q.k != 1) or (bits > 1 and q.k > (1 << (bits - 1)) - 1):
                continue
            w, ssq, nnz, fl = quantize_packed(q, x, bits)
            got = unpack_codes(w.cpu().numpy().reshape(-1), vals.size, bits)
            assert np.array_equal(got, want), (i, qd, bits)
            assert int(ssq[0]) == int(np.sum(want * want)) and int(nnz[0]) == int(np.count_nonzero(want))
            assert int(fl[0]) == 0
    rng = np.random.default_rng(41)
    quants = [qx.sign(), qx.uniform(1, 0.6), qx.uniform(7, 0.3), qx.uniform(127, 0.02), qx.custom([-1.0, -0.2, 0.3, 0.9])]
    for trial in range(30):
        q = quants[trial % len(quants)]
        dt = np.float32 if trial % 2 else np.float64
        B, n = int(rng.integers(1, 5)), int(rng.integers(1, 5000))
        ld = n + int(rng.integers(0, 3))  # odd strides defeat 16-byte alignment
        buf = (rng.standard_normal((B, ld)) * 2).astype(dt)
        x = torch.from_numpy(buf).cuda()[:, :n]
        bits = packed_bits(q) if trial % 3 else (1 if q.k == 1 else packed_bits(q))
        w, ssq, nnz, fl = quantize_packed(q, x, bits)
        w = w.cpu().numpy()
        for b in range(B):
            want = oracle.quantize(q, buf[b, :n])
            assert np.array_equal(unpack_codes(w[b], n, bits), want), (trial, b)
            assert int(ssq[b]) == int(np.sum(want * want)) and int(nnz[b]) == int(np.count_nonzero(want))
    # NaN is flagged; fields that cannot hold the codes are refused
    x = torch.tensor([0.5, float("nan"), -2.0], dtype=torch.float32, device="cuda")
    assert int(quantize_packed(qx.sign(), x, 2)[3][0]) == 4
    with pytest.raises(ValueError):
        quantize_packed(qx.uniform(7, 0.3), x, 2)
    with pytest.raises(ValueError):
        quantize_packed(qx.uniform(2, 0.3), x, 1)


def test_apply_and_call(qx):
    q = qx.uniform(4, 1.0)
    assert q([0.49, 0.5, 1.49, 1.5, -0.5, -1.5]).tolist() == [0, 1, 1, 2, -1, -2]
    assert qx.sign()([-3.5, -0.0, 0.0, 1e-12, 2.0]).tolist() == [-1, 0, 0, 1, 1]
    s = qx.Signal(-3, [0.2, -1.7, 0.0])
    out = qx.apply(qx.uniform(2, 1.0), s)
    assert out.start == -3 and out.samples.tolist() == [0, -2, 0] and out.bound == 2


def test_xcorr_full_matches_reference(qx, golden):
    meta, arr = golden
    for i, d in enumerate(meta["xcorr"]):
        u = qx.IntSignal(d["u_start"], arr[f"x{i}_u"], d["ku"])
        v = qx.IntSignal(d["v_start"], arr[f"x{i}_v"], d["kv"])
        c = qx.xcorr_int_bf(u, v)
        assert c.first_lag == d["first_lag"], i
        assert np.array_equal(c.values, arr[f"x{i}_c"]), i
        assert c.norm_x == d["norm_x"] and c.norm_y == d["norm_y"]
        assert qx.argmax_set(c) == d["argmax"]


def test_acceptance_criterion2_on_gpu(qx, golden):
    """The 1000 seeded pairs of the reference's acceptance criterion 2,
    correlated on the GPU, hash to the reference's brute-force digests."""
    import test_oracle_golden as T

    meta, _ = golden
    acc = meta["acceptance_c2"]
    fixed = T._edge_pairs()
    for rec in acc["records"]:
        if "skipped" in rec:
            continue
        (su, u, ku), (sv, v, kv) = T._acceptance_pair(acc["seed"], rec["case"], fixed)
        c = qx.xcorr_int_gpu(qx.IntSignal(su, u, ku), qx.IntSignal(sv, v, kv))
        assert sha(c.values) == rec["sha"] and c.first_lag == rec["first_lag"], rec


def _q(qx, d):
    if d["kind"] == "sign":
        return qx.sign()
    if d["kind"] == "uniform":
        return qx.uniform(d["k"], d["step"])
    return qx.custom(d["thresholds"])


def test_estimate_matches_reference(qx, golden):
    meta, arr = golden
    for i, d in enumerate(meta["estimate"]):
        x = qx.Signal(d["x_start"], arr[f"e{i}_x"])
        y = qx.Signal(d["y_start"], arr[f"e{i}_y"])
        want = d["result"]
        kw = dict(d["kw"])
        if "raises" in want:
            with pytest.raises(Exception) as ei:
                qx.estimate(x, y, _q(qx, d["qx"]), _q(qx, d["qy"]), **kw)
            assert type(ei.value).__name__ == want["raises"], (i, want)
            continue
        r = qx.estimate(x, y, _q(qx, d["qx"]), _q(qx, d["qy"]), **kw)
        assert list(r.lags) == want["lags"], (i, r, want)
        assert r.peak_value_int == want["peak"]
        assert r.tie_broken == want["tie_broken"]
        assert [[a, b] for a, b in r.tie_break_values] == want["tie_break_values"]
        assert r.method == want["method"]


def test_c1(qx, golden):
    from paper_2509_19974_b200 import workloads as W

    meta, _ = golden
    x, y = W.c1(0)
    r = qx.estimate(qx.Signal(0, x), qx.Signal(0, y), qx.sign(), qx.sign())
    g = meta["configs"]["c1"]
    assert list(r.lags) == g["lags"] == [-137] and r.peak_value_int == g["peak"] == 14839


def test_c2_golden_pairs(qx, golden):
    import torch

    from paper_2509_19974_b200 import workloads as W
    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    meta, _ = golden
    xs, ys, lag = W.c2(pairs=3)
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    for b in (1, 2, 4, 8):
        q = W.bit_quantizer(b, W.C2_SIGMA)
        res = qx.estimate_batch(xd, yd, q, q).numpy()
        vals, _ = xcorr_full_device(xd, yd, q, q)
        for g in [g for g in meta["configs"]["c2"] if g["b"] == b]:
            p = g["pair"]
            assert res["value"][p] == g["peak"] and res["lag"][p] == g["lags"][0]
            assert res["ties"][p] == len(g["lags"])
            assert res["sumsq_x"][p] == g["sumsq_u"] and res["sumsq_y"][p] == g["sumsq_v"]
            assert sha(vals[p].cpu().numpy()) == g["sha"], (b, p)
            assert g["lags"][0] == g["expected"]


def test_c3_golden_window(qx, golden):
    import torch

    from paper_2509_19974_b200 import workloads as W
    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    meta, _ = golden
    xs, ys, lag = W.c3(pairs=256)
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    for b in (2, 4):
        q = W.bit_quantizer(b, W.C3_SIGMA)
        res = qx.estimate_batch(xd, yd, q, q, lag_lo=-512, lag_hi=512).numpy()
        vals, _ = xcorr_full_device(xd, yd, q, q)
        first = -(W.C3_N - 1)
        win = vals[:, -512 - first:-512 - first + 1025].cpu().numpy()
        for g in [g for g in meta["configs"]["c3"] if g["b"] == b]:
            p = g["pair"]
            assert res["value"][p] == g["peak"] and res["lag"][p] == g["lags"][0], (b, p)
            assert res["ties"][p] == len(g["lags"])
            assert sha(win[p]) == g["sha"]


def test_c4_small_and_c5_small(qx, golden):
    import torch

    from paper_2509_19974_b200 import workloads as W
    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    meta, _ = golden
    g = meta["configs"]["c4_small"]
    x4, y4, l4 = W.c4(n=g["n"], delay=g["delay"])
    q4 = W.bit_quantizer(4, W.C4_SIGMA)
    r = qx.estimate(qx.Signal(0, x4), qx.Signal(0, y4), q4, q4)
    assert list(r.lags) == g["lags"] and r.peak_value_int == g["peak"]
    vals, _ = xcorr_full_device(torch.from_numpy(x4).cuda(), torch.from_numpy(y4).cuda(), q4, q4)
    assert sha(vals[0].cpu().numpy()) == g["sha"]
    g5 = meta["configs"]["c5_small"]
    t5, s5, off, sn2 = W.c5(stream=g5["stream"], template=g5["template"], offset=g5["offset"])
    for case in g5["cases"]:
        qa, qb = _q(qx, case["qx"]), _q(qx, case["qy"])
        nvalid = g5["stream"] - g5["template"]
        res = qx.estimate_batch(t5[None], s5[None], qa, qb, lag_lo=0, lag_hi=nvalid).numpy()
        assert res["value"][0] == case["peak"] and res["lag"][0] == case["lags"][0]
        assert res["ties"][0] == len(case["lags"]) and case["lags"][0] == off


def test_random_pairs_against_oracle(qx, oracle):
    """Seeded sweep of lengths, quantisers, dtypes and windows vs the oracle."""
    import torch

    rng = np.random.default_rng(7)
    quants = [qx.sign(), qx.uniform(1, 0.7), qx.uniform(7, 0.3), qx.uniform(127, 0.02),
              qx.custom([-1.0, -0.2, 0.3, 1.1]), qx.uniform(40, 0.05)]
    for trial in range(60):
        B = int(rng.integers(1, 5))
        nx = int(rng.integers(1, 3000))
        ny = int(rng.integers(1, 3000))
        dt = np.float32 if trial % 2 else np.float64
        x = (rng.standard_normal((B, nx)) * rng.uniform(0.1, 3)).astype(dt)
        y = (rng.standard_normal((B, ny)) * rng.uniform(0.1, 3)).astype(dt)
        qa = quants[int(rng.integers(len(quants)))]
        qb = quants[int(rng.integers(len(quants)))]
        nout = nx + ny - 1
        t_lo = int(rng.integers(0, nout))
        t_hi = int(rng.integers(t_lo, nout))
        first = -(nx - 1)
        res = qx.estimate_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), qa, qb,
                                lag_lo=first + t_lo, lag_hi=first + t_hi).numpy()
        for b in range(B):
            u, v = oracle.quantize(qa, x[b]), oracle.quantize(qb, y[b])
            if not u.any() or not v.any():
                assert res["status"][b] == 2
                continue
            c = oracle.xcorr_bf(u, v, t_lo, t_hi)
            m, f, n = oracle.argmax(c)
            assert (res["value"][b], res["lag"][b], res["ties"][b]) == (m, first + t_lo + f, n), trial
            assert res["sumsq_x"][b] == oracle.sumsq(u) and res["sumsq_y"][b] == oracle.sumsq(v)


def test_ntt_argmax_ties_and_windows(qx):
    """The fused argmax of the last NTT pass (shared warp threshold, per-CTA
    partials merged by k_merge_partials): impulse trains make every correlation
    value small, so maxima tie many times across lanes, warps and CTAs; windows
    start and end inside column tiles.  Expected records from the sparse sum."""
    import torch

    rng = np.random.default_rng(11)
    q = qx.uniform(1, 1.0)
    for n in (1 << 11, 1 << 14, 3 * 5000, 1 << 18, (1 << 19) + 3):  # the last one: large-P outer passes
        B = 6
        x = np.zeros((B, n), np.float32)
        y = np.zeros((B, n), np.float32)
        for r in range(B):
            x[r, rng.choice(n, 2 + 3 * r, replace=False)] = rng.choice([-1.0, 1.0], 2 + 3 * r)
            y[r, rng.choice(n, 3 + 2 * r, replace=False)] = rng.choice([-1.0, 1.0], 3 + 2 * r)
        x[B - 1] = 0.0
        x[B - 1, [5, n - 7]] = 1.0  # two equal impulses against a constant row: long runs of ties
        y[B - 1] = 1.0
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        windows = [(-(n - 1), n - 1), (-37, 1000), (n // 3, n - 1), (-(n - 1), -(n - 1) + 40), (-1, -1)]
        for lo, hi in windows:
            res = qx.estimate_batch(xd, yd, q, q, path="ntt", lag_lo=lo, lag_hi=hi).numpy()
            for r in range(B):
                ix, iy = np.nonzero(x[r])[0], np.nonzero(y[r])[0]
                lag = (iy[None, :] - ix[:, None]).ravel()
                val = (x[r, ix][:, None] * y[r, iy][None, :]).ravel().astype(np.int64)
                c = np.zeros(hi - lo + 1, np.int64)
                keep = (lag >= lo) & (lag <= hi)
                np.add.at(c, lag[keep] - lo, val[keep])
                m = int(c.max())
                f = int(np.argmax(c))
                assert (int(res["value"][r]), int(res["lag"][r]), int(res["ties"][r])) == \
                    (m, lo + f, int((c == m).sum())), (n, lo, hi, r)


def test_medium_pairs_against_oracle(qx, oracle):
    """Seeded sweep over the middle of the NTT size range (P = 2^13 .. 2^19, every
    four-step shape, operands with and without the zero-upper half), random
    windows, quantisers and dtypes, against the oracle's Kronecker substitution."""
    import torch

    rng = np.random.default_rng(21)
    quants = [qx.sign(), qx.uniform(1, 0.7), qx.uniform(7, 0.3), qx.uniform(127, 0.02),
              qx.custom([-1.0, -0.2, 0.3, 1.1])]
    for trial in range(24):
        lp = 13 + trial % 7
        tot = int(rng.integers((1 << (lp - 1)) + 2, (1 << lp) + 1))  # nx + ny - 1 in (2^(lp-1), 2^lp]
        nx = int(rng.integers(max(1, tot // 8), tot - max(1, tot // 8)))
        ny = tot + 1 - nx
        dt = np.float32 if trial % 3 else np.float64
        B = 2
        x = (rng.standard_normal((B, nx)) * rng.uniform(0.3, 2)).astype(dt)
        y = (rng.standard_normal((B, ny)) * rng.uniform(0.3, 2)).astype(dt)
        qa = quants[int(rng.integers(len(quants)))]
        qb = quants[int(rng.integers(len(quants)))]
        nout = nx + ny - 1
        t_lo = int(rng.integers(0, nout)) if trial % 2 else 0
        t_hi = int(rng.integers(t_lo, nout)) if trial % 2 else nout - 1
        first = -(nx - 1)
        res = qx.estimate_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), qa, qb, path="ntt",
                                lag_lo=first + t_lo, lag_hi=first + t_hi).numpy()
        for b in range(B):
            u, v = oracle.quantize(qa, x[b]), oracle.quantize(qb, y[b])
            c = oracle.xcorr_ks(u, v, qa.k, qb.k)[t_lo:t_hi + 1]
            m, f, n = oracle.argmax(c)
            assert (res["value"][b], res["lag"][b], res["ties"][b]) == (m, first + t_lo + f, n), (trial, lp, nx, ny)


def test_row_layouts_agree_on_every_path(qx):
    """Rows that overlap (stride < length), are padded (stride > length) or are
    one shared row (stride 0) give the records of their contiguous copies, on
    the NTT, tensor-core window and popc paths (float32 and float64)."""
    import torch

    rng = np.random.default_rng(15)
    for dt in (torch.float32, torch.float64):
        for path, n, win, q in [("ntt", 5000, (None, None), qx.uniform(7, 0.3)),
                                ("ntt", 70000, (-300, 9000), qx.uniform(1, 0.6)),
                                ("direct", 4096, (-512, 512), qx.uniform(7, 0.3)),
                                ("direct", 3000, (-40, 1999), qx.sign()),
                                ("popc", 6000, (None, None), qx.sign())]:
            B = 5
            base_x = torch.from_numpy(rng.standard_normal(n * (B + 2))).to(dt).cuda()
            base_y = torch.from_numpy(rng.standard_normal(n * (B + 2))).to(dt).cuda()
            for ld in (n // 3, n + 13, 0):
                x = base_x.as_strided((B, n), (ld, 1))
                y = base_y.as_strided((B, n), (ld if ld else n, 1))  # y keeps distinct rows when x is shared
                got = qx.estimate_batch(x, y, q, q, path=path, lag_lo=win[0], lag_hi=win[1]).numpy()
                want = qx.estimate_batch(x.contiguous(), y.contiguous(), q, q, path=path, lag_lo=win[0],
                                         lag_hi=win[1]).numpy()
                assert np.array_equal(got, want), (dt, path, n, ld)


def test_signal_starts_shift_lags_on_every_path(qx):
    """Signal.start offsets only translate the lag axis (first_lag = y.start -
    (x.start + N_x - 1), intxcorr.py:85-86): a call with starts and a window
    equals the zero-start call on the translated window, lags shifted back."""
    import torch

    rng = np.random.default_rng(16)
    for path, n, q in [("ntt", 9000, qx.uniform(7, 0.3)), ("direct", 4096, qx.uniform(1, 0.6)),
                       ("popc", 5000, qx.sign()), ("ntt", (1 << 19) + 5, qx.uniform(1, 0.6))]:
        x = torch.from_numpy(rng.standard_normal((3, n)).astype(np.float32)).cuda()
        y = torch.from_numpy(rng.standard_normal((3, n)).astype(np.float32)).cuda()
        for sx, sy in [(0, 0), (17, -250), (-100000, 3), (5, 5)]:
            d = sy - sx
            for lo, hi in [(-700, 600), (d - 3, d + 3), (-(n - 1) + d, -(n - 1) + d + 1000)]:
                if lo - d < -(n - 1) or hi - d > n - 1:
                    continue
                a = qx.estimate_batch(x, y, q, q, path=path, x_start=sx, y_start=sy, lag_lo=lo, lag_hi=hi).numpy()
                b = qx.estimate_batch(x, y, q, q, path=path, lag_lo=lo - d, lag_hi=hi - d).numpy()
                assert np.array_equal(a["lag"], b["lag"] + d), (path, n, sx, sy, lo, hi)
                for f in ("value", "ties", "sumsq_x", "sumsq_y", "status"):
                    assert np.array_equal(a[f], b[f]), (path, n, sx, sy, lo, hi, f)


def _sparse_peak(xr, yr, lo, hi):
    """(max, smallest lag, count) of the correlation of two impulse trains over lags lo..hi"""
    ix, iy = np.nonzero(xr)[0], np.nonzero(yr)[0]
    lag = (iy[None, :] - ix[:, None]).ravel()
    val = (np.rint(xr[ix])[:, None] * np.rint(yr[iy])[None, :]).ravel().astype(np.int64)
    c = np.zeros(hi - lo + 1, np.int64)
    keep = (lag >= lo) & (lag <= hi)
    np.add.at(c, lag[keep] - lo, val[keep])
    m = int(c.max())
    return m, lo + int(np.argmax(c)), int((c == m).sum())


def test_window_and_template_paths_with_ties(qx):
    """Tensor-core window path (int8 tiles, extra lags, both tile sizes), the popc
    path and the blocked template search on impulse trains: small values, so
    maxima tie across epilogue lanes, tiles, CTAs and blocks; the smallest lag
    and the tie count must match the sparse sum."""
    import torch

    rng = np.random.default_rng(12)
    for k in (1, 7):
        q = qx.uniform(k, 1.0)
        for n in (4096, 3001):
            B = 8
            x = np.zeros((B, n), np.float32)
            y = np.zeros((B, n), np.float32)
            for r in range(B):
                x[r, rng.choice(n, 4 + 5 * r, replace=False)] = rng.choice([-1.0, 1.0], 4 + 5 * r)
                y[r, rng.choice(n, 6 + 3 * r, replace=False)] = rng.choice([-1.0, 1.0], 6 + 3 * r)
            xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
            for lo, hi in [(-512, 512), (-2056, 2055), (-5, 3), (100, 100), (-1500, 37), (-(n - 1), -(n - 1) + 900)]:
                for path in (["direct", "ntt", "popc"] if k == 1 else ["direct", "ntt"]):
                    res = qx.estimate_batch(xd, yd, q, q, path=path, lag_lo=lo, lag_hi=hi).numpy()
                    for r in range(B):
                        assert (int(res["value"][r]), int(res["lag"][r]), int(res["ties"][r])) == \
                            _sparse_peak(x[r], y[r], lo, hi), (k, n, lo, hi, path, r)
    # template search: impulse template against an impulse stream, several blocks,
    # some of them without a single non-zero stream sample
    for k, nt, ns in [(1, 4096, 4096 + 5 * 8192 + 77), (1, 4096, 60000), (7, 4096, 50000), (1, 1000, 30000)]:
        q = qx.uniform(k, 1.0)
        tpl = np.zeros(nt, np.float32)
        st = np.zeros(ns, np.float32)
        tpl[rng.choice(nt, 9, replace=False)] = rng.choice([-1.0, 1.0], 9)
        st[rng.choice(ns // 2, 40, replace=False)] = rng.choice([-1.0, 1.0], 40)  # second half silent
        got = qx.template_search(torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda(), q, q)
        assert got == _sparse_peak(tpl, st, 0, ns - nt), (k, nt, ns)
        for block in (5000, 1 << 14):  # NTT blocks: ties across block summaries
            got = qx.template_search(torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda(), q, q, block=block,
                                     path="ntt")
            assert got == _sparse_peak(tpl, st, 0, ns - nt), (k, nt, ns, block)


def test_popc_path_against_oracle(qx, oracle):
    """Word-parallel 1-level path (path="popc", and what "auto" picks for
    C1-sized pairs): sign / uniform(1) / custom k=1 codes, with and without
    zero codes (the 1-POPC and 2-POPC forms), ragged lengths, windows,
    batches, both float dtypes; values, lags, ties and statistics equal the
    oracle's and the NTT path's."""
    import torch

    from paper_2509_19974_b200 import _native

    rng = np.random.default_rng(31)
    quants = [qx.sign(), qx.uniform(1, 0.7), qx.custom([-0.3, 0.4]), qx.uniform(1, 5.0)]
    for trial in range(40):
        B = int(rng.integers(1, 4))
        nx = int(rng.integers(1, 9000)) if trial % 5 else int(rng.integers(16000, 40000))
        ny = int(rng.integers(1, 9000)) if trial % 7 else int(rng.integers(16000, 40000))
        dt = np.float32 if trial % 2 else np.float64
        x = (rng.standard_normal((B, nx)) * rng.uniform(0.1, 3)).astype(dt)
        y = (rng.standard_normal((B, ny)) * rng.uniform(0.1, 3)).astype(dt)
        if trial % 3 == 0:  # exact zeros: sign() codes 0
            x[:, ::7] = 0
            y[:, ::5] = 0
        qa, qb = quants[trial % 4], quants[(trial // 4) % 4]
        nout = nx + ny - 1
        t_lo, t_hi = (0, nout - 1) if trial % 4 == 0 else sorted(int(v) for v in rng.integers(0, nout, 2))
        first = -(nx - 1)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        with _native.profile(timed=False) as prof:
            res = qx.estimate_batch(xd, yd, qa, qb, lag_lo=first + t_lo, lag_hi=first + t_hi, path="popc").numpy()
        assert prof.result.get("popc", (0, 0))[0] >= 1, prof.result  # fused, or planes + correlation
        ntt = qx.estimate_batch(xd, yd, qa, qb, lag_lo=first + t_lo, lag_hi=first + t_hi, path="ntt").numpy()
        assert np.array_equal(res, ntt), (trial, res, ntt)
        for b in range(B):
            u, v = oracle.quantize(qa, x[b]), oracle.quantize(qb, y[b])
            if not u.any() or not v.any():
                assert res["status"][b] == 2
                continue
            m, f, n = oracle.argmax(oracle.xcorr_bf(u, v, t_lo, t_hi))
            assert (res["value"][b], res["lag"][b], res["ties"][b]) == (m, first + t_lo + f, n), trial
            assert res["sumsq_y"][b] == oracle.sumsq(v) and res["nnz_x"][b] == np.count_nonzero(u)
    # C1 takes this path by default; NaN raises like the reference's float path
    from paper_2509_19974_b200 import workloads as W

    x, y = W.c1(0)
    with _native.profile(timed=False) as prof:
        r = qx.estimate_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), qx.sign(), qx.sign()).numpy()
    assert list(prof.result) == ["popc"] and (int(r["lag"][0]), int(r["value"][0])) == (-137, 14839)
    x[5] = np.nan
    r = qx.estimate_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), qx.sign(), qx.sign()).numpy()
    assert r["status"][0] == 9


def test_popc_batches_and_cluster_counts(qx):
    """The cluster popc kernel splits a pair over several 8-CTA clusters
    (few pairs) or gives each pair one cluster in several waves (batches
    larger than the resident clusters); every split gives the NTT path's
    records, statistics included, on random and constant (all-tie) rows."""
    import torch

    rng = np.random.default_rng(32)
    for B, nx, ny in ((1, 16384, 16384), (3, 5000, 7001), (40, 300, 257), (200, 64, 64), (2, 65536, 300)):
        x = torch.from_numpy(rng.standard_normal((B, nx)).astype(np.float32)).cuda()
        y = torch.from_numpy(rng.standard_normal((B, ny)).astype(np.float32)).cuda()
        if B == 3:
            x[1] = 1.0  # every lag of pair 1 ties on overlap counts
        q = qx.sign()
        a = qx.estimate_batch(x, y, q, q, path="popc").numpy()
        b = qx.estimate_batch(x, y, q, q, path="ntt").numpy()
        assert np.array_equal(a, b), (B, nx, ny)


def test_multiprime_path_saturated(qx, oracle):
    """Saturated b=8 codes defeat the Cauchy-Schwarz single-prime test, so
    the 2-prime CRT path must reproduce the exact (large) values."""
    import torch

    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    rng = np.random.default_rng(9)
    n = 1 << 16
    x = (rng.standard_normal(n) + 30).astype(np.float32)
    y = (rng.standard_normal(n) + 30).astype(np.float32)
    y[::97] *= -1
    x[::89] = 0.0
    q = qx.uniform(127, 0.1)
    u, v = oracle.quantize(q, x), oracle.quantize(q, y)
    want = oracle.xcorr_ks(u, v, 127, 127)
    assert np.abs(want).max() > 600_000_000  # beyond a single prime's centred range
    vals, _ = xcorr_full_device(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), q, q)
    assert np.array_equal(vals[0].cpu().numpy(), want)
    res = qx.estimate_batch(x[None], y[None], q, q).numpy()
    m, f, cnt = oracle.argmax(want)
    assert (res["value"][0], res["lag"][0], res["ties"][0]) == (m, -(n - 1) + f, cnt)


def test_launch_groups_mixed_primes(qx, oracle):
    """A batch split into launch groups (chunk_pairs) where some pairs finish on
    one prime (Cauchy-Schwarz) and others need the two-prime CRT: records and
    full correlograms equal the oracle and do not depend on the grouping."""
    import torch

    from paper_2509_19974_b200 import _native
    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    rng = np.random.default_rng(10)
    B, n = 7, 1 << 16
    x = rng.standard_normal((B, n)).astype(np.float32)
    y = rng.standard_normal((B, n)).astype(np.float32)
    for b in (1, 4, 6):  # saturated rows: beyond a single prime's centred range
        x[b] += 30
        y[b] += 30
        y[b, ::97] *= -1
    q = qx.uniform(127, 0.1)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    want = []
    for b in range(B):
        c = oracle.xcorr_ks(oracle.quantize(q, x[b]), oracle.quantize(q, y[b]), 127, 127)
        want.append(c)
    assert max(np.abs(c).max() for c in want) > 600_000_000 > min(np.abs(c).max() for c in want)
    for chunk in (0, 1, 3):
        with _native.option("chunk_pairs", chunk):
            res = qx.estimate_batch(xd, yd, q, q, path="ntt").numpy()
            vals, _ = xcorr_full_device(xd, yd, q, q)
        for b in range(B):
            m, f, cnt = oracle.argmax(want[b])
            assert (res["value"][b], res["lag"][b], res["ties"][b]) == (m, -(n - 1) + f, cnt), (chunk, b)
            assert np.array_equal(vals[b].cpu().numpy(), want[b]), (chunk, b)


def test_errors_match_reference(qx):
    with pytest.raises(qx.DegenerateQuantization, match="x quantizes"):
        qx.estimate(qx.Signal(0, [0.01, -0.02, 0.03]), qx.Signal(0, [1.0, -1.0, 1.0]), qx.uniform(4, 1.0),
                    qx.uniform(4, 1.0))
    with pytest.raises(qx.DegenerateQuantization, match="y quantizes"):
        qx.estimate(qx.Signal(0, [1.0, -1.0, 1.0]), qx.Signal(0, [0.01, -0.02, 0.03]), qx.uniform(4, 1.0),
                    qx.uniform(4, 1.0))
    with pytest.raises(ValueError):
        qx.estimate(qx.Signal(0, [1.0, -1.0]), qx.Signal(0, [1.0, -1.0]), qx.sign(), qx.sign(), method="phat")
    huge = qx.IntSignal(0, [1, 1], bound=1 << 40)
    with pytest.raises(ValueError):
        qx.xcorr_int_bf(huge, huge)
    with pytest.raises(qx.DegenerateInput):
        qx.xcorr_int_ks(qx.IntSignal(0, [0, 0], 1), qx.IntSignal(0, [1], 1))
    with pytest.raises(ValueError):
        qx.estimate(qx.Signal(0, [1.0, np.nan]), qx.Signal(0, [1.0, 2.0]), qx.sign(), qx.sign())
    with pytest.raises(ValueError):
        qx.estimate_batch(np.ones((1, 8), np.float32), np.ones((1, 8), np.float32), qx.sign(), qx.sign(),
                          lag_lo=100, lag_hi=200)


def test_host_entry_point(qx, oracle):
    from paper_2509_19974_b200 import workloads as W

    xs, ys, lag = W.c2(pairs=2, n=1 << 14)
    q = W.bit_quantizer(2, W.C2_SIGMA)
    res = qx.estimate_batch_host(xs, ys, q, q)
    want = oracle.estimate_batch_f32(xs, ys, q, q)
    assert np.array_equal(res["value"], want[:, 0])
    assert np.array_equal(res["lag"], want[:, 1] - (xs.shape[1] - 1))
    assert np.array_equal(res["ties"], want[:, 2])


def test_sweep_host_entry_point(qx, oracle):
    """qx_estimate_sweep_host: several quantiser pairs, chunked staging with
    copy/compute overlap, full-lag (NTT) and windowed (tensor-core) paths."""
    from paper_2509_19974_b200 import workloads as W

    xs, ys, lag = W.c2(pairs=11, n=1 << 12)
    qs = [(W.bit_quantizer(b, W.C2_SIGMA), W.bit_quantizer(b, W.C2_SIGMA)) for b in (1, 2, 4, 8)]
    qs.append((qx.uniform(3, 0.4), qx.sign()))
    for lo, hi in ((None, None), (-700, 700)):
        res = qx.estimate_sweep_host(xs, ys, qs, lag_lo=lo, lag_hi=hi)
        assert res.shape == (len(qs), xs.shape[0])
        for q, (a, b) in enumerate(qs):
            one = qx.estimate_batch_host(xs, ys, a, b, lag_lo=lo, lag_hi=hi)
            assert np.array_equal(res[q], one), q
            if lo is None:
                want = oracle.estimate_batch_f32(xs, ys, a, b)
                assert np.array_equal(res[q]["value"], want[:, 0])
                assert np.array_equal(res[q]["lag"], want[:, 1] - (xs.shape[1] - 1))
                assert np.array_equal(res[q]["ties"], want[:, 2])


@pytest.mark.parametrize("lanes", [None, "1", "3"])
def test_device_sweep_entry_point(qx, oracle, lanes):
    """qx_estimate_sweep: device rows, quantiser pairs on forked compute lanes
    joined back to the caller's stream; equals one estimate_batch per pair and
    the oracle, and a kernel on the caller's stream right after the call sees
    finished results."""
    import torch
    from paper_2509_19974_b200 import _native as N, workloads as W

    with N.option("sweep_lanes", int(lanes or 0)):
        _device_sweep_checks(qx, oracle, torch, W)


def _device_sweep_checks(qx, oracle, torch, W):
    xs, ys, lag = W.c2(pairs=6, n=1 << 12, seed=5)
    qs = [(W.bit_quantizer(b, W.C2_SIGMA), W.bit_quantizer(b, W.C2_SIGMA)) for b in (1, 2, 4, 8)]
    qs.append((qx.uniform(3, 0.4), qx.sign()))
    dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    for lo, hi in ((None, None), (-700, 700)):
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            res = qx.estimate_sweep(dx, dy, qs, lag_lo=lo, lag_hi=hi)
            summed = torch.stack([r.value for r in res]).sum()  # consumer on the caller's stream
        side.synchronize()
        assert len(res) == len(qs)
        tot = 0
        for q, (a, b) in enumerate(qs):
            one = qx.estimate_batch(dx, dy, a, b, lag_lo=lo, lag_hi=hi)
            torch.cuda.synchronize()
            assert torch.equal(res[q].raw, one.raw), q
            tot += int(one.value.sum())
            if lo is None:
                want = oracle.estimate_batch_f32(xs, ys, a, b)
                assert np.array_equal(res[q].value.cpu().numpy(), want[:, 0])
                assert np.array_equal(res[q].lag.cpu().numpy(), want[:, 1] - (xs.shape[1] - 1))
        assert int(summed) == tot


@pytest.mark.parametrize("pairs", [1, 5, 17, 40, 67])
@pytest.mark.parametrize("knobs", [{}, {"sweep_lanes": 1}, {"sweep_chunks": 7, "sweep_taper": 3},
                                   {"sweep_lanes": 2, "sweep_chunks": 64}, {"sweep_even": 1}])
def test_sweep_host_chunk_schedules(qx, pairs, knobs):
    """Every chunk/lane/taper schedule of qx_estimate_sweep_host covers each
    pair exactly once: results equal per-quantiser estimate_batch_host calls
    for ragged batch sizes (1 pair, primes, more chunks than pairs)."""
    import contextlib

    from paper_2509_19974_b200 import _native as N, workloads as W

    with contextlib.ExitStack() as stack:
        for k, v in knobs.items():
            stack.enter_context(N.option(k, v))
        _sweep_host_checks(qx, W, pairs)
    # overlapping rows (0 < ld < n, through the C ABI) are staged whole
    # whatever the chunk option (a chunk count would read past the buffer)
    import ctypes

    from paper_2509_19974_b200.quantize import native_quantizer

    with N.option("sweep_chunks", 5):
        base = np.random.default_rng(pairs).standard_normal(2000 + 160 * pairs).astype(np.float32)
        sx = N.QxSignals(base.ctypes.data, N.QX_F32, 0, 2000, 160, 0)
        sy = N.QxSignals(base[37:].ctypes.data, N.QX_F32, 0, 1900, 160, 0)
        q = qx.uniform(3, 0.4)
        nq, _ = native_quantizer(q)
        res = np.zeros(pairs, dtype=N.RESULT_DTYPE)
        st = N.load().qx_estimate_sweep_host(N.context(), ctypes.byref(sx), ctypes.byref(sy), pairs, 1,
                                             ctypes.byref(nq), ctypes.byref(nq), N.INT64_MIN, N.INT64_MAX, 0,
                                             res.ctypes.data)
        assert st == 0
        xo = np.lib.stride_tricks.as_strided(base, (pairs, 2000), (640, 4))
        yo = np.lib.stride_tricks.as_strided(base[37:], (pairs, 1900), (640, 4))
        assert np.array_equal(res, qx.estimate_batch_host(np.ascontiguousarray(xo), np.ascontiguousarray(yo), q, q))


def _sweep_host_checks(qx, W, pairs):
    xs, ys, lag = W.c2(pairs=pairs, n=1 << 10, seed=pairs)
    qs = [(W.bit_quantizer(b, W.C2_SIGMA), W.bit_quantizer(b, W.C2_SIGMA)) for b in (1, 2, 8)]
    qs.append((qx.uniform(3, 0.4), qx.sign()))
    for lo, hi in ((None, None), (-300, 300)):
        res = qx.estimate_sweep_host(xs, ys, qs, lag_lo=lo, lag_hi=hi)
        assert res.shape == (len(qs), pairs)
        for q, (a, b) in enumerate(qs):
            one = qx.estimate_batch_host(xs, ys, a, b, lag_lo=lo, lag_hi=hi)
            assert np.array_equal(res[q], one), (q, lo)


def test_big_mul_cuda_backend(qx):
    """The reference's plugin slot big_mul (intxcorr.py:183-205) with backend
    "cuda": worked product and identities (pkg/tests/test_intxcorr.py:139-149),
    random 4096-bit operands against the interpreter (150-158), and large
    unbalanced operands that need the multi-prime NTT path and every carry
    plane; auto switches to cuda from CUDA_MIN_BITS."""
    from paper_2509_19974_b200 import intxcorr as IX

    assert qx.big_mul(257, 515, "cuda") == 132355
    assert qx.big_mul(123456789, 0, "cuda") == 0
    assert qx.big_mul(123456789, 1, "cuda") == 123456789
    assert qx.big_mul(-7, 9, "cuda") == -63
    assert qx.big_mul(-7, -9, "cuda") == 63
    rng = np.random.default_rng(5)
    for _ in range(10):
        a = int.from_bytes(rng.bytes(512), "little")
        b = int.from_bytes(rng.bytes(512), "little")
        assert qx.big_mul(a, b, "cuda") == a * b
    for na, nb in ((1 << 17, 1 << 17), (1 << 20, 3 << 16), (5, 1 << 21)):
        a = int.from_bytes(rng.bytes(na), "little") | (1 << (8 * na - 1))
        b = int.from_bytes(rng.bytes(nb), "little") | 1
        assert qx.big_mul(a, -b, "cuda") == -(a * b)
    allones = (1 << (1 << 20)) - 1  # every limb 0xffff: maximal coefficients and carries
    assert qx.big_mul(allones, allones, "cuda") == allones * allones
    a = (1 << IX.CUDA_MIN_BITS) + 12345
    assert qx.big_mul(a, a, "auto") == a * a


def test_c2_full_size_properties(qx, oracle):
    """BASELINE config 2 at full size (64 pairs x 2^18, b = 1, 2, 4, 8): every
    pair finds its true delay; a sample of pairs is checked exactly against
    the oracle's Kronecker-substitution correlation (GMP)."""
    import torch

    from paper_2509_19974_b200 import workloads as W

    xs, ys, lag = W.c2()
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    for b in (1, 2, 4, 8):
        q = W.bit_quantizer(b, W.C2_SIGMA)
        res = qx.estimate_batch(xd, yd, q, q).numpy()
        assert np.array_equal(res["lag"], lag), b
        assert np.all(res["ties"] == 1) and np.all(res["status"] == 0)
        sel = [0, 17, 63]
        want = oracle.estimate_batch_f32(xs[sel], ys[sel], q, q, threads=3)
        assert np.array_equal(res["value"][sel], want[:, 0])
        assert np.array_equal(res["lag"][sel], want[:, 1] - (W.C2_N - 1))


def test_template_search_matches_oracle(qx, oracle, golden):
    """Overlap-save template search (config 5 path): tiny blocks force many
    overlapping strided windows plus a remainder block."""
    from paper_2509_19974_b200 import workloads as W

    rng = np.random.default_rng(21)
    for trial in range(6):
        nt = int(rng.integers(1, 300))
        ns = int(rng.integers(nt, 5000))
        st = rng.laplace(size=ns).astype(np.float32 if trial % 2 else np.float64)
        off = int(rng.integers(0, ns - nt + 1))
        tpl = st[off:off + nt].copy()
        st = st + rng.normal(0, 0.5, ns).astype(st.dtype)
        q = [qx.sign(), qx.uniform(1, 0.8), qx.uniform(7, 0.3)][trial % 3]
        block = int(rng.integers(1, 700))
        got = qx.template_search(tpl, st, q, q, stream_start=5, block=block)
        u, v = oracle.quantize(q, tpl), oracle.quantize(q, st)
        first = -(nt - 1)
        c = oracle.xcorr_bf(u, v, 0 - first, ns - nt - first)
        m, f, n = oracle.argmax(c)
        assert got == (m, f + 5, n), (trial, got, (m, f, n))
    meta, _ = golden
    g5 = meta["configs"]["c5_small"]
    t5, s5, off, sn2 = W.c5(stream=g5["stream"], template=g5["template"], offset=g5["offset"])
    for case in g5["cases"]:
        qa, qb = _q(qx, case["qx"]), _q(qx, case["qy"])
        assert qx.template_search(t5, s5, qa, qb, block=8191) == (case["peak"], case["lags"][0], len(case["lags"]))


def test_template_search_tensor_core_blocks(qx, oracle, golden):
    """Default blocks: 2048-lag tiles on the tcgen05 window path in
    shared-template mode (template built once per SM; stream rows of
    block + nt - 1 samples, including rows whose length is not a multiple of
    4), equal to the oracle and to the NTT path."""
    from paper_2509_19974_b200 import workloads as W

    rng = np.random.default_rng(22)
    for trial, nt in enumerate((4096, 64, 2052, 1000, 4)):
        ns = int(rng.integers(nt + 3 * 2048, nt + 9 * 2048))
        st = rng.laplace(size=ns).astype(np.float32)
        off = int(rng.integers(0, ns - nt + 1))
        tpl = st[off:off + nt].copy()
        st = st + rng.normal(0, 0.7, ns).astype(np.float32)
        q = [qx.sign(), qx.uniform(1, 0.8), qx.uniform(7, 0.3)][trial % 3]
        got = qx.template_search(tpl, st, q, q, stream_start=11)
        assert got == qx.template_search(tpl, st, q, q, stream_start=11, path="ntt"), trial
        u, v = oracle.quantize(q, tpl), oracle.quantize(q, st)
        first = -(nt - 1)
        c = oracle.xcorr_bf(u, v, 0 - first, ns - nt - first)
        m, f, n = oracle.argmax(c)
        assert got == (m, f + 11, n), (trial, got, (m, f, n))
    meta, _ = golden
    g5 = meta["configs"]["c5_small"]
    t5, s5, off, sn2 = W.c5(stream=g5["stream"], template=g5["template"], offset=g5["offset"])
    for case in g5["cases"]:
        qa, qb = _q(qx, case["qx"]), _q(qx, case["qy"])
        assert qx.template_search(t5, s5, qa, qb) == (case["peak"], case["lags"][0], len(case["lags"]))


def test_template_search_fp4_mode(qx, oracle):
    """Template search on the fp4 (e2m1, kind::mxf4) tensor-core mode: codes
    |c| <= 4 (sign, uniform k = 1..4), 8192-lag blocks; the profile proves the
    fp4 kernel ran, and the summary equals the oracle's and the i8 mode's
    (option tc_f4=0) on the same inputs, including a remainder block, short
    templates and a k=4 worst case near the f32-exact bound."""
    from paper_2509_19974_b200 import _native

    rng = np.random.default_rng(23)
    cases = [(4096, qx.sign()), (4096, qx.uniform(1, 0.8)), (2052, qx.uniform(4, 0.4)), (1000, qx.uniform(2, 0.5)),
             (64, qx.uniform(3, 0.3)), (4, qx.sign()), (4096, qx.uniform(4, 0.05))]
    for trial, (nt, q) in enumerate(cases):
        ns = nt - 1 + 8192 * int(rng.integers(2, 5)) + int(rng.integers(0, 8192))
        st = rng.laplace(size=ns).astype(np.float32)
        off = int(rng.integers(0, ns - nt + 1))
        tpl = st[off:off + nt].copy()
        st = st + rng.normal(0, 0.7, ns).astype(np.float32)
        with _native.profile(timed=False) as prof:
            got = qx.template_search(tpl, st, q, q, stream_start=3)
        assert prof.result.get("direct_f4", (0, 0))[0] >= 1, (trial, prof.result)
        with _native.option("tc_f4", 0), _native.profile(timed=False) as prof:
            i8 = qx.template_search(tpl, st, q, q, stream_start=3)
        assert "direct_f4" not in prof.result or prof.result["direct_f4"][0] == 0, prof.result
        u, v = oracle.quantize(q, tpl), oracle.quantize(q, st)
        first = -(nt - 1)
        m, f, n = oracle.argmax(oracle.xcorr_bf(u, v, 0 - first, ns - nt - first))
        assert got == i8 == (m, f + 3, n), (trial, got, i8, (m, f, n))


def test_template_search_random_modes_and_errors(qx, oracle, monkeypatch):
    """Randomised template searches across every mode the default picks
    (fp4 for k <= 4, int8 for k > 4, NTT for templates the window path does not
    take) and explicit block sizes, against the oracle; NaN in the stream and
    an all-zero template raise the reference's exceptions."""
    from paper_2509_19974_b200.errors import DegenerateQuantization

    rng = np.random.default_rng(26)
    quants = [qx.sign(), qx.uniform(1, 0.6), qx.uniform(3, 0.4), qx.uniform(4, 0.2), qx.uniform(7, 0.3),
              qx.custom([-0.5, 0.2])]
    for trial in range(14):
        nt = int(rng.choice([4, 12, 100, 512, 1023, 2048, 4096, 4100]))
        ns = nt + int(rng.integers(0, 60000))
        st = rng.laplace(size=ns).astype(np.float32)
        off = int(rng.integers(0, ns - nt + 1))
        tpl = st[off:off + nt].copy()
        st = st + rng.normal(0, 0.6, ns).astype(np.float32)
        qa, qb = quants[int(rng.integers(len(quants)))], quants[int(rng.integers(len(quants)))]
        if (qa.k == 1) != (qb.k == 1) or (qa.kind == "custom") != (qb.kind == "custom"):
            qb = qa
        block = None if trial % 3 else int(rng.integers(1, 20000))
        start = int(rng.integers(-50, 50))
        got = qx.template_search(tpl, st, qa, qb, stream_start=start, block=block)
        u, v = oracle.quantize(qa, tpl), oracle.quantize(qb, st)
        if not u.any() or not v.any():
            continue
        m, f, n = oracle.argmax(oracle.xcorr_bf(u, v, nt - 1, ns - 1))
        assert got == (m, f + start, n), (trial, nt, ns, qa, qb, block, got, (m, f + start, n))
    st = rng.laplace(size=20000).astype(np.float32)
    tpl = st[500:500 + 1024].copy()
    bad = st.copy()
    bad[12345] = np.nan
    with pytest.raises(ValueError):
        qx.template_search(tpl, bad, qx.sign(), qx.sign())
    with pytest.raises(DegenerateQuantization):
        qx.template_search(np.zeros(1024, np.float32), st, qx.sign(), qx.sign())


def test_sharded_paths_over_nccl(qx):
    """The multi-GPU entry points on a real NCCL process group (one rank on
    this GPU; the 2-rank protocol itself is gloo-tested on the CPU and on
    this GPU in test_multigpu_gpu.py): qx_template_search_nccl (via
    parallel.template_search_sharded) equals the single-call template search;
    qx_summary_reduce_nccl keeps a summary; qx_estimate_batch_nccl gathers
    the records of estimate_batch."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2509_19974_b200 import _native as N
    from paper_2509_19974_b200 import parallel as PL

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(25)
        st = rng.laplace(size=60000).astype(np.float32)
        tpl = st[31337:31337 + 1024].copy()
        st = st + rng.normal(0, 0.8, st.size).astype(np.float32)
        q = qx.sign()
        with N.profile(timed=False) as prof:
            got = PL.template_search_sharded(torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda(), q, q,
                                             stream_start=-5)
        assert got == qx.template_search(tpl, st, q, q, stream_start=-5) and got[1] == 31337 - 5
        assert dist.get_backend() == "nccl" and prof.launches >= 2
        s = torch.tensor([17, -3, 2, 0, 1, 0, 0, 0], dtype=torch.int64, device="cuda")
        assert PL.reduce_summary(s).tolist() == [17, -3, 2, 0, 1, 0, 0, 0]
        xs = torch.from_numpy(rng.standard_normal((8, 4096)).astype(np.float32)).cuda()
        ys = torch.roll(xs, 100, dims=1) + 0.1
        qu = qx.uniform(7, 0.4)
        mine, allr = PL.estimate_batch_sharded(xs, ys, qu, qu, lag_lo=-512, lag_hi=512)
        want = qx.estimate_batch(xs, ys, qu, qu, lag_lo=-512, lag_hi=512).raw
        assert torch.equal(mine.raw, want) and torch.equal(allr, want)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("f4", [0, 1])
def test_template_blocks_every_block(qx, oracle, f4):
    """Every block summary of the shared-template window modes (i8 pitch 32,
    fp4 pitch 64) against the oracle, for templates whose length leaves the
    shifted copies past the pitch-16 K (nt = 4, 8, 40, 1000, 2052: the copies
    need K >= nt + pitch - 1)."""
    import torch

    from paper_2509_19974_b200 import _native as N

    with N.option("tc_f4", f4):
        _every_block_checks(qx, oracle, torch, f4)


def _every_block_checks(qx, oracle, torch, f4):
    block = 4096 if f4 == 0 else 8192
    for seed, (nt, q) in enumerate([(4, qx.sign()), (8, qx.sign()), (40, qx.uniform(1, 0.8)),
                                    (1000, qx.sign()), (2052, qx.uniform(1, 0.8))]):
        rng = np.random.default_rng(seed)
        ns = nt - 1 + block * 3 + 17
        st = rng.laplace(size=ns).astype(np.float32)
        tpl = st[100:100 + nt].copy()
        st = st + rng.normal(0, 0.7, ns).astype(np.float32)
        x, y = torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda()
        nfull = (ns - nt + 1) // block
        xr, yr = x.as_strided((nfull, nt), (0, 1)), y.as_strided((nfull, block + nt - 1), (block, 1))
        r = qx.estimate_batch(xr, yr, q, q, lag_lo=0, lag_hi=block - 1).numpy()
        u = oracle.quantize(q, tpl)
        for b in range(nfull):
            v = oracle.quantize(q, st[b * block:b * block + block + nt - 1])
            want = oracle.argmax(oracle.xcorr_bf(u, v, nt - 1, nt - 1 + block - 1))
            assert (int(r["value"][b]), int(r["lag"][b]), int(r["ties"][b])) == want, (nt, b, f4)


def test_large_transform_path(qx, oracle):
    """P > 2^19 (outer radix-2^m pass around 2^19 sub-transforms, config 4's
    path): full correlograms and windowed peaks equal the oracle's KS."""
    import torch

    from paper_2509_19974_b200.intxcorr import xcorr_full_device

    rng = np.random.default_rng(33)
    for nx, ny, q in [((1 << 19) + 5, (1 << 18) + 77, qx.uniform(7, 0.4)),
                      ((1 << 20) + 11, (1 << 20) - 3, qx.sign())]:
        s = rng.laplace(size=max(nx, 1000 + ny)).astype(np.float32)
        x = s[:nx].copy()
        y = s[1000:1000 + ny] + rng.normal(0, 0.7, ny).astype(np.float32)
        u, v = oracle.quantize(q, x), oracle.quantize(q, y)
        want = oracle.xcorr_ks(u, v, q.k, q.k)
        vals, st = xcorr_full_device(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), q, q)
        assert np.array_equal(vals[0].cpu().numpy(), want)
        m, f, n = oracle.argmax(want)
        res = qx.estimate_batch(x[None], y[None], q, q).numpy()
        assert (res["value"][0], res["lag"][0], res["ties"][0]) == (m, f - (nx - 1), n)
        assert res["lag"][0] == -1000


def test_large_transform_path_in_chunks(qx, oracle):
    """P > 2^19 with more pairs than one launch group (chunk_pairs = 1 and 2
    over a batch of 3): every group's inner passes must read that group's
    outer-pass rows, and the records must not depend on the grouping."""
    import torch

    from paper_2509_19974_b200 import _native

    rng = np.random.default_rng(34)
    nx, ny, q = (1 << 19) + 9, (1 << 19) - 100, qx.uniform(3, 0.5)
    x = rng.laplace(size=(3, nx)).astype(np.float32)
    y = np.stack([np.roll(x[b], 100 * (b + 1))[:ny] for b in range(3)]) + rng.normal(0, 0.5, (3, ny)).astype(np.float32)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    whole = qx.estimate_batch(xd, yd, q, q, path="ntt").numpy()
    for b in range(3):
        u, v = oracle.quantize(q, x[b]), oracle.quantize(q, y[b])
        m, f, n = oracle.argmax(oracle.xcorr_ks(u, v, q.k, q.k))
        assert (whole["value"][b], whole["lag"][b], whole["ties"][b]) == (m, f - (nx - 1), n), b
    for chunk in (1, 2):
        with _native.option("chunk_pairs", chunk):
            part = qx.estimate_batch(xd, yd, q, q, path="ntt").numpy()
        assert np.array_equal(part, whole), chunk


def test_large_transform_dtypes_quantizers_and_layouts(qx):
    """Large-P path over float32/float64 rows, the three quantiser modes (k = 1,
    uniform, custom thresholds), operands longer than P/2 (no zero-upper
    specialisation), padded row strides and a row shared by every pair
    (ld = 0), on impulse trains with the sparse sum as the expected answer."""
    import torch

    rng = np.random.default_rng(13)
    quants = [qx.uniform(1, 1.0), qx.uniform(3, 1.0), qx.custom([-2.5, -1.5, -0.5, 0.5, 1.5, 2.5])]
    for dt in (np.float32, np.float64):
        for nx, ny in [((1 << 19) + 3, (1 << 19) - 50), (700_000, 300_000), (300_001, 745_000)]:
            B, pad = 3, 17
            xb = np.zeros((B, nx + pad), dt)
            yb = np.zeros((B, ny + pad), dt)
            for r in range(B):
                xb[r, rng.choice(nx, 5 + r, replace=False)] = rng.choice([-3.0, -1.0, 1.0, 2.0], 5 + r)
                yb[r, rng.choice(ny, 4 + r, replace=False)] = rng.choice([-2.0, -1.0, 1.0, 3.0], 4 + r)
            xb[:, nx:] = 9.0  # the row padding must never be read
            yb[:, ny:] = 9.0
            xd, yd = torch.from_numpy(xb).cuda()[:, :nx], torch.from_numpy(yb).cuda()[:, :ny]  # ld = n + pad
            for q in quants:
                k = q.k
                res = qx.estimate_batch(xd, yd, q, q, path="ntt").numpy()
                lo, hi = -(nx - 1) + 1000, ny - 1 - 7
                win = qx.estimate_batch(xd, yd, q, q, path="ntt", lag_lo=lo, lag_hi=hi).numpy()
                for r in range(B):
                    cx, cy = np.clip(xb[r, :nx], -k, k), np.clip(yb[r, :ny], -k, k)
                    assert (int(res["value"][r]), int(res["lag"][r]), int(res["ties"][r])) == \
                        _sparse_peak(cx, cy, -(nx - 1), ny - 1), (dt, nx, ny, k, r)
                    assert (int(win["value"][r]), int(win["lag"][r]), int(win["ties"][r])) == \
                        _sparse_peak(cx, cy, lo, hi), (dt, nx, ny, k, r, "window")
            # one x row for every pair
            q = quants[1]
            shared = qx.estimate_batch(xd[:1].expand(B, nx), yd, q, q, path="ntt").numpy()
            for r in range(B):
                cx, cy = np.clip(xb[0, :nx], -3, 3), np.clip(yb[r, :ny], -3, 3)
                assert (int(shared["value"][r]), int(shared["lag"][r]), int(shared["ties"][r])) == \
                    _sparse_peak(cx, cy, -(nx - 1), ny - 1), (dt, nx, ny, r, "shared row")


def test_large_transform_statuses_in_a_batch(qx):
    """Per-pair statuses on the large-P path: an all-zero row (degenerate) and a
    NaN row beside healthy pairs keep their own records."""
    import torch

    rng = np.random.default_rng(14)
    n = (1 << 19) + 40
    x = np.zeros((4, n), np.float32)
    y = np.zeros((4, n), np.float32)
    for r in range(4):
        x[r, rng.choice(n, 6, replace=False)] = 1.0
        y[r, rng.choice(n, 6, replace=False)] = 1.0
    x[1] = 0.0          # quantises to all zeros
    y[2, 12345] = np.nan
    q = qx.uniform(1, 1.0)
    res = qx.estimate_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), q, q, path="ntt").numpy()
    assert res["status"][1] == 2 and res["status"][2] == 9, res["status"]
    for r in (0, 3):
        assert res["status"][r] == 0
        assert (int(res["value"][r]), int(res["lag"][r]), int(res["ties"][r])) == \
            _sparse_peak(x[r], y[r], -(n - 1), n - 1), r


def test_c4_full_size(qx, oracle):
    """BASELINE config 4 at full size (2^24-sample Laplacian pair, 0 dB, 4-bit):
    the GPU finds the planted delay and agrees with the oracle's exact
    correlation at a sample of lags (int64 dot products on the CPU)."""
    import torch

    from paper_2509_19974_b200 import workloads as W

    x, y, lag = W.c4()
    q = W.bit_quantizer(4, W.C4_SIGMA)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    res = qx.estimate_batch(xd, yd, q, q).numpy()[0]
    assert res["status"] == 0 and res["lag"] == lag == -731_205 and res["ties"] == 1
    u, v = oracle.quantize(q, x), oracle.quantize(q, y)
    assert res["sumsq_x"] == oracle.sumsq(u) and res["sumsq_y"] == oracle.sumsq(v)
    n = len(u)
    t_peak = lag + n - 1
    assert oracle.xcorr_bf(u, v, t_peak, t_peak)[0] == res["value"]


def test_calls_on_different_streams_are_ordered(qx):
    """Entry points that share a context's scratch on different streams are
    ordered (an async estimate_batch on one stream followed by a
    call on another stream must not race on the scratch and counters)."""
    import torch

    from paper_2509_19974_b200 import workloads as W

    xs, ys, _ = W.c2(pairs=16, n=1 << 16, seed=41)
    xs2, ys2, _ = W.c2(pairs=16, n=1 << 16, seed=42)
    q = W.bit_quantizer(4, W.C2_SIGMA)
    x1, y1 = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    x2, y2 = torch.from_numpy(xs2).cuda(), torch.from_numpy(ys2).cuda()
    want1 = qx.estimate_batch(x1, y1, q, q).raw.clone()
    want2 = qx.estimate_batch(x2, y2, q, q).raw.clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(4):
        with torch.cuda.stream(s1):
            r1 = qx.estimate_batch(x1, y1, q, q)
        with torch.cuda.stream(s2):
            r2 = qx.estimate_batch(x2, y2, q, q)
        with torch.cuda.stream(s1):
            r3 = qx.estimate_batch(x1, y1, q, q, path="ntt")
        h = qx.estimate_batch_host(xs2, ys2, q, q)  # the context's host stream
        torch.cuda.synchronize()
        assert torch.equal(r1.raw, want1) and torch.equal(r2.raw, want2) and torch.equal(r3.raw, want1)
        assert np.array_equal(h, want2.cpu().numpy().view(h.dtype).reshape(-1))
    assert torch.cuda.current_device() == 0


def test_estimate_plan_matches_estimate_batch(qx, oracle):
    """EstimatePlan (qx_plan_create / qx_plan_run) returns estimate_batch's
    records on every path, for new rows each call, and re-derives its
    scratch pointers after another call regrew the context's arenas."""
    import torch

    rng = np.random.default_rng(77)
    cases = [  # (B, nx, ny, quantiser, window, expected path)
        (1, 16384, 16384, qx.sign(), None, "popc"),
        (3, 3000, 2500, qx.sign(), None, "popc"),
        (4, 4096, 4096, qx.uniform(1, 0.5), (-512, 512), "direct"),
        (2, 20000, 30000, qx.uniform(7, 0.3), None, "ntt"),
    ]
    for B, nx, ny, q, win, want in cases:
        lo, hi = win if win else (None, None)
        x0 = torch.from_numpy(rng.standard_normal((B, nx)).astype(np.float32)).cuda()
        y0 = torch.from_numpy(rng.standard_normal((B, ny)).astype(np.float32)).cuda()
        plan = qx.EstimatePlan(x0, y0, q, q, lag_lo=lo, lag_hi=hi)
        assert plan.path == want, (plan.path, want)
        for it in range(3):
            x = torch.from_numpy(rng.standard_normal((B, nx)).astype(np.float32)).cuda()
            y = torch.from_numpy(rng.standard_normal((B, ny)).astype(np.float32)).cuda()
            if it == 1:  # regrow the context scratch in between
                big = torch.zeros((64, 1 << 18), dtype=torch.float32, device="cuda")
                qx.estimate_batch(big + 1, big + 1, qx.uniform(7, 0.3), qx.uniform(7, 0.3))
            a = plan(x, y).numpy()
            b = qx.estimate_batch(x, y, q, q, lag_lo=lo, lag_hi=hi).numpy()
            assert np.array_equal(a, b), (B, nx, ny, it)
            # the same rows from host memory (qx_plan_run_host), pageable and pinned
            xh, yh = x.cpu().numpy(), y.cpu().numpy()
            assert np.array_equal(plan.run_host(xh, yh), b), (B, nx, ny, it, "host")
            # pinned rows: read in place over PCIe (zero-copy, the default for small rows), and staged
            xp, yp = x.cpu().pin_memory(), y.cpu().pin_memory()
            assert np.array_equal(plan.run_host(xp.numpy(), yp.numpy()), b), (B, nx, ny, it, "pinned")
            from paper_2509_19974_b200 import _native

            with _native.option("zero_copy", 0):
                assert np.array_equal(plan.run_host(xp.numpy(), yp.numpy()), b), (B, nx, ny, it, "pinned, staged")
        with pytest.raises(ValueError):
            plan(x[:, :-1] if nx > 1 else x, y)
