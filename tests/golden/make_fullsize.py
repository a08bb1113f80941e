"""Full-size golden records for BASELINE configs 2-5 (test infrastructure).

Run in the development container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fullsize.py [c2 c3 c4 c5]

The reference's own Python Kronecker substitution takes ~1 h for one config-4
pair, so these records come from the C oracle
(oracle/qx_oracle.c: float64 quantise, KS with GMP mpn_mul, argmax), which is
pinned against vectors the reference itself produced (tests/golden/golden.*,
tests/test_oracle_golden.py).  This script re-checks that pin on the overlap:
the first 3 C2 pairs x 4 depths and the first 256 C3 pairs x 2 depths must
reproduce golden.json's reference digests, and a few C5 blocks are compared
with the reference's own xcorr_int_bf when /root/reference is present.

Digest format (the reference's acceptance pattern,
pkg/tests/test_acceptance.py:131-134): sha256 of the int64 little-endian
bytes of the correlogram values; [:16] hex for per-pair digests.

Records (value, lag, ties) use the reference lag convention
(signals.py:100-105): lag = first_lag + t.

Writes tests/golden/fullsize.npz (per-pair / per-block records) and
tests/golden/fullsize.json (aggregate digests, parameters).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402  (C oracle, pinned)

from paper_2509_19974_b200 import workloads as W  # noqa: E402  (seeded generators only)

THREADS = os.cpu_count() or 8
NPZ = os.path.join(HERE, "fullsize.npz")
JSN = os.path.join(HERE, "fullsize.json")


def sha16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()[:16]


def load():
    arrays, meta = {}, {}
    if os.path.exists(NPZ):
        with np.load(NPZ) as z:
            arrays = {k: z[k] for k in z.files}
    if os.path.exists(JSN):
        meta = json.load(open(JSN))
    return arrays, meta


def ref_golden():
    return json.load(open(os.path.join(HERE, "golden.json")))["configs"]


# ------------------------------------------------------------------- C2
C2_GOLDEN_PAIRS = 8 * W.C2_PAIRS  # bench.py's per-rank batches at up to 8 GPUs (rank r: pairs 64r..64r+63)


def make_c2(arrays, meta):
    xs, ys, lag = W.c2(pairs=C2_GOLDEN_PAIRS)
    n = xs.shape[1]
    rec = np.zeros((4, C2_GOLDEN_PAIRS, 3), np.int64)
    sumsq = np.zeros((4, C2_GOLDEN_PAIRS, 2), np.int64)
    shas = [[""] * C2_GOLDEN_PAIRS for _ in range(4)]

    def one(job):
        bi, p = job
        q = W.bit_quantizer((1, 2, 4, 8)[bi], W.C2_SIGMA)
        u, v = O.quantize(q, xs[p]), O.quantize(q, ys[p])
        c = O.xcorr_ks(u, v, int(q.k), int(q.k))
        m, f, t = O.argmax(c)
        return bi, p, (m, f - (n - 1), t), (O.sumsq(u), O.sumsq(v)), sha16(c)

    with ThreadPoolExecutor(THREADS) as ex:
        for bi, p, r, s, h in ex.map(one, [(bi, p) for bi in range(4) for p in range(C2_GOLDEN_PAIRS)]):
            rec[bi, p], sumsq[bi, p], shas[bi][p] = r, s, h
    # pin: golden.json holds the reference's own digests for pairs 0-2
    for g in ref_golden()["c2"]:
        bi, p = (1, 2, 4, 8).index(g["b"]), g["pair"]
        assert shas[bi][p] == g["sha"] and rec[bi, p, 0] == g["peak"] and rec[bi, p, 1] == g["lags"][0], g
        assert rec[bi, p, 2] == len(g["lags"]) and tuple(sumsq[bi, p]) == (g["sumsq_u"], g["sumsq_v"])
    arrays["c2_rec"], arrays["c2_sumsq"] = rec, sumsq
    meta["c2"] = {"bits": [1, 2, 4, 8], "pairs": C2_GOLDEN_PAIRS, "n": n, "sha16": shas,
                  "what": "full correlograms (lags -(n-1)..n-1) of every pair and bit depth; rec[b][p] = "
                          "(peak, smallest lag, ties), sumsq = (sum u^2, sum v^2)",
                  "planted_lag_hits": int(sum((rec[bi, :, 1] == lag).sum() for bi in range(4)))}


# ------------------------------------------------------------------- C3
def make_c3(arrays, meta):
    n, half = W.C3_N, W.C3_MAXD
    t_lo = n - 1 - half
    rec = np.zeros((2, W.C3_PAIRS, 3), np.int32)
    digests = []
    hits = []
    chunk = 4096
    for bi, b in enumerate((2, 4)):
        q = W.bit_quantizer(b, W.C3_SIGMA)
        h = hashlib.sha256()
        hit = 0
        for first in range(0, W.C3_PAIRS, chunk):
            xs, ys, lag = W.c3(pairs=chunk, first=first)

            def one(p):
                u, v = O.quantize(q, xs[p]), O.quantize(q, ys[p])
                return O.xcorr_bf(u, v, t_lo, t_lo + 2 * half)

            with ThreadPoolExecutor(THREADS) as ex:
                wins = list(ex.map(one, range(chunk)))
            for p, w in enumerate(wins):
                m, f, t = O.argmax(w)
                rec[bi, first + p] = (m, f - half, t)
                h.update(np.ascontiguousarray(w, dtype=np.int64).tobytes())
            hit += int((rec[bi, first:first + chunk, 1] == lag).sum())
            if first == 0:  # pin: the reference's windowed digests for pairs 0-255
                for g in ref_golden()["c3"]:
                    if g["b"] == b:
                        p = g["pair"]
                        assert sha16(wins[p]) == g["sha"] and rec[bi, p, 0] == g["peak"], g
                        assert rec[bi, p, 1] == g["lags"][0] and rec[bi, p, 2] == len(g["lags"]), g
        digests.append(h.hexdigest())
        hits.append(hit)
        print(f"c3 b={b}: {hit}/{W.C3_PAIRS} planted, digest {digests[-1][:16]}", flush=True)
    arrays["c3_rec"] = rec
    meta["c3"] = {"bits": [2, 4], "pairs": W.C3_PAIRS, "n": n, "lag_lo": -half, "lag_hi": half,
                  "window_sha256": digests, "planted_lag_hits": hits,
                  "what": "rec[b][p] = (peak, smallest lag, ties) over lags -512..512; window_sha256[b] = sha256 "
                          "of every pair's 1025 window values (int64 LE) concatenated in pair order"}


# ------------------------------------------------------------------- C4
def make_c4(arrays, meta):
    x, y, lag = W.c4()
    n = x.size
    q = W.bit_quantizer(4, W.C4_SIGMA)
    u, v = O.quantize(q, x), O.quantize(q, y)
    t0 = time.time()
    c = O.xcorr_ks(u, v, int(q.k), int(q.k))
    dt = time.time() - t0
    m, f, t = O.argmax(c)
    # O(N) spot check of the peak lag with a direct int64 dot (independent of KS)
    d = f - (n - 1)
    direct = int(np.dot(u[max(0, -d):n - max(0, d)], v[max(0, d):n - max(0, -d)]))
    assert direct == m, (direct, m)
    meta["c4"] = {"n": n, "delay": W.C4_DELAY, "peak": int(m), "lag": int(d), "ties": int(t),
                  "planted_lag": int(lag), "sha256": hashlib.sha256(c.tobytes()).hexdigest(),
                  "sumsq": [O.sumsq(u), O.sumsq(v)], "ks_seconds": dt,
                  "what": "full correlogram (2^25 - 1 lags) of the config-4 pair at b=4: sha256 of its int64 "
                          "LE values, and its (peak, smallest lag, ties)"}
    print("c4", meta["c4"], flush=True)


# ------------------------------------------------------------------- C5
C5_BLOCK = 1 << 16   # records per 65,536 valid lags
C5_TASK = 1 << 18    # lags per oracle KS call


def c5_quantizers(b, sn2):
    from paper_2509_19974_b200 import quantize as Q

    if b == 1:
        return Q.sign(), Q.sign()
    return Q.uniform(1, 1.5 * math.sqrt(2.0)), Q.uniform(1, 1.5 * math.sqrt(2.0 + sn2))


def make_c5(arrays, meta):
    t0 = time.time()
    tpl, st, off, sn2 = W.c5()
    nt, ns = tpl.size, st.size
    nvalid = ns - nt + 1
    out = {"stream": ns, "template": nt, "offset": off, "sn2": sn2, "block": C5_BLOCK, "cases": []}
    for b in (1, 2):
        qa, qb = c5_quantizers(b, sn2)
        u = O.quantize(qa, tpl)
        v = O.quantize(qb, st)
        nblk = (nvalid + C5_BLOCK - 1) // C5_BLOCK
        rec = np.zeros((nblk, 3), np.int64)

        def one(s0):
            s1 = min(nvalid, s0 + C5_TASK)
            c = O.xcorr_ks(u, v[s0:s1 + nt - 1], int(qa.k), int(qb.k))
            return s0, c[nt - 1:nt - 1 + (s1 - s0)]  # valid lags s0 .. s1-1

        h = hashlib.sha256()
        with ThreadPoolExecutor(THREADS) as ex:
            for s0, vals in ex.map(one, range(0, nvalid, C5_TASK)):
                h.update(vals.tobytes())
                for j in range(0, vals.size, C5_BLOCK):
                    m, f, t = O.argmax(vals[j:j + C5_BLOCK])
                    rec[(s0 + j) // C5_BLOCK] = (m, s0 + j + f, t)
        best = rec[:, 0].max()
        holders = rec[rec[:, 0] == best]
        summary = (int(best), int(holders[:, 1].min()), int(holders[:, 2].sum()))
        arrays[f"c5_b{b}_blocks"] = rec
        out["cases"].append({"b": b, "qx": [qa.kind, int(qa.k), float(qa.step)],
                             "qy": [qb.kind, int(qb.k), float(qb.step)], "peak": summary[0], "lag": summary[1],
                             "ties": summary[2], "valid_sha256": h.hexdigest(),
                             "sumsq": [O.sumsq(u), O.sumsq(v)]})
        print(f"c5 b={b}: {summary} digest {h.hexdigest()[:16]} ({time.time() - t0:.0f} s)", flush=True)
        # cross-check a few blocks against the reference's own brute force
        _c5_reference_spot(tpl, st, qa, qb, rec, nt)
    out["what"] = ("valid lags 0..stream-template of estimate(x=template, y=stream): blocks[i] = (peak, smallest "
                   "lag, ties) over lags [i*65536, (i+1)*65536); valid_sha256 = sha256 of all valid-lag values "
                   "(int64 LE) in lag order")
    meta["c5"] = out


def _c5_reference_spot(tpl, st, qa, qb, rec, nt):
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        return
    sys.path.insert(0, ref)
    import qxcorr
    from qxcorr.intxcorr import xcorr_int_bf

    def rq(q):
        return qxcorr.Quantizer(kind=q.kind, k=int(q.k), step=float(q.step), thresholds=tuple(q.thresholds))

    peak_blk = int(np.argmax(rec[:, 0]))
    for i in sorted({0, 1, peak_blk, rec.shape[0] // 2, rec.shape[0] - 1}):
        s0 = i * C5_BLOCK
        s1 = min(st.size - nt + 1, s0 + C5_BLOCK)
        u = qxcorr.apply(rq(qa), qxcorr.Signal(0, tpl))
        v = qxcorr.apply(rq(qb), qxcorr.Signal(s0, st[s0:s1 + nt - 1]))
        c = xcorr_int_bf(u, v)
        vals = c.values[nt - 1:nt - 1 + (s1 - s0)]
        m = int(vals.max())
        lags = np.flatnonzero(vals == m)
        assert (m, s0 + int(lags[0]), lags.size) == tuple(int(a) for a in rec[i]), (i, m, lags[:3], rec[i])


if __name__ == "__main__":
    which = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
    arrays, meta = load()
    meta["numpy"] = np.__version__
    meta["oracle"] = "oracle/qx_oracle.c (KS + GMP mpn_mul), pinned by tests/test_oracle_golden.py"
    for name in which:
        t0 = time.time()
        globals()[f"make_{name}"](arrays, meta)
        meta.setdefault("seconds", {})[name] = round(time.time() - t0, 1)
        np.savez_compressed(NPZ, **arrays)
        with open(JSN, "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        print(name, "done in", round(time.time() - t0, 1), "s", flush=True)
