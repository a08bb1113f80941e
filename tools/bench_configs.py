"""Per-config throughput of the engine on one GPU (BASELINE configs 1-5).

Times each config's hot path with CUDA events (inputs resident in HBM, warm
tables), checks every estimate against the pinned oracle's full-size records
(tests/golden/fullsize.*, tools/fullsize_golden.py), and returns / prints
one JSON object.  C3 runs a 16384-pair slice of the 65,536-pair workload
(per-pair cost is shape-only; `c3full` runs all 65,536 pairs); C5 runs the
full 2^28-sample stream.  Roofline fractions: HBM from MEASURED_PEAKS.json
hbm_gbs; i8 tensor from the measured 8190 MACs/clk/SM (profiles/r01_tc_rate.json);
fp4 tensor (the C5 path) from the measured 16336 MACs/clk/SM (profiles/r01_tc_fp4.txt,
tools/tc_fp4.cu, M128 x N>=128 kind::mxf4).
bench.py imports run() for its `other_configs` key.
usage: python tools/bench_configs.py [c1 c1batch c2 c3 c3full c4 c5]"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import workloads as W

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import fullsize_golden as G  # noqa: E402

I8_MACS_PER_CLK_SM = 8190.0  # tools/tc_rate.cu, M128 x N128/N256
FP4_MACS_PER_CLK_SM = 16336.0  # tools/tc_fp4.cu rate probe, M128 x N128/N256 kind::mxf4


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm = json.load(open(path)).get("hbm_gbs", 6550.4) if os.path.exists(path) else 6550.4
    props = torch.cuda.get_device_properties(0)
    clk = 1.965e9
    i8 = I8_MACS_PER_CLK_SM * props.multi_processor_count * clk
    fp4 = FP4_MACS_PER_CLK_SM * props.multi_processor_count * clk
    return hbm, i8, fp4


def run(which) -> dict:
    res = {}
    hbm, i8, fp4 = _peaks()
    if "c1" in which:
        x, y = W.c1(0)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        plan = P.EstimatePlan(xd, yd, P.sign(), P.sign())
        ms, r = timed(lambda: plan(xd, yd), reps=200, warm=20)
        ms_eb, r2 = timed(lambda: P.estimate_batch(xd, yd, P.sign(), P.sign()), reps=200, warm=20)
        r, r2 = r.numpy()[0], r2.numpy()[0]
        assert r == r2
        G.check_c1(int(r["lag"]), int(r["value"]))
        res["c1"] = {"ms_per_estimate": ms, "ms_per_estimate_estimate_batch": ms_eb, "lag": int(r["lag"]),
                     "peak": int(r["value"]),
                     "note": "single pair, back-to-back calls incl. the Python call (EstimatePlan = qx_plan_run; "
                             "estimate_batch rebuilds the call each time)",
                     "path": "popc: bit planes kernel + PDL correlation kernel (lane = lag, overlap-exact)"}
    if "c1batch" in which:
        x, y = W.c1(0)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        xb, yb = xd.expand(1024, -1), yd.expand(1024, -1)
        ms, r = timed(lambda: P.estimate_batch(xb, yb, P.sign(), P.sign()), reps=10)
        rr = r.numpy()
        G.check_c1(int(rr["lag"][0]), int(rr["value"][0]))
        assert (G.records(rr) == G.records(rr[:1])).all()
        res["c1_batch1024"] = {"ms": ms, "estimates_per_s": 1024 / ms * 1e3}
    if "c2" in which:
        xs, ys, lag = W.c2()
        xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
        for b in (1, 2, 4, 8):
            q = W.bit_quantizer(b, W.C2_SIGMA)
            ms, r = timed(lambda: P.estimate_batch(xd, yd, q, q))
            G.check_c2((1, 2, 4, 8).index(b), 0, r.numpy())
            res[f"c2_b{b}"] = {"ms": ms, "estimates_per_s": 64 / ms * 1e3,
                               "gsamples_per_s": 64 * 2 * W.C2_N / ms / 1e6}
    if "c3" in which or "c3full" in which:
        npairs = W.C3_PAIRS if "c3full" in which else 16384
        xs, ys, lag = W.c3(pairs=npairs)
        xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
        del xs, ys
        for b in (2, 4):
            q = W.bit_quantizer(b, W.C3_SIGMA)
            ms, r = timed(lambda: P.estimate_batch(xd, yd, q, q, lag_lo=-512, lag_hi=512), reps=3)
            ok = float(np.mean(r.numpy()["lag"] == lag))
            G.check_c3((2, 4).index(b), 0, r.numpy())
            res[f"c3_b{b}"] = {"pairs": npairs, "ms": ms, "estimates_per_s": npairs / ms * 1e3,
                               "gsamples_per_s": npairs * 2 * W.C3_N / ms / 1e6, "frac_correct_lag": ok,
                               "hbm_frac": npairs * 2 * W.C3_N * 4 / (ms / 1e3) / 1e9 / hbm,
                               "path": "tcgen05 kind::i8 window (M=64 tile + 1 CUDA-core lag)"}
        del xd, yd
    if "c4" in which:
        x, y, lag = W.c4()
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        q = W.bit_quantizer(4, W.C4_SIGMA)
        ms, r = timed(lambda: P.estimate_batch(xd, yd, q, q), reps=3)
        G.check_c4(r.numpy()[0])
        res["c4"] = {"ms": ms, "gsamples_per_s": 2 * W.C4_N / ms / 1e6,
                     "path": "ntt P=2^25 (outer 2^6 x inner 2^19)"}
        del xd, yd
    if "c5" in which:
        t0 = time.time()
        tpl, st, off, sn2 = W.c5()
        gen_s = time.time() - t0
        td, sd = torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda()
        macs = len(tpl) * (len(st) - len(tpl) + 1)
        for b in (1, 2):
            if b == 1:
                qa = qb = P.sign()
            else:
                qa, qb = P.uniform(1, 1.5 * math.sqrt(2.0)), P.uniform(1, 1.5 * math.sqrt(2.0 + sn2))
            ms, r = timed(lambda: P.template_search(td, sd, qa, qb), reps=10, warm=2)
            G.check_c5(b, r)
            res[f"c5_b{b}"] = {"ms": ms, "gsamples_per_s": (len(st) + len(tpl)) / ms / 1e6, "peak": r[0],
                               "lag": r[1], "fp4_tensor_frac": macs / (ms / 1e3) / fp4,
                               "hbm_frac": len(st) * 4 / (ms / 1e3) / 1e9 / hbm,
                               "path": "tcgen05 kind::mxf4 window (e2m1 codes, exact f32 sums), shared template "
                                       "(N=64 copies, SW32 Hankel), 8192-lag blocks, one C-ABI call"}
        res["c5_generation_s"] = gen_s
        del td, sd
    torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    print(json.dumps(run(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])))
