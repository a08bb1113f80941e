"""C2 end-to-end (qx_estimate_sweep_host) under the sweep schedule knobs,
beside the plain pinned-H2D bound of the same bytes.  One process; the knobs
are context options (qx_context_set_option), set before each series; explicit
chunk plans (QX_SWEEP_PLAN) are read at context creation only and need one
process per plan (PLANS=... runs them through the environment of a fresh
interpreter).  Usage: python tools/e2e_knobs.py [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19974_b200 as P  # noqa: E402
from paper_2509_19974_b200 import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
xs, ys, lag = W.c2()
qs = [W.bit_quantizer(b, W.C2_SIGMA) for b in (1, 2, 4, 8)]
sweep = [(q, q) for q in qs]
hx, hy = torch.from_numpy(xs).pin_memory(), torch.from_numpy(ys).pin_memory()
hxn, hyn = hx.numpy(), hy.numpy()
est = len(qs) * xs.shape[0]

dx, dy = torch.empty_like(hx, device="cuda"), torch.empty_like(hy, device="cuda")
for _ in range(2):
    dx.copy_(hx, non_blocking=True), dy.copy_(hy, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    dx.copy_(hx, non_blocking=True), dy.copy_(hy, non_blocking=True)
e1.record()
torch.cuda.synchronize()
h2d = e0.elapsed_time(e1) / reps
print(f"pinned H2D {xs.nbytes + ys.nbytes} B: {h2d:.3f} ms ({(xs.nbytes + ys.nbytes) / h2d / 1e6:.1f} GB/s)"
      f" -> bound {est / h2d * 1e3:.0f} est/s")

KNOBS = [{}, {"QX_SWEEP_TAPER": "1"}, {"QX_SWEEP_TAPER": "4"}, {"QX_SWEEP_TAPER": "8"}, {"QX_SWEEP_CHUNKS": "16"},
         {"QX_SWEEP_CHUNKS": "12"}, {"QX_SWEEP_CHUNKS": "10"}, {"QX_SWEEP_CHUNKS": "6"},
         {"QX_SWEEP_CHUNKS": "4"}, {"QX_SWEEP_LANES": "2"}, {"QX_SWEEP_EVEN": "1"}]
PLANS = os.environ.get("PLANS", "4,12,16,16,12,4;4,8,16,16,16,4;2,6,12,16,16,10,2;4,12,24,20,4;"
                       "8,16,16,16,8;4,28,28,4;4,10,16,16,10,6,2;6,12,16,16,10,4").split(";")
KNOBS += [{}]
if os.environ.get("LANES_ONLY"):
    KNOBS = [{}, {"QX_SWEEP_LANES": "5"}, {"QX_SWEEP_LANES": "6"}, {"QX_SWEEP_LANES": "8"},
             {"QX_SWEEP_LANES": "8", "QX_SWEEP_CHUNKS": "16"}, {"QX_SWEEP_LANES": "8", "QX_SWEEP_CHUNKS": "4"},
             {"QX_SWEEP_LANES": "8", "QX_SWEEP_RESTAGE": "0"}, {"QX_SWEEP_RESTAGE": "0"}, {}]
if os.environ.get("COPY_ONLY"):
    KNOBS = [{}, {"QX_SWEEP_COMPUTE": "0"}, {"QX_SWEEP_COMPUTE": "0", "QX_SWEEP_CHUNKS": "1"},
             {"QX_SWEEP_RESTAGE": "0"}, {}]
if os.environ.get("RESTAGE_ONLY"):
    KNOBS = [{}, {"QX_SWEEP_RESTAGE": "0"}, {"QX_SWEEP_RESTAGE": "0", "QX_SWEEP_CHUNKS": "1"},
             {"QX_SWEEP_RESTAGE": "0", "QX_SWEEP_CHUNKS": "2"}, {"QX_SWEEP_RESTAGE": "0", "QX_SWEEP_CHUNKS": "4"},
             {"QX_SWEEP_RESTAGE": "0", "QX_SWEEP_EVEN": "1"}, {"QX_SWEEP_RESTAGE": "0", "QX_SWEEP_CHUNKS": "16"},
             {"QX_SWEEP_RESTAGE": "0", "QX_SWEEP_LANES": "1", "QX_SWEEP_CHUNKS": "1"}, {}]
for kn in KNOBS:
    from paper_2509_19974_b200 import _native  # noqa: E402

    DEFAULT = {"QX_SWEEP_TAPER": 2, "QX_SWEEP_CHUNKS": 0, "QX_SWEEP_LANES": 0, "QX_SWEEP_EVEN": 0,
               "QX_SWEEP_RESTAGE": 1, "QX_SWEEP_COMPUTE": 1}
    for k, v in DEFAULT.items():
        _native.set_option(k[3:].lower(), int(kn.get(k, v)))
    for _ in range(2):
        P.estimate_sweep_host(hxn, hyn, sweep)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res = P.estimate_sweep_host(hxn, hyn, sweep)
        ts.append(time.perf_counter() - t0)
    for r in res:
        assert kn.get("QX_SWEEP_COMPUTE") == "0" or np.array_equal(r["lag"], lag)
    ts = np.array(ts) * 1e3
    print(f"{str(kn):55s} median {np.median(ts):.3f} ms  min {ts.min():.3f}  -> {est / np.median(ts) * 1e3:.0f} est/s"
          f"  ({h2d / np.median(ts):.2f} of H2D bound)")
