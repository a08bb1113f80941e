"""A/B of the C2 NTT passes: per-kernel device ms per bit-depth step (serial
estimate_batch calls, event-timed launches) and the lane-sweep step time, for
the library in QX_NATIVE_LIB (or the in-tree one)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native, workloads as W

xs, ys, lag = W.c2()
xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
qs = [W.bit_quantizer(b, W.C2_SIGMA) for b in (1, 2, 4, 8)]
sw = [(q, q) for q in qs]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    res = P.estimate_sweep(xd, yd, sw)
torch.cuda.synchronize()
if not os.environ.get("QX_AB_NOCHECK"):
    for r in res:
        assert np.array_equal(r.lag.cpu().numpy(), lag)
ts = []
for _ in range(15):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    P.estimate_sweep(xd, yd, sw)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
with _native.profile(timed=True) as kp:
    for _ in range(5):
        flush.zero_()
        for q in qs:
            P.estimate_batch(xd, yd, q, q)
    torch.cuda.synchronize()
k = {n: round(m / 5, 4) for n, (c, m) in kp.result.items()}
print(os.environ.get("QX_NATIVE_LIB", "in-tree"), f"step median {np.median(ts):.4f} ms min {min(ts):.4f}", k)
