"""A/B of the C3 window kernel: median ms of estimate_batch on all 65,536 pairs
(b = argv[1]) for the library in QX_NATIVE_LIB (or the in-tree one)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import workloads as W

b = int(sys.argv[1]) if len(sys.argv) > 1 else 4
xs, ys, lag = W.c3()
xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
q = W.bit_quantizer(b, W.C3_SIGMA)
for _ in range(3):
    r = P.estimate_batch(xd, yd, q, q, lag_lo=-512, lag_hi=512)
torch.cuda.synchronize()
assert np.array_equal(r.lag.cpu().numpy(), lag)
ts = []
for _ in range(9):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    P.estimate_batch(xd, yd, q, q, lag_lo=-512, lag_hi=512)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(os.environ.get("QX_NATIVE_LIB", "in-tree"), f"b={b}", f"median {np.median(ts):.3f} ms", f"min {min(ts):.3f}")
