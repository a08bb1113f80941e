"""Short driver for ncu: BASELINE config 3 slice (argv[1] pairs, default 4096), b = argv[2] (default 4), window -512..512."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
xs, ys, lag = W.c3(pairs=n)
xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
q = W.bit_quantizer(int(sys.argv[2]) if len(sys.argv) > 2 else 4, W.C3_SIGMA)
for _ in range(3):
    r = P.estimate_batch(xd, yd, q, q, lag_lo=-512, lag_hi=512)
torch.cuda.synchronize()
assert np.array_equal(r.lag.cpu().numpy(), lag)
print("ok")
if os.environ.get("QX_PROF"):
    from paper_2509_19974_b200 import _native
    torch.cuda.synchronize()
    with _native.profile(timed=True) as pr:
        for _ in range(5):
            P.estimate_batch(xd, yd, q, q, lag_lo=-512, lag_hi=512)
    print({k: (c, ms / 5) for k, (c, ms) in pr.result.items()})
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        P.estimate_batch(xd, yd, q, q, lag_lo=-512, lag_hi=512)
    e.record()
    torch.cuda.synchronize()
    print("call ms", s.elapsed_time(e) / 5)
