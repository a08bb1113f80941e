"""Short driver for ncu: BASELINE config 2 (64 pairs x 2^18, float32) at one
bit depth, a few iterations.  Usage: python tools/prof_c2.py [bits] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import workloads as W

b = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
xs, ys, lag = W.c2()
xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
q = W.bit_quantizer(b, W.C2_SIGMA)
for _ in range(iters):
    r = P.estimate_batch(xd, yd, q, q)
torch.cuda.synchronize()
assert np.array_equal(r.lag.cpu().numpy(), lag)
print("ok", b, iters)
