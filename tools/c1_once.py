"""A few C1 calls (one 2^14 float64 pair, sign, full lags) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import workloads as W

x, y = W.c1(0)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    r = P.estimate_batch(xd, yd, P.sign(), P.sign())
torch.cuda.synchronize()
print(r.numpy())
