"""C1 popc kernel phase times (QX_POPC_TIMING=1 makes the correlation kernel
print them); `warm` runs 2000 back-to-back calls first (clocks up)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native as N, workloads as W

x, y = W.c1(0)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for i in range(3):
    if "warm" in sys.argv:
        for _ in range(2000):
            P.estimate_batch(xd, yd, P.sign(), P.sign())
    with N.option("popc_timing", 1):
        r = P.estimate_batch(xd, yd, P.sign(), P.sign())
        torch.cuda.synchronize()
    print("----", r.numpy())
