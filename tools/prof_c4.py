"""Per-kernel device time of BASELINE config 4 (one 2^24 pair, b=4, P=2^25)
through the library's event profiler; also a short ncu driver (argv[1] = iters)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native, workloads as W

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
x, y, lag = W.c4()
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
q = W.bit_quantizer(4, W.C4_SIGMA)
for _ in range(iters):
    r = P.estimate_batch(xd, yd, q, q)
torch.cuda.synchronize()
assert r.numpy()["lag"][0] == lag
if os.environ.get("QX_PROF"):
    with _native.profile(timed=True) as pr:
        for _ in range(5):
            P.estimate_batch(xd, yd, q, q)
    print({k: (c // 5, round(ms / 5, 4)) for k, (c, ms) in pr.result.items()})
print("ok")
