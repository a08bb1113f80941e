"""Would slicing one NTT batch over the compute lanes pay?  The same work two
ways: 64 pairs in one estimate_batch (serial kernels) against the sweep entry
point running 4 (or 2) identical quantiser pairs over 16 (32) of the pairs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import workloads as W

xs, ys, lag = W.c2()
xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
q = W.bit_quantizer(4, W.C2_SIGMA)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


print("64 pairs, one call      :", timed(lambda: P.estimate_batch(xd, yd, q, q, path="ntt")))
print("4 lanes x 16 pairs      :", timed(lambda: P.estimate_sweep(xd[:16], yd[:16], [(q, q)] * 4, path="ntt")))
print("2 lanes x 32 pairs      :", timed(lambda: P.estimate_sweep(xd[:32], yd[:32], [(q, q)] * 2, path="ntt")))
