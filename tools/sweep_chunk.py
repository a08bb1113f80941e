"""Time BASELINE config 2 (all 4 bit depths) for several QX_CHUNK_PAIRS values."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native
from paper_2509_19974_b200 import workloads as W

xs, ys, lag = W.c2()
xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
qs = [W.bit_quantizer(b, W.C2_SIGMA) for b in (1, 2, 4, 8)]
for chunk in sys.argv[1:]:
    _native.set_option("chunk_pairs", int(chunk))  # the knobs are context options, not per-call environment
    for _ in range(3):
        for q in qs:
            P.estimate_batch(xd, yd, q, q)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        for q in qs:
            P.estimate_batch(xd, yd, q, q)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"chunk {chunk:>3}: {ms:.3f} ms/step  {256 / ms * 1e3:.0f} est/s", flush=True)
