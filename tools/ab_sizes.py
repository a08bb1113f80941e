"""Per-kernel device time of the NTT passes at several transform sizes with the
same number of points per launch (pairs * P = 2^25): us per butterfly-stage
unit (2^24 butterflies), to compare CTA-residency regimes of the passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native, workloads as W

q = W.bit_quantizer(4, 1.0)
for ln in (15, 16, 17, 18):
    n = 1 << ln
    pairs = (1 << 24) >> ln
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(pairs, n, device="cuda", generator=g)
    y = torch.randn(pairs, n, device="cuda", generator=g)
    for _ in range(3):
        P.estimate_batch(x, y, q, q, path="ntt")
    torch.cuda.synchronize()
    with _native.profile(timed=True) as kp:
        for _ in range(5):
            P.estimate_batch(x, y, q, q, path="ntt")
        torch.cuda.synchronize()
    lp = ln + 1
    l1, l2 = (lp + 1) // 2, lp // 2
    units = {"ntt_pass1": 2 * l1, "ntt_pass2": 3 * l2, "ntt_pass3": l1}
    print(f"P=2^{lp} l1={l1} l2={l2} pairs={pairs}",
          {k: (round(m / 5 * 1e3, 1), round(m / 5 * 1e3 / units[k], 2)) for k, (c, m) in kp.result.items() if k in units})
