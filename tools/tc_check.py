"""Quick check of the tcgen05 window path against the oracle (small shapes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch

import oracle as O
import paper_2509_19974_b200 as P

rng = np.random.default_rng(5)
bad = 0
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    B = int(rng.integers(1, 300))
    nx = int(rng.integers(1, 4500))
    ny = int(rng.integers(1, 5000))
    q = [P.sign(), P.uniform(7, 0.3), P.uniform(1, 0.8), P.uniform(127, 0.02)][trial % 4]
    x = rng.standard_normal((B, nx)).astype(np.float32)
    y = rng.standard_normal((B, ny)).astype(np.float32)
    nout = nx + ny - 1
    t_lo = int(rng.integers(0, nout))
    special = [1, 15, 16, 17, 1024, 1025, 1040, 1041, 2048, 2049, 2064, 2065, 4096, 4097, 4112]
    w = special[trial % len(special)] if trial % 2 else int(rng.integers(1, 4113))
    if trial % 3 == 0:  # aligned window start (fast builder path needs L0 % 4 == 0)
        t_lo = max(0, (nx - 1) - 4 * int(rng.integers(0, 256)))
    t_hi = min(nout - 1, t_lo + w - 1)
    first = -(nx - 1)
    r = P.estimate_batch(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), q, q, lag_lo=first + t_lo,
                         lag_hi=first + t_hi, path="direct").numpy()
    for b in range(B):
        u, v = O.quantize(q, x[b]), O.quantize(q, y[b])
        c = O.xcorr_bf(u, v, t_lo, t_hi)
        m, f, n = O.argmax(c)
        got = (int(r["value"][b]), int(r["lag"][b]), int(r["ties"][b]))
        if got != (m, first + t_lo + f, n) or r["sumsq_x"][b] != O.sumsq(u) or r["sumsq_y"][b] != O.sumsq(v):
            bad += 1
            if bad < 5:
                print("MISMATCH", trial, b, nx, ny, t_lo, t_hi, got, (m, first + t_lo + f, n))
    print(trial, B, nx, ny, t_hi - t_lo + 1, "bad", bad, flush=True)
print("TOTAL BAD", bad)
