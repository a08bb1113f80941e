"""Dump the NTT path's (value, lag, ties) records on C2-shaped inputs (full lags,
a bounded window, impulse trains with exact ties) to an .npy, for comparing two
builds of the native library (QX_NATIVE_LIB): python tools/ab_dump.py out.npy"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import workloads as W

xs, ys, lag = W.c2()
xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
out = []
for b in (1, 2, 4, 8):
    q = W.bit_quantizer(b, W.C2_SIGMA)
    out.append(P.estimate_batch(xd, yd, q, q, path="ntt").numpy())
    out.append(P.estimate_batch(xd, yd, q, q, path="ntt", lag_lo=-5000, lag_hi=777).numpy())
    out.append(P.estimate_batch(xd, yd, q, q, path="ntt", lag_lo=100000, lag_hi=262143).numpy())
# impulse trains: every correlation value is 0 or +-1 -> many exact ties
rng = np.random.default_rng(5)
n = 1 << 18
xi = np.zeros((16, n), np.float32)
yi = np.zeros((16, n), np.float32)
for r in range(16):
    xi[r, rng.choice(n, 3 + r, replace=False)] = rng.choice([-1.0, 1.0], 3 + r)
    yi[r, rng.choice(n, 2 + r, replace=False)] = rng.choice([-1.0, 1.0], 2 + r)
q1 = P.uniform(1, 1.0)
xt, yt = torch.from_numpy(xi).cuda(), torch.from_numpy(yi).cuda()
out.append(P.estimate_batch(xt, yt, q1, q1, path="ntt").numpy())
out.append(P.estimate_batch(xt, yt, q1, q1, path="ntt", lag_lo=-3000, lag_hi=200000).numpy())
# all-zero rows (degenerate) and a constant row
z = torch.zeros(4, n, device="cuda")
o = torch.ones(4, n, device="cuda")
out.append(P.estimate_batch(z, o, q1, q1, path="ntt").numpy())
out.append(P.estimate_batch(o, o, q1, q1, path="ntt").numpy())
torch.cuda.synchronize()
rec = np.concatenate([np.stack([r["value"], r["lag"], r["ties"]], 1) for r in out])
np.save(sys.argv[1], rec)
print("dumped", rec.shape, "ties max", rec[:, 2].max(), os.environ.get("QX_NATIVE_LIB", "in-tree"))
