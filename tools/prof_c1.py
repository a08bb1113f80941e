"""C1 (one 2^14 float64 pair, sign, full lags): per-call wall/event time vs
library kernel time, and a batch of independent C1-shaped pairs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native, workloads as W

x, y = W.c1(0)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
q = P.sign()
for _ in range(20):
    r = P.estimate_batch(xd, yd, q, q)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    r = P.estimate_batch(xd, yd, q, q)
torch.cuda.synchronize()
print(f"call: {(time.perf_counter() - t0) / n * 1e6:.1f} us")
plan = P.EstimatePlan(xd, yd, q, q)
for _ in range(20):
    plan(xd, yd)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    r = plan(xd, yd)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"plan call: issue {(t1 - t0) / n * 1e6:.1f} us, with drain {(time.perf_counter() - t0) / n * 1e6:.1f} us")
with _native.profile(timed=True) as pr:
    for _ in range(n):
        P.estimate_batch(xd, yd, q, q)
print({k: (c // n, round(ms / n * 1e3, 2)) for k, (c, ms) in pr.result.items()}, "(launches/call, us/call)")
for B in (64, 1024):
    xb, yb = xd.expand(B, -1), yd.expand(B, -1)
    P.estimate_batch(xb, yb, q, q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        r = P.estimate_batch(xb, yb, q, q)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    assert (r.numpy()["lag"] == -137).all()
    print(f"batch {B}: {dt * 1e3:.3f} ms, {B / dt:.0f} est/s")
