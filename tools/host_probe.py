"""Host-side cost per C1 call, piece by piece (issue rate, no sync)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native as N, workloads as W

x, y = W.c1(0)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
out = torch.empty((1, 8), dtype=torch.int64, device="cuda")
plan = P.EstimatePlan(xd, yd, P.sign(), P.sign())
L = N.load()
n = 2000


def rate(name, fn):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:42s} issue {(t1 - t0) / n * 1e6:6.2f} us   with drain {(t2 - t0) / n * 1e6:6.2f} us")


h, xp, yp, op = plan._h, xd.data_ptr(), yd.data_ptr(), out.data_ptr()
sh = torch._C._cuda_getCurrentRawStream(0)
libc = ctypes.CDLL(None)
rate("ctypes libc getpid", lambda: libc.getpid())
rate("torch stream handle", lambda: torch._C._cuda_getCurrentRawStream(0))
rate("3x data_ptr", lambda: (xd.data_ptr(), yd.data_ptr(), out.data_ptr()))
rate("torch.empty (1,8) int64", lambda: torch.empty((1, 8), dtype=torch.int64, device="cuda"))
rate("qx_plan_run (raw ints)", lambda: L.qx_plan_run(h, xp, yp, op, sh))
rate("EstimatePlan(out=)", lambda: plan(xd, yd, out=out))
rate("EstimatePlan()", lambda: plan(xd, yd))
rate("estimate_batch(out=)", lambda: P.estimate_batch(xd, yd, P.sign(), P.sign(), out=out))
empty = torch.zeros(1, device="cuda")
rate("torch tiny kernel (add_)", lambda: empty.add_(1))
