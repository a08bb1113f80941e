"""qx_plan_run_host per-call time on BASELINE config 1 from page-locked rows: read in place over
PCIe (zero_copy = 1, the default) against staged on the device (zero_copy = 0)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native, workloads as W
x, y = W.c1(0)
xh = torch.from_numpy(x).pin_memory().numpy(); yh = torch.from_numpy(y).pin_memory().numpy()
plan = P.EstimatePlan(x, y, P.sign(), P.sign())
print(type(plan))
for zc in (1, 0, 1):
    _native.set_option("zero_copy", zc)
    for _ in range(50): r = plan.run_host(xh, yh)
    t = time.perf_counter()
    for _ in range(2000): r = plan.run_host(xh, yh)
    dt = (time.perf_counter() - t) / 2000
    print("zero_copy", zc, f"{dt*1e6:.2f} us/call", int(r["lag"][0]), int(r["value"][0]))
