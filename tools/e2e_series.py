import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native, workloads as W
xs, ys, lag = W.c2()
sweep = [(W.bit_quantizer(b, W.C2_SIGMA),)*2 for b in (1, 2, 4, 8)]
for trial in range(2):
    hx, hy = torch.from_numpy(xs).pin_memory(), torch.from_numpy(ys).pin_memory()
    for mode in ("0", None):
        _native.set_option("sweep_compute", 0 if mode else 1)
        ts = []
        for i in range(40):
            t0 = time.perf_counter(); P.estimate_sweep_host(hx.numpy(), hy.numpy(), sweep); ts.append(1e3*(time.perf_counter()-t0))
        print(trial, "copy-only" if mode else "e2e", " ".join(f"{t:.2f}" for t in ts), flush=True)
