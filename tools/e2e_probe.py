"""H2D bandwidth from pinned memory and qx_estimate_sweep_host time per chunk
count (QX_SWEEP_CHUNKS) on BASELINE config 2 (64 pairs x 2^18, b = 1,2,4,8)."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

if len(sys.argv) > 1:
    import paper_2509_19974_b200 as P
    from paper_2509_19974_b200 import workloads as W

    xs, ys, lag = W.c2()
    hx, hy = torch.from_numpy(xs).pin_memory().numpy(), torch.from_numpy(ys).pin_memory().numpy()
    sweep = [(W.bit_quantizer(b, W.C2_SIGMA),) * 2 for b in (1, 2, 4, 8)]
    P.estimate_sweep_host(hx, hy, sweep)
    t0 = time.perf_counter()
    for _ in range(5):
        P.estimate_sweep_host(hx, hy, sweep)
    dt = (time.perf_counter() - t0) / 5
    print(f"chunks={os.environ.get('QX_SWEEP_CHUNKS', 'default')}: {dt * 1e3:.2f} ms/step, {256 / dt:.0f} est/s")
else:
    h = torch.empty(134217728, dtype=torch.uint8).pin_memory()
    d = torch.empty_like(h, device="cuda")
    d.copy_(h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"H2D 128 MiB pinned: {dt * 1e3:.2f} ms = {h.numel() / dt / 1e9:.1f} GB/s")
    for c in ("1", "2", "4", "8"):
        subprocess.run([sys.executable, __file__, "sweep"], env=dict(os.environ, QX_SWEEP_CHUNKS=c))
    subprocess.run([sys.executable, __file__, "sweep"], env={k: v for k, v in os.environ.items() if k != "QX_SWEEP_CHUNKS"})
