"""Packed quantiser throughput: C2-shaped rows (64 x 2^18 float32) at every
field width, HBM GB/s of the kernel (float bytes read + packed bytes written)
from CUDA events over repeated launches."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native, workloads as W

x = torch.randn((64, 1 << 18), dtype=torch.float32, device="cuda") * 1.1
out = {}
for b in (1, 2, 4, 8):
    q = W.bit_quantizer(b, W.C2_SIGMA)
    bits = 1 if b == 1 else b
    for _ in range(3):
        w = P.quantize_packed(q, x, bits)[0]
    torch.cuda.synchronize()
    n = 50
    with _native.profile(timed=True) as pr:  # events around each launch on its stream
        for _ in range(n):
            P.quantize_packed(q, x, bits)
    c, tot = pr.result["quantize"]
    ms = tot / c
    byts = x.numel() * 4 + w.numel() * 4
    out[f"b{b}"] = {"ms": ms, "gbs": byts / ms / 1e6, "bytes": byts}
print(json.dumps(out))
