"""Per-run timing of the template search (config 5 shape): the 2-SM block
run alone (a stream of exactly n * 32768 valid lags), the full 2^28 search,
and the same with the 2-SM mode off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P
from paper_2509_19974_b200 import _native

rng = np.random.default_rng(5)
nt = 4096
for nblk in (8191, 2048):
    ns = nblk * 32768 + nt - 1
    st = rng.laplace(size=ns).astype(np.float32)
    tpl = st[1000:1000 + nt].copy()
    td, sd = torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda()
    q = P.sign()
    for _ in range(2):
        r = P.template_search(td, sd, q, q)
    torch.cuda.synchronize()
    with _native.profile(timed=True) as pr:
        P.template_search(td, sd, q, q)
    print(nblk, "blocks of 32768:", {k: (c, round(ms, 4)) for k, (c, ms) in pr.result.items()}, r, flush=True)
    del td, sd
