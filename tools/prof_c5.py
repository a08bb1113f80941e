"""Short driver for the template-search path (BASELINE config 5 shape,
reduced stream): argv[1] = log2 stream length (default 24), b = 2."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2509_19974_b200 as P

ls = int(sys.argv[1]) if len(sys.argv) > 1 else 24
rng = np.random.default_rng(5)
st = rng.laplace(size=1 << ls).astype(np.float32)
off = 123457 % ((1 << ls) - 4096)
tpl = st[off:off + 4096].copy()
st += rng.normal(0, 0.8, st.size).astype(np.float32)
td, sd = torch.from_numpy(tpl).cuda(), torch.from_numpy(st).cuda()
qa, qb = P.uniform(1, 1.5 * math.sqrt(2.0)), P.uniform(1, 1.5 * math.sqrt(2.0 + 0.64))
for _ in range(3):
    r = P.template_search(td, sd, qa, qb)
torch.cuda.synchronize()
assert r[1] == off, r
print("ok", r)
if os.environ.get("QX_PROF"):
    from paper_2509_19974_b200 import _native
    torch.cuda.synchronize()
    with _native.profile(timed=True) as pr:
        P.template_search(td, sd, qa, qb)
    print({k: (c, round(ms, 4)) for k, (c, ms) in pr.result.items()})
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    P.template_search(td, sd, qa, qb)
    e.record()
    torch.cuda.synchronize()
    print("template_search ms", s.elapsed_time(e))
