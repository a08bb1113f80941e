"""Randomised template-search parity sweep over every mode (default, QX_TC_T4=1, QX_TC_F2=1) against the oracle: python tools/sweep_template_search.py [seed] [trials]."""
import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np, torch
import paper_2509_19974_b200 as qx
import oracle
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 99)
quants = [qx.sign(), qx.uniform(1, 0.6), qx.uniform(2, 0.5), qx.uniform(3, 0.4), qx.uniform(4, 0.2), qx.uniform(7, 0.3), qx.custom([-0.5, 0.2])]
bad = 0
for trial in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    nt = int(rng.choice([4, 8, 36, 100, 512, 1023, 1024, 2048, 3000, 4092, 4096, 4100]))
    ns = nt + int(rng.integers(0, 90000))
    st = rng.laplace(size=ns).astype(np.float32)
    off = int(rng.integers(0, ns - nt + 1))
    tpl = st[off:off + nt].copy()
    st = st + rng.normal(0, rng.uniform(0.2, 1.5), ns).astype(np.float32)
    qa = quants[int(rng.integers(len(quants)))]
    qb = qa if rng.random() < 0.5 else quants[int(rng.integers(len(quants)))]
    if (qa.k == 1) != (qb.k == 1) or (qa.kind == "custom") != (qb.kind == "custom"):
        qb = qa
    for env in ({}, {"tc_f4": 0}):  # the fp4 tensor-core search, and the int8 / NTT fallbacks
        from paper_2509_19974_b200 import _native

        _native.set_option("tc_f4", int(env.get("tc_f4", 1)))
        try:
            got = qx.template_search(tpl, st, qa, qb, stream_start=3)
        except Exception as e:
            got = ("exc", type(e).__name__)
        u, v = oracle.quantize(qa, tpl), oracle.quantize(qb, st)
        if not u.any() or not v.any():
            continue
        m, f, n = oracle.argmax(oracle.xcorr_bf(u, v, nt - 1, ns - 1))
        if got != (m, f + 3, n):
            bad += 1
            print("BAD", trial, env, nt, ns, qa, qb, got, (m, f + 3, n), flush=True)
print("template sweep bad", bad)
