"""Exact-arithmetic model of the NTT correlation kernels' index math.

Mirrors paper_2509_19974_b200/csrc/qx_ntt.cu: four-step P = N1*N2 transform,
pass 1 = column DIF over n1 (+ forward four-step twiddle), pass 2 = row DIF of
both operands, pointwise product, row DIT, inverse four-step twiddle with
folded 1/P, pass 3 = column DIT.  In-tile transforms are grouped into radix-2^r
register groups exactly as the kernels do, so an indexing mistake shows up
here on the CPU instead of on the GPU.  Used by tests/test_ntt_model.py.
"""

from __future__ import annotations

import numpy as np

PRIMES = {  # p: (2-adicity, primitive root)
    1012924417: (21, 5),
    1004535809: (21, 3),
    998244353: (23, 3),
    469762049: (26, 3),
    167772161: (25, 3),
}


def proot(p):
    return PRIMES[p][1]


def root_of_unity(p, n):
    """Primitive n-th root of unity mod p (n a power of two)."""
    g = proot(p)
    assert (p - 1) % n == 0
    return pow(g, (p - 1) // n, p)


def schedule(l):
    """Register-group radices for a length-2^l transform (DIF order):
    ceil(l/4) groups of radix 2^3..2^4, larger groups first."""
    n = -(-l // 4)
    base, extra = divmod(l, n)
    return [base + 1] * extra + [base] * (n - extra)


def dif_group(x, p, l, s0, r, tw):
    """One DIF group pass over vector x (len 2^l), stages s0..s0+r-1."""
    L = 1 << l
    B = L >> s0
    S = B >> r
    for g in range(L >> r):
        b, j0 = divmod(g, S)
        idx = [b * B + j0 + k * S for k in range(1 << r)]
        v = [x[i] for i in idx]
        for t in range(r):
            h = 1 << (r - 1 - t)
            for k in range(1 << r):
                if k & h:
                    continue
                kp = k & (h - 1)
                w = tw[(j0 + kp * S) << (s0 + t)]
                a, c = v[k], v[k + h]
                v[k] = (a + c) % p
                v[k + h] = (a - c) * w % p
        for i, val in zip(idx, v):
            x[i] = val


def dit_group(x, p, l, s0, r, tw):
    """One DIT group pass (bit-reversed input order), stages s0..s0+r-1."""
    L = 1 << l
    Bp = 1 << (s0 + r)
    for g in range(L >> r):
        b = g >> s0
        j0 = g & ((1 << s0) - 1)
        idx = [b * Bp + j0 + (k << s0) for k in range(1 << r)]
        v = [x[i] for i in idx]
        for t in range(r):
            h = 1 << t
            for k in range(1 << r):
                if k & h:
                    continue
                kpp = k & (h - 1)
                j = j0 + (kpp << s0)
                w = tw[j << (l - s0 - t - 1)]
                a, c = v[k], v[k + h] * w % p
                v[k] = (a + c) % p
                v[k + h] = (a - c) % p
        for i, val in zip(idx, v):
            x[i] = val


def ntt_dif(x, p, l, root):
    L = 1 << l
    tw = [pow(root, e, p) for e in range(L // 2)]
    s0 = 0
    for r in schedule(l):
        dif_group(x, p, l, s0, r, tw)
        s0 += r


def ntt_dit(x, p, l, root):
    L = 1 << l
    tw = [pow(root, e, p) for e in range(L // 2)]
    s0 = 0
    for r in reversed(schedule(l)):
        dit_group(x, p, l, s0, r, tw)
        s0 += r


def bitrev(i, bits):
    return int(format(i, f"0{bits}b")[::-1], 2) if bits else 0


def correlate_fourstep(u, v, p, lp):
    """Full linear correlation c[t] = sum_m u[m] v[m + t - (nu-1)] via the
    kernels' four-step pipeline; returns the signed (centred) values."""
    P = 1 << lp
    l1 = (lp + 1) // 2
    l2 = lp // 2
    N1, N2 = 1 << l1, 1 << l2
    w = root_of_unity(p, P)
    wi = pow(w, p - 2, p)
    w1 = pow(w, N2, p)  # N1-th root
    w2 = pow(w, N1, p)  # N2-th root
    nu, nv = len(u), len(v)
    assert nu + nv - 1 <= P

    def pass1(sig, reverse):
        n = len(sig)
        Y = np.zeros((N1, N2), dtype=object)
        for n2 in range(N2):
            col = [0] * N1
            for n1 in range(N1):
                idx = n1 * N2 + n2
                if idx < n:
                    c = sig[n - 1 - idx] if reverse else sig[idx]
                    col[n1] = c % p
            ntt_dif(col, p, l1, w1)
            for pos in range(N1):
                k1 = bitrev(pos, l1)
                Y[pos, n2] = col[pos] * pow(w, n2 * k1, p) % p
        return Y

    Yu = pass1(u, True)
    Yv = pass1(v, False)
    Z = np.zeros((N1, N2), dtype=object)
    inv_p = pow(P, p - 2, p)
    for pos in range(N1):
        k1 = bitrev(pos, l1)
        ru = list(Yu[pos])
        rv = list(Yv[pos])
        ntt_dif(ru, p, l2, w2)
        ntt_dif(rv, p, l2, w2)
        prod = [a * b % p for a, b in zip(ru, rv)]
        ntt_dit(prod, p, l2, pow(w2, p - 2, p))
        for n2 in range(N2):
            Z[pos, n2] = prod[n2] * pow(wi, n2 * k1, p) * inv_p % p
    out = [0] * P
    for n2 in range(N2):
        col = list(Z[:, n2])
        ntt_dit(col, p, l1, pow(w1, p - 2, p))
        for n1 in range(N1):
            out[n1 * N2 + n2] = col[n1]
    half = (p - 1) // 2
    return [x - p if x > half else x for x in out[: nu + nv - 1]]


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for lp in (10, 11, 12):
        p = 998244353
        nu = int(rng.integers(1, (1 << lp) // 2 + 1))
        nv = (1 << lp) - nu + 1 - int(rng.integers(0, 3))
        u = rng.integers(-3, 4, nu).tolist()
        v = rng.integers(-3, 4, nv).tolist()
        got = correlate_fourstep(u, v, p, lp)
        want = np.correlate(np.array(v), np.array(u), "full").tolist()
        print(lp, nu, nv, got == want, schedule((lp + 1) // 2), schedule(lp // 2))
