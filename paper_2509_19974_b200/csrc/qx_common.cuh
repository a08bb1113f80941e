// qx_common.cuh -- device helpers shared by the correlation kernels.
//
// Modular arithmetic for the NTT path (primes p < 2^30, so lazily reduced
// values in [0, 4p) fit a 32-bit word) and the exact quantiser-level
// evaluation that replaces the reference's float64 Quantizer.__call__
// (quantize.py:53-65) by threshold compares.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qx {

// ------------------------------------------------------------ modular ops

// [0,4p) -> [0,2p)
__device__ __forceinline__ uint32_t red2p(uint32_t x, uint32_t p2) { return min(x, x - p2); }
// [0,2p) -> [0,p)
__device__ __forceinline__ uint32_t redp(uint32_t x, uint32_t p) { return min(x, x - p); }

// Shoup multiplication by a precomputed constant w (< p) with
// wq = floor(w * 2^32 / p): any a < 2^32 -> a*w mod p in [0, 2p).
__device__ __forceinline__ uint32_t shoup(uint32_t a, uint32_t w, uint32_t wq, uint32_t p)
{
    uint32_t q = __umulhi(a, wq);
    return a * w - q * p;
}

// Montgomery product a*b*2^-32 mod p, valid when a*b < p*2^32; result in
// (0, 2p).  pinv = p^-1 mod 2^32.  (t - m p) / 2^32 with m = lo(t)*pinv has
// no borrow in the low word, so it is hi(t) - hi(m p), in (-p, p).
__device__ __forceinline__ uint32_t montmul(uint32_t a, uint32_t b, uint32_t p, uint32_t pinv)
{
    uint32_t lo = a * b;
    uint32_t hi = __umulhi(a, b);
    uint32_t m = lo * pinv;
    return hi - __umulhi(m, p) + p;
}

struct ModP {
    uint32_t p, p2, pinv;
    uint32_t zero;  // runtime 0: keeps two-input adds as ALU IADD3 (see below)
};

// The FMA-heavy pipe carries every 32-bit multiply (3 per Shoup product), so
// the butterflies keep all additions on the ALU pipe: every add is written
// with three inputs, which only IADD3 (ALU) can execute, instead of the
// two-input form ptxas likes to issue as IMAD.IADD on the FMA pipe.

// DIF (Gentleman-Sande) butterfly, inputs/outputs in [0, 2p):
//   (a, b) -> (a + b, (a - b) * w)
__device__ __forceinline__ void bfly_dif(uint32_t& a, uint32_t& b, uint2 w, const ModP& m)
{
    const uint32_t s = a + b + m.zero;  // IADD3
    const uint32_t d = a - b + m.p2;    // IADD3
    a = red2p(s, m.p2);                 // VIADDMNMX
    b = shoup(d, w.x, w.y, m.p);
}

// DIF butterfly with twiddle 1: (a + b, a - b), same ranges as bfly_dif
__device__ __forceinline__ void bfly_dif1(uint32_t& a, uint32_t& b, const ModP& m)
{
    const uint32_t s = a + b + m.zero;  // IADD3
    const uint32_t d = a - b + m.p2;    // IADD3
    a = red2p(s, m.p2);
    b = red2p(d, m.p2);
}

// DIT butterfly with twiddle 1, same ranges as bfly_dit
__device__ __forceinline__ void bfly_dit1(uint32_t& a, uint32_t& b, const ModP& m)
{
    const uint32_t x = red2p(a, m.p2);
    const uint32_t t = red2p(b, m.p2);
    a = x + t + m.zero;
    b = x - t + m.p2;
}

// DIT (Cooley-Tukey) butterfly, inputs/outputs in [0, 4p):
//   (a, b) -> (a + w b, a - w b)
__device__ __forceinline__ void bfly_dit(uint32_t& a, uint32_t& b, uint2 w, const ModP& m)
{
    const uint32_t x = red2p(a, m.p2);
    const uint32_t t = shoup(b, w.x, w.y, m.p);
    a = x + t + m.zero;                // IADD3
    b = x - t + m.p2;                  // IADD3
}

// ------------------------------------------------------------- quantiser

// Level evaluation modes (chosen on the host from the Quantizer):
//   QM_K1      -- k == 1 (sign, uniform(1,.), custom k=1): two compares
//   QM_UNIFORM -- uniform(k, step): fp32/fp64 estimate, exact fix-up
//                 against the threshold table (at most a step or two)
//   QM_BSEARCH -- custom with k > 1: branchless binary search
//   QM_CODES   -- input already integer codes with |c| <= k (IntSignal)
//   QM_RESIDUE -- input already NTT residues in [0, 2p) (inner transforms of
//                 the large-P path), no statistics
enum QMode : int { QM_K1 = 0, QM_UNIFORM = 1, QM_BSEARCH = 2, QM_CODES = 3, QM_RESIDUE = 4 };

// Threshold semantics (built on the host by qx_thresholds.cpp): T[i],
// i in [0, 2k), is the smallest value of the input type whose reference
// level is >= i - k + 1, so level(v) = -k + #{i : v >= T[i]}.  The table
// is padded with +inf to a power of two (tsize) for the binary search.
struct QParams {
    int mode;
    int k;
    int tsize;      // padded table length (power of two, >= 2k)
    int tbits;      // log2(tsize)
    double inv_step; // 1/step for QM_UNIFORM's estimate
    const void* thr; // device table (float for f32 input, double for f64)
};

template <typename T>
__device__ __forceinline__ int level_k1(T v, T t0, T t1)
{
    return (v >= t0 ? 1 : 0) + (v >= t1 ? 1 : 0) - 1;
}

template <typename T>
__device__ __forceinline__ int level_bsearch(T v, const T* s, int tbits)
{
    int pos = 0;
    for (int b = tbits - 1; b >= 0; --b) {
        int step = 1 << b;
        if (s[pos + step - 1] <= v) pos += step;
    }
    return pos + (s[pos] <= v ? 1 : 0);
}

// Fast exact uniform level: the estimate e of |v|/step + 0.5 is within 2^-15
// of the float64 value (k <= 128), so floor(e) is exact unless e lies within
// 2^-14 of an integer; only then (rare, and NaN) take the threshold compare.
__device__ __forceinline__ int level_uniform_fast(float v, const float* s, int k, float inv_step)
{
    const float e = fmaf(fabsf(v), inv_step, 0.5f);
    const float fl = floorf(e);
    const float fr = e - fl;
    int lv = e >= (float)k + 0.5f ? k : (int)fl;
    const bool safe = (fr >= 0x1p-14f) & (fr <= 1.0f - 0x1p-14f) | (e >= (float)k + 0.5f);
    if (__builtin_expect(!safe, 0)) {
        lv = e >= (float)k ? k : (int)e;
        const int sg = v < 0.f ? -lv : lv;
        int l2 = sg;
        if (l2 < k && v >= s[l2 + k]) ++l2;
        if (l2 > -k && !(v >= s[l2 + k - 1])) --l2;
        return l2;
    }
    return v < 0.f ? -lv : lv;
}

// Conversion-free uniform level for batches (no F2I/FRND, which issue on
// the quarter-rate conversion pipe): round-to-nearest of |v|/step through
// the 1.5*2^23 magic constant (one FFMA, one integer subtract).  The
// reference rounds half away from zero; the two roundings agree unless
// |v|/step is within 2^-14 of a half-integer (the fp32 product is within
// 2^-15 of the float64 quotient for k <= 128), and values >= 2^22 saturate
// monotonically and clamp to k.  `bad` is raised for those rare samples (and
// NaN, +-inf); callers redo a batch with `bad` set through the exact
// threshold compares.
__device__ __forceinline__ int level_uniform_nb(float v, int k, float inv_step, bool& bad)
{
    const float a = fabsf(v);
    const float t = fmaf(a, inv_step, 12582912.0f);
    const int lv = min(__float_as_int(t) - 0x4B400000, k);
    const float d = fmaf(a, inv_step, -(t - 12582912.0f));
    bad |= !(fabsf(fabsf(d) - 0.5f) >= 0x1p-14f);
    return v < 0.f ? -lv : lv;
}

template <typename T>
__device__ __forceinline__ int level_uniform(T v, const T* s, int k, T inv_step)
{
    // estimate: round-half-away of |v|/step, clamped.  For k <= 128 the
    // estimate of |v|/step + 0.5 (<= 128.5) is within 2^-16 of the float64
    // value, so it is off by at most one level; one exact compare in each
    // direction fixes it: level >= j  <=>  v >= s[j + k - 1].
    T a = v < T(0) ? -v : v;
    T e = a * inv_step + T(0.5);
    int lv = e >= T(k) ? k : (int)e;   // NaN -> 0 (flagged separately)
    if (v < T(0)) lv = -lv;
    if (lv < k && v >= s[lv + k]) ++lv;
    if (lv > -k && !(v >= s[lv + k - 1])) --lv;
    return lv;
}

}  // namespace qx
