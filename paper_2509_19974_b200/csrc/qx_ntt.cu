// qx_ntt.cu -- exact full-lag integer cross-correlation by number-theoretic
// transform (the GPU replacement of the reference's Kronecker-substitution
// path, intxcorr.py:259-265: pack -> one big multiply -> unpack; here the
// "big multiply" is a cyclic convolution mod word-sized primes, which is what
// KS + GMP's FFT multiply compute underneath).
//
// Layout: P = 2^lp = N1 * N2 points, element n stored
// at row n1 = n / N2, column n2 = n % N2 of a row-major N1 x N2 matrix.
//   pass 1  per operand, tiles of 32 columns: load floats, quantise, column
//           DIF NTT over n1 (length N1), forward four-step twiddle -> Y
//   pass 2  tiles of 32 rows: row DIF of both operands (length N2),
//           pointwise product, row DIT (inverse), inverse twiddle * R^2/P -> Z
//   pass 3  tiles of 32 columns: column DIT (inverse) -> exact residues in
//           natural order -> centred lift -> argmax / values / residues
// Forward transforms are DIF (natural in, bit-reversed out), inverses DIT
// (bit-reversed in, natural out) so no permutation pass exists.  Inside a
// tile each lane owns one vector (column or row); the 32 vectors of element e
// sit at shared words e*33 + lane (one pad word per row), which is
// bank-conflict-free both for the transform (lane = vector) and for
// row-contiguous global I/O (lane = element), and turns every register-group
// access into base + compile-time offset.  Each register group of R radix-2
// stages reads its 2^R - 1 twiddles (Shoup pairs) as a contiguous block of a
// per-transform table staged in shared memory (warp-broadcast loads).
// tools/ntt_model.py is an exact-arithmetic model of the same index math.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <type_traits>

#include "qx_argmax.cuh"
#include "qx_internal.h"

#ifndef QX_NTT_THREADS
#define QX_NTT_THREADS 512
#endif

namespace qx {

constexpr int kThreads = QX_NTT_THREADS;
// loads in flight per thread in the twiddled transposed stores of passes 1 and 2
#ifndef QX_TW_UNROLL
#define QX_TW_UNROLL 8
#endif
// next-wave L2 prefetch placement: 1 = after the CTA's own load phase (all
// three passes), 0 = at kernel start (pass 2) / own tile (pass 1), as in r02 v3
#ifndef QX_PF_LATE
#define QX_PF_LATE 1
#endif
#define QX_STR_(x) #x
#define QX_UNROLL(n) _Pragma(QX_STR_(unroll n))
constexpr int kWarps = kThreads / 32;
constexpr int kPad = 33;  // words per element row of a 32-vector tile

// register-group schedule of a length-2^LOG transform: ceil(LOG/4) groups,
// radices 2^3..2^4, larger first (DIF order; DIT uses the reverse), and the
// layout of the per-group twiddle blocks.
#ifndef QX_NTT_MAXR
#define QX_NTT_MAXR 4
#endif

template <int LOG>
struct Sched {
    static constexpr int L = 1 << LOG;
    // at least two groups: the first reads global memory, the last writes it
    static constexpr int NG = (LOG + QX_NTT_MAXR - 1) / QX_NTT_MAXR < 2 ? 2 : (LOG + QX_NTT_MAXR - 1) / QX_NTT_MAXR;
    static constexpr int BASE = LOG / NG;
    static constexpr int EXTRA = LOG % NG;
    static constexpr int r(int i) { return i < EXTRA ? BASE + 1 : BASE; }
    static constexpr int s0(int i) { return i == 0 ? 0 : s0(i - 1) + r(i - 1); }
    // DIT group i = DIF group NG-1-i
    static constexpr int rd(int i) { return r(NG - 1 - i); }
    static constexpr int s0d(int i) { return i == 0 ? 0 : s0d(i - 1) + rd(i - 1); }
    // distinct j0 values per group and twiddle-block offsets (uint2 units)
    static constexpr int nj_dif(int i) { return L >> (s0(i) + r(i)); }
    static constexpr int nj_dit(int i) { return 1 << s0d(i); }
    static constexpr int twoff_dif(int i) { return i == 0 ? 0 : twoff_dif(i - 1) + nj_dif(i - 1) * (1 << r(i - 1)); }
    static constexpr int twoff_dit(int i) { return i == 0 ? 0 : twoff_dit(i - 1) + nj_dit(i - 1) * (1 << rd(i - 1)); }
    static constexpr int TW_DIF = twoff_dif(NG);
    static constexpr int TW_DIT = twoff_dit(NG);
};

// ---------------------------------------------------------------- groups

// DIF group I on 2^R registers (element k at j0 + k*S of its block).
// Twiddles: block j0 of group I, stage t at [2^R - 2^(R-t), +2^(R-1-t)).
// A group with a single block position (nj == 1: the last DIF group) has
// twiddle omega^0 = 1 at kp == 0 of every stage, known at compile time:
// those 2^R - 1 butterflies skip the product (a reduction instead).
template <int LOG, int I>
__device__ __forceinline__ void dif_regs(uint32_t (&x)[1 << Sched<LOG>::r(I)], int j0, const uint2* stw,
                                         const ModP& m)
{
    constexpr int R = Sched<LOG>::r(I);
    constexpr bool unit0 = Sched<LOG>::nj_dif(I) == 1;
    const uint2* tw = stw + Sched<LOG>::twoff_dif(I) + j0 * (1 << R);
#pragma unroll
    for (int t = 0; t < R; ++t) {
        const int h = 1 << (R - 1 - t);
        const int off = (1 << R) - (1 << (R - t));
#pragma unroll
        for (int kp = 0; kp < h; ++kp) {
            if (unit0 && kp == 0) {
#pragma unroll
                for (int blk = 0; blk < (1 << R); blk += 2 * h) bfly_dif1(x[blk], x[blk + h], m);
                continue;
            }
            const uint2 w = tw[off + kp];
#pragma unroll
            for (int blk = 0; blk < (1 << R); blk += 2 * h) bfly_dif(x[blk + kp], x[blk + kp + h], w, m);
        }
    }
}

// DIT group I (element k at j0 + (k << S0) of its block); stage t twiddles
// at [2^t - 1, +2^t).
template <int LOG, int I>
__device__ __forceinline__ void dit_regs(uint32_t (&x)[1 << Sched<LOG>::rd(I)], int j0, const uint2* stw,
                                         const ModP& m)
{
    constexpr int R = Sched<LOG>::rd(I);
    constexpr bool unit0 = Sched<LOG>::nj_dit(I) == 1;  // first DIT group: twiddle 1 at kp == 0
    const uint2* tw = stw + Sched<LOG>::twoff_dit(I) + j0 * (1 << R);
#pragma unroll
    for (int t = 0; t < R; ++t) {
        const int h = 1 << t;
#pragma unroll
        for (int kp = 0; kp < h; ++kp) {
            if (unit0 && kp == 0) {
#pragma unroll
                for (int blk = 0; blk < (1 << R); blk += 2 * h) bfly_dit1(x[blk], x[blk + h], m);
                continue;
            }
            const uint2 w = tw[h - 1 + kp];
#pragma unroll
            for (int blk = 0; blk < (1 << R); blk += 2 * h) bfly_dit(x[blk + kp], x[blk + kp + h], w, m);
        }
    }
}

// DIF group I over one or two smem tiles (two share the twiddle loads)
template <int LOG, int I, int NT>
__device__ __forceinline__ void dif_group_smem(uint32_t* s0, uint32_t* s1, const uint2* stw, const ModP& m)
{
    using SC = Sched<LOG>;
    constexpr int R = SC::r(I), S0 = SC::s0(I), B = SC::L >> S0, S = B >> R, NGRP = SC::L >> R;
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int g = threadIdx.x >> 5; g < NGRP; g += kWarps) {
        const int j0 = g & (S - 1);
        const int off = ((g / S) * B + j0) * kPad + lane;
        uint32_t x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) x[k] = s0[off + k * S * kPad];
        if constexpr (NT == 2) {
            uint32_t y[1 << R];
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) y[k] = s1[off + k * S * kPad];
            dif_regs<LOG, I>(y, j0, stw, m);
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) s1[off + k * S * kPad] = y[k];
        }
        dif_regs<LOG, I>(x, j0, stw, m);
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) s0[off + k * S * kPad] = x[k];
    }
}

template <int LOG, int I>
__device__ __forceinline__ void dit_group_smem(uint32_t* s, const uint2* stw, const ModP& m)
{
    using SC = Sched<LOG>;
    constexpr int R = SC::rd(I), S0 = SC::s0d(I), NGRP = SC::L >> R;
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int g = threadIdx.x >> 5; g < NGRP; g += kWarps) {
        const int j0 = g & ((1 << S0) - 1);
        const int off = ((g >> S0) * (1 << (S0 + R)) + j0) * kPad + lane;
        uint32_t x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) x[k] = s[off + (k << S0) * kPad];
        dit_regs<LOG, I>(x, j0, stw, m);
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) s[off + (k << S0) * kPad] = x[k];
    }
}

// DIF groups [I, NG-1) with a barrier after each
template <int LOG, int I, int NT>
__device__ __forceinline__ void dif_middle(uint32_t* s0, uint32_t* s1, const uint2* stw, const ModP& m)
{
    if constexpr (I < Sched<LOG>::NG - 1) {
        dif_group_smem<LOG, I, NT>(s0, s1, stw, m);
        __syncthreads();
        dif_middle<LOG, I + 1, NT>(s0, s1, stw, m);
    }
}

// DIT groups [I, NG-1)
template <int LOG, int I>
__device__ __forceinline__ void dit_middle(uint32_t* s, const uint2* stw, const ModP& m)
{
    if constexpr (I < Sched<LOG>::NG - 1) {
        dit_group_smem<LOG, I>(s, stw, m);
        __syncthreads();
        dit_middle<LOG, I + 1>(s, stw, m);
    }
}

// Warp-strided loop g = first, first + step, ... < end whose global loads run
// one iteration ahead: two register buffers alternate roles (2x unrolled), so
// no buffer-rotation moves land on the FMA pipe.
template <typename Buf, typename Fetch, typename Body>
__device__ __forceinline__ void prefetched_loop(int first, int end, int step, Fetch fetch, Body body)
{
    Buf ba, bb;
    if (first < end) fetch(ba, first);
#pragma unroll 1
    for (int g = first; g < end; g += 2 * step) {
        if (g + step < end) fetch(bb, g + step);
        body(ba, g);
        if (g + step >= end) break;
        if (g + 2 * step < end) fetch(ba, g + 2 * step);
        body(bb, g + step);
    }
}

// Next-wave L2 prefetch: the passes run one CTA per SM and load their
// whole tile before computing on it, so an SM idles through every tile's
// load latency.  Each CTA therefore pulls the tile of the CTA one wave
// later (linear block id + number of SMs) into L2, one 128-B segment per
// prefetch; that CTA's loads then wait on L2 instead of HBM.
__device__ __forceinline__ bool next_wave_block(int& bx, int& by, int& bz)
{
    unsigned nsm;
    asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    const long long L = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z) + nsm;
    const long long n = (long long)gridDim.x * gridDim.y * gridDim.z;
    if (L >= n) return false;
    bx = (int)(L % gridDim.x);
    by = (int)((L / gridDim.x) % gridDim.y);
    bz = (int)(L / ((long long)gridDim.x * gridDim.y));
    return true;
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

template <typename T, int N>
struct RegBuf {
    T v[N];
};

// copy a twiddle table (uint2) into shared memory, all threads
__device__ __forceinline__ void stage_table(uint2* dst, const uint2* __restrict__ src, int n)
{
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int i = threadIdx.x; i < n / 2; i += kThreads) d4[i] = __ldg(&s4[i]);
}

// ------------------------------------------------------------ statistics

__device__ __forceinline__ bool cs_single(const unsigned long long* stats, int64_t pair, uint32_t p0)
{
    // |c| <= sqrt(Su*Sv) (Cauchy-Schwarz on the codes); a single prime
    // suffices when that is <= (p0-1)/2.
    const unsigned long long su = stats[pair * 8 + 0], sv = stats[pair * 8 + 4];
    const unsigned long long h = (p0 - 1) / 2;
    return (unsigned __int128)su * sv <= (unsigned __int128)h * h;
}

// ------------------------------------------------------------ quantiser

template <typename T, int QM>
__device__ __forceinline__ int quant_level(T v, const T* sthr, int k, int tbits, T inv_step, T t0, T t1)
{
    if constexpr (QM == QM_K1) return level_k1(v, t0, t1);
    else if constexpr (QM == QM_UNIFORM) return level_uniform(v, sthr, k, inv_step);
    else return level_bsearch(v, sthr, tbits) - k;
}

template <typename T, int QM>
__device__ __forceinline__ int load_code(const T* __restrict__ src, int64_t i, const T* sthr, int k,
                                         int tbits, T inv_step, T t0, T t1, unsigned& flags)
{
    if constexpr (QM == QM_CODES) {
        const long long c = src[i];
        if (c > k || c < -k) flags |= SF_CODE_RANGE;
        return (int)c;
    } else {
        const T v = __ldg(&src[i]);
        if (v != v) flags |= SF_NONFINITE;
        return quant_level<T, QM>(v, sthr, k, tbits, inv_step, t0, t1);
    }
}

// ------------------------------------------------------------------ pass 1

struct Pass1Args {
    OperandDesc op[2];
    uint32_t* Y;          // Y^T: [pair][op][n2][k1pos]
    const uint2* gtw;     // DIF group twiddles for N1
    const uint2* twf;     // forward four-step twiddles, transposed [n2][k1pos] (Shoup pairs)
    const uint2* twab;    // the same factored: [n2][32 A + N1/32 B] (NttTables::twab), or null
    unsigned long long* stats;
    ModP m;
    uint32_t p0;
    int N2;
    int zero_upper;
    int skip_cs;
    int op_base;     // operand index of blockIdx.y == 0 (1 when launched per operand)
    int pair_shift;  // statistics record = pair >> pair_shift (inner transforms)
    int64_t pair0;
    int64_t row0;    // pair index of row 0 of op[].data (inner transforms: the launch group's first
                     // sub-transform, whose rows start the group-local outer-pass buffer)
};

template <int LOG1>
constexpr size_t pass1_smem(size_t tsz)
{
    return (size_t)(1 << LOG1) * kPad * 4 + (size_t)Sched<LOG1>::TW_DIF * 8 + (size_t)kMaxThr * tsz;
}

template <typename T, int QM>
__device__ __forceinline__ int level_of(T v, const T* sthr, int k, int tbits, T inv_step, T t0, T t1)
{
    if constexpr (QM == QM_UNIFORM && std::is_same<T, float>::value)
        return level_uniform_fast(v, sthr, k, inv_step);
    else
        return quant_level<T, QM>(v, sthr, k, tbits, inv_step, t0, t1);
}

template <int LOG1, typename T, int QM, bool ZU>
__global__ void __launch_bounds__(kThreads, 1) k_pass1(const __grid_constant__ Pass1Args a)
{
    constexpr int N1 = 1 << LOG1;
    using SC = Sched<LOG1>;
    constexpr int R0 = SC::r(0), S = N1 >> R0, RAD0 = 1 << R0;
    constexpr int RL = SC::r(SC::NG - 1), RADL = 1 << RL;
    extern __shared__ __align__(16) uint32_t smem[];
    uint2* stw = reinterpret_cast<uint2*>(smem + N1 * kPad);
    T* sthr = reinterpret_cast<T*>(stw + SC::TW_DIF);

    const int op = a.op_base + blockIdx.y;
    const int64_t pl = blockIdx.z, pair = a.pair0 + pl;
    if (a.skip_cs && cs_single(a.stats, pair >> a.pair_shift, a.p0)) return;
    const OperandDesc& d = a.op[blockIdx.y];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int N2 = a.N2;
    const int c0 = blockIdx.x * 32;
    const int col = c0 + lane;
    const ModP m = a.m;

    stage_table(stw, a.gtw, SC::TW_DIF);
    if constexpr (QM != QM_CODES) {
        for (int i = threadIdx.x; i < d.q.tsize; i += kThreads) sthr[i] = (T)d.q.thr[i];
    }
    __syncthreads();
    T t0 = T(0), t1 = T(0);
    if constexpr (QM == QM_K1) { t0 = sthr[0]; t1 = sthr[1]; }
    const T inv_step = (T)d.q.inv_step;
    const int k = d.q.k, tbits = d.q.tbits;
    const T* src = reinterpret_cast<const T*>(d.data) + (pair - a.row0) * d.ld;
    const int64_t n = d.n;
    const bool rev = d.reverse;
    // every element of this tile's loaded rows is in range (no per-element checks)
    const int rows_loaded = ZU ? N1 / 2 : N1;
    const bool full = (int64_t)(rows_loaded - 1) * N2 + c0 + 31 < n;
    const T* base = rev ? src + (n - 1 - col) : src + col;
    const int rstride = rev ? -N2 : N2;
    constexpr int NLD = ZU ? RAD0 / 2 : RAD0;  // rows actually loaded per group

    // pull the tile's rows (128 B each: the 32 columns) into L2 up front; the
    // register loads run one group ahead and then wait on L2, not HBM
    // (C2: pass 1 0.888 -> 0.879 ms per 4-depth step; prefetching the next
    // wave's tile instead measured 0.888)
#if !QX_PF_LATE
    if (full) {
        for (int r = threadIdx.x; r < rows_loaded; r += kThreads)
            prefetch_l2(rev ? base - lane + 31 - (int64_t)r * N2 : base - lane + (int64_t)r * N2);
    }
#endif
    // per-thread sums stay far below 2^32 (<= 64 samples of k^2 <= 2^14)
    unsigned ssq = 0, nnz = 0;
    unsigned flags = 0;
    auto to_res = [&](int c) -> uint32_t {
        ssq += (unsigned)(c * c);
        nnz += (c != 0);
        return c < 0 ? (uint32_t)(c + (int)m.p) : (uint32_t)c;
    };
    // first DIF group straight from global memory (coalesced: lane = column)
    if (full) {
        // register double buffer: the next group's raw samples are in flight
        // while this group is quantised and transformed
        using Raw = typename std::conditional<QM == QM_CODES, long long, T>::type;
        using Buf = RegBuf<Raw, NLD>;
        auto fetch = [&](Buf& b, int g) {
#pragma unroll
            for (int kk = 0; kk < NLD; ++kk) b.v[kk] = __ldg(&base[(g + kk * S) * rstride]);
        };
        auto body = [&](const Buf& b, int g) {
                uint32_t x[RAD0];
                if constexpr (QM == QM_UNIFORM && std::is_same<T, float>::value) {
                    // branch-free levels of the whole group; a rare exact redo
                    // (near a rounding half-point, NaN, inf) for the group
                    int c[NLD];
                    bool bad = false;
#pragma unroll
                    for (int kk = 0; kk < NLD; ++kk) c[kk] = level_uniform_nb(b.v[kk], k, inv_step, bad);
                    if (__builtin_expect(bad, 0)) {
#pragma unroll
                        for (int kk = 0; kk < NLD; ++kk) {
                            if (b.v[kk] != b.v[kk]) flags |= SF_NONFINITE;
                            c[kk] = quant_level<T, QM>(b.v[kk], sthr, k, tbits, inv_step, t0, t1);
                        }
                    }
#pragma unroll
                    for (int kk = 0; kk < RAD0; ++kk) x[kk] = kk < NLD ? to_res(c[kk]) : 0u;
                } else {
#pragma unroll
                for (int kk = 0; kk < RAD0; ++kk) {
                    if (kk >= NLD) { x[kk] = 0; continue; }
                    int c = 0;
                    if constexpr (QM == QM_RESIDUE) {
                        x[kk] = (uint32_t)b.v[kk];
                        continue;
                    } else if constexpr (QM == QM_CODES) {
                        c = (int)b.v[kk];
                        if (b.v[kk] > k || b.v[kk] < -k) flags |= SF_CODE_RANGE;
                    } else {
                        if (b.v[kk] != b.v[kk]) flags |= SF_NONFINITE;
                        c = level_of<T, QM>(b.v[kk], sthr, k, tbits, inv_step, t0, t1);
                    }
                    x[kk] = to_res(c);
                }
                }
                dif_regs<LOG1, 0>(x, g, stw, m);
                uint32_t* p = smem + g * kPad + lane;
#pragma unroll
                for (int kk = 0; kk < RAD0; ++kk) p[kk * S * kPad] = x[kk];
        };
        if constexpr (sizeof(Raw) == 8 && NLD > 8) {
            // 8-byte samples (float64 rows, int64 codes): two buffers of
            // NLD values would not fit the 128-register budget (ptxas spilled
            // 108-436 B); one buffer, its loads still issued together
#pragma unroll 1
            for (int g = warp; g < S; g += kWarps) {
                Buf b;
                fetch(b, g);
                body(b, g);
            }
        } else {
            prefetched_loop<Buf>(warp, S, kWarps, fetch, body);
        }
    } else {
#pragma unroll 1
        for (int g = warp; g < S; g += kWarps) {
            uint32_t x[RAD0];
#pragma unroll
            for (int kk = 0; kk < RAD0; ++kk) {
                x[kk] = 0;
                if (kk >= NLD) continue;
                const int64_t idx = (int64_t)(g + kk * S) * N2 + col;
                if (idx < n)
                    x[kk] = to_res(
                        load_code<T, QM>(src, rev ? n - 1 - idx : idx, sthr, k, tbits, inv_step, t0, t1, flags));
            }
            dif_regs<LOG1, 0>(x, g, stw, m);
            uint32_t* p = smem + g * kPad + lane;
#pragma unroll
            for (int kk = 0; kk < RAD0; ++kk) p[kk * S * kPad] = x[kk];
        }
    }
    // statistics: warp reduce, one atomic per warp
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
        flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if (QM != QM_RESIDUE && lane == 0 && a.p0 == m.p) {  // only the first prime's pass counts
        unsigned long long* st = a.stats + (pair * 2 + op) * 4;
        if (ssq) atomicAdd(st + 0, (unsigned long long)ssq);
        if (nnz) atomicAdd(st + 1, (unsigned long long)nnz);
        if (flags) atomicOr(st + 2, (unsigned long long)flags);
    }
#if QX_PF_LATE
    // this tile's samples are in registers or shared memory: pull the tile of the
    // CTA one wave later into L2 now, so its DRAM reads run under this CTA's
    // transform instead of beside the next wave's own loads
    if constexpr (sizeof(T) == 4) {  // (8-byte rows: the extra live values spill)
        int bx, by, bz;
        if (next_wave_block(bx, by, bz)) {
            const OperandDesc& dn = a.op[by];
            const T* sn = reinterpret_cast<const T*>(dn.data) + (a.pair0 + bz - a.row0) * dn.ld;
            const int64_t nn = dn.n;
            const int cn = bx * 32;
            if ((int64_t)(rows_loaded - 1) * N2 + cn + 31 < nn) {
                const T* bn = dn.reverse ? sn + (nn - 1 - cn - 31) : sn + cn;
                const int64_t rs = dn.reverse ? -(int64_t)N2 : (int64_t)N2;
                for (int r = threadIdx.x; r < rows_loaded; r += kThreads) prefetch_l2(bn + r * rs);
            }
        }
    }
#endif
    __syncthreads();
    dif_middle<LOG1, 1, 1>(smem, nullptr, stw, m);
    // last DIF group (in shared memory)
#pragma unroll 1
    for (int g = warp; g < (N1 >> RL); g += kWarps) {
        uint32_t x[RADL];
        uint32_t* p = smem + g * RADL * kPad + lane;
#pragma unroll
        for (int kk = 0; kk < RADL; ++kk) x[kk] = p[kk * kPad];
        dif_regs<LOG1, SC::NG - 1>(x, 0, stw, m);
#pragma unroll
        for (int kk = 0; kk < RADL; ++kk) p[kk * kPad] = x[kk];
    }
    __syncthreads();
    // transposed store Y^T[n2][k1pos] (lane = k1pos, contiguous) with the
    // forward four-step twiddle (table in the same transposed layout)
    uint32_t* Yt = a.Y + (pl * 2 + op) * ((int64_t)N1 * N2);
    if constexpr (N1 >= 32) {
        if (a.twab) {
            // factored twiddle: one per-lane A and a warp-uniform B per row
            // (two Shoup products instead of one 8-byte L2 load per element)
            // (row pointers hoisted: every access of an unrolled chunk is base +
            // immediate; indexing Yt[o + e] cost five address instructions per store)
            constexpr int NB = N1 / 32, U = NB < QX_TW_UNROLL ? NB : QX_TW_UNROLL;
#pragma unroll 1
            for (int c = warp; c < 32; c += kWarps) {
                const uint2* tb = a.twab + (int64_t)(c0 + c) * (32 + NB);
                const uint2 A = __ldg(&tb[lane]);
                uint32_t* yp = Yt + ((int64_t)(c0 + c) * N1 + lane);
                const uint32_t* sp = smem + lane * kPad + c;
                tb += 32;
#pragma unroll 1
                for (int j0 = 0; j0 < NB; j0 += U, yp += 32 * U, sp += 32 * U * kPad, tb += U) {
                    uint2 B[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) B[u] = __ldg(&tb[u]);
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        yp[32 * u] = shoup(shoup(sp[32 * u * kPad], A.x, A.y, m.p), B[u].x, B[u].y, m.p);
                }
            }
            return;
        }
    }
#pragma unroll 1
    for (int c = warp; c < 32; c += kWarps) {
        const int o = (c0 + c) * N1;
        QX_UNROLL(QX_TW_UNROLL)
        for (int e = lane; e < N1; e += 32)
        {
            const uint2 w = __ldg(&a.twf[o + e]);
            Yt[o + e] = shoup(smem[e * kPad + c], w.x, w.y, m.p);
        }
    }
}


// ------------------------------------------------------------------ pass 2

struct Pass2Args {
    const uint32_t* Y;      // Y^T of both operands
    uint32_t* Z;            // [pair][k1pos][n2]
    const uint2* gtwf;      // DIF group twiddles for N2
    const uint2* gtwi;      // DIT group twiddles for N2
    const uint2* twinv;     // inverse four-step twiddles [k1pos][n2] (Shoup pairs, incl. R/P)
    const uint2* twib;      // the same factored: [k1pos][32 A + N2/32 B] (NttTables::twib), or null
    const unsigned long long* stats;
    ModP m;
    uint32_t p0;
    int N1;
    int skip_cs;
    int pair_shift;
    int64_t pair0;
};

template <int LOG2>
constexpr size_t pass2_smem()
{
    return (size_t)2 * (1 << LOG2) * kPad * 4 + (size_t)(Sched<LOG2>::TW_DIF + Sched<LOG2>::TW_DIT) * 8;
}

template <int LOG2>
__global__ void __launch_bounds__(kThreads, 1) k_pass2(const __grid_constant__ Pass2Args a)
{
    constexpr int N2 = 1 << LOG2;
    using SC = Sched<LOG2>;
    constexpr int R0 = SC::r(0), S = N2 >> R0, RAD0 = 1 << R0;
    constexpr int RL = SC::r(SC::NG - 1), RADL = 1 << RL;
    static_assert(SC::rd(0) == RL, "fused group needs matching radices");
    static_assert(SC::NG >= 2, "first and last groups must differ");
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* su = smem;
    uint32_t* sv = smem + N2 * kPad;
    uint2* stf = reinterpret_cast<uint2*>(sv + N2 * kPad);
    uint2* sti = stf + SC::TW_DIF;

    const int64_t pl = blockIdx.y, pair = a.pair0 + pl;
    if (a.skip_cs && cs_single(a.stats, pair >> a.pair_shift, a.p0)) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int N1 = a.N1;
    const int r0 = blockIdx.x * 32;
    const ModP m = a.m;
    const int64_t P = (int64_t)N1 * N2;
    // row vector r0+lane, element n2 at Y^T[n2*N1 + r0 + lane]: coalesced
    const uint32_t* Yu = a.Y + pl * 2 * P + r0 + lane;
    const uint32_t* Yv = Yu + P;

    auto prefetch_next_wave = [&]() {
        int bx, by, bz;
        // the next wave's tile: both operands' row segments
        if (next_wave_block(bx, by, bz)) {
            const uint32_t* Yn = a.Y + (int64_t)by * 2 * P + bx * 32;
            for (int i = threadIdx.x; i < 2 * N2; i += kThreads)
                prefetch_l2(Yn + (i >= N2 ? P : 0) + (int64_t)(i % N2) * N1);
        }
    };
#if !QX_PF_LATE
    prefetch_next_wave();
#endif
    stage_table(stf, a.gtwf, SC::TW_DIF);
    stage_table(sti, a.gtwi, SC::TW_DIT);
    __syncthreads();
    // first DIF group of both operands straight from global memory, the next
    // group's loads in flight during this group's butterflies
    {
        using Buf = RegBuf<uint32_t, 2 * RAD0>;
        prefetched_loop<Buf>(
            warp, S, kWarps,
            [&](Buf& b, int g) {
#pragma unroll
                for (int kk = 0; kk < RAD0; ++kk) {
                    b.v[kk] = __ldg(&Yu[(g + kk * S) * N1]);
                    b.v[RAD0 + kk] = __ldg(&Yv[(g + kk * S) * N1]);
                }
            },
            [&](const Buf& b, int g) {
                uint32_t xu[RAD0], xv[RAD0];
#pragma unroll
                for (int kk = 0; kk < RAD0; ++kk) {
                    xu[kk] = b.v[kk];
                    xv[kk] = b.v[RAD0 + kk];
                }
                dif_regs<LOG2, 0>(xu, g, stf, m);
                dif_regs<LOG2, 0>(xv, g, stf, m);
                const int off = g * kPad + lane;
#pragma unroll
                for (int kk = 0; kk < RAD0; ++kk) {
                    su[off + kk * S * kPad] = xu[kk];
                    sv[off + kk * S * kPad] = xv[kk];
                }
            });
    }
#if QX_PF_LATE
    // issued once this CTA's own loads have landed: the next wave's DRAM reads
    // run under this tile's transform, not beside the loads of either wave
    prefetch_next_wave();
#endif
    __syncthreads();
    dif_middle<LOG2, 1, 2>(su, sv, stf, m);
    // last DIF group of both, pointwise product, first DIT group (same
    // element grouping: consecutive blocks of 2^RL)
#pragma unroll 1
    for (int g = warp; g < (N2 >> RL); g += kWarps) {
        uint32_t xu[RADL], xv[RADL];
        const int off = g * RADL * kPad + lane;
#pragma unroll
        for (int kk = 0; kk < RADL; ++kk) {
            xu[kk] = su[off + kk * kPad];
            xv[kk] = sv[off + kk * kPad];
        }
        dif_regs<LOG2, SC::NG - 1>(xu, 0, stf, m);
        dif_regs<LOG2, SC::NG - 1>(xv, 0, stf, m);
#pragma unroll
        for (int kk = 0; kk < RADL; ++kk) xu[kk] = montmul(xu[kk], xv[kk], m.p, m.pinv);
        dit_regs<LOG2, 0>(xu, 0, sti, m);
#pragma unroll
        for (int kk = 0; kk < RADL; ++kk) su[off + kk * kPad] = xu[kk];
    }
    __syncthreads();
    // remaining DIT groups (1 .. NG-1)
    dit_middle<LOG2, 1>(su, sti, m);
    dit_group_smem<LOG2, SC::NG - 1>(su, sti, m);
    __syncthreads();
    // transposed store Z[k1pos][n2] (lane = n2) with the inverse four-step
    // twiddle (includes R/P: the product's Montgomery R^-1 cancels)
    uint32_t* Z = a.Z + pl * P;
    if constexpr (N2 >= 32) {
        if (a.twib) {
            // factored twiddle (see pass 1): per-lane A, warp-uniform B per row
            constexpr int NB = N2 / 32, U = NB < QX_TW_UNROLL ? NB : QX_TW_UNROLL;
#pragma unroll 1
            for (int c = warp; c < 32; c += kWarps) {
                const uint2* tb = a.twib + (int64_t)(r0 + c) * (32 + NB);
                const uint2 A = __ldg(&tb[lane]);
                uint32_t* zp = Z + ((int64_t)(r0 + c) * N2 + lane);
                const uint32_t* sp = su + lane * kPad + c;
                tb += 32;
#pragma unroll 1
                for (int j0 = 0; j0 < NB; j0 += U, zp += 32 * U, sp += 32 * U * kPad, tb += U) {
                    uint2 B[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) B[u] = __ldg(&tb[u]);
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        zp[32 * u] = shoup(shoup(sp[32 * u * kPad], A.x, A.y, m.p), B[u].x, B[u].y, m.p);
                }
            }
            return;
        }
    }
#pragma unroll 1
    for (int c = warp; c < 32; c += kWarps) {
        const int o = (r0 + c) * N2;
        QX_UNROLL(QX_TW_UNROLL)
        for (int e = lane; e < N2; e += 32) {
            const uint2 w = __ldg(&a.twinv[o + e]);
            Z[o + e] = shoup(su[e * kPad + c], w.x, w.y, m.p);
        }
    }
}

// ------------------------------------------------------ argmax reduction
// (Best, write_result, argmax_finish: qx_argmax.cuh)

__global__ void k_stats_to_results(const unsigned long long* stats, long long* res, int64_t batch)
{
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b < batch) write_result(res + b * 8, Best{0, 0, 0}, 0, stats + b * 8);
}

cudaError_t stats_to_results(const unsigned long long* stats, void* results, int64_t batch, cudaStream_t s)
{
    k_stats_to_results<<<(unsigned)((batch + 127) / 128), 128, 0, s>>>(stats, (long long*)results, batch);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ pass 3

struct Pass3Args {
    const uint32_t* Z;  // [pair][k1pos][n2]
    uint32_t* R;        // residue output (multi-prime)
    const uint2* gtwi;  // DIT group twiddles for N1
    const unsigned long long* stats;
    ArgmaxOut am;
    int64_t* values;
    int64_t nout;
    int64_t vld;        // row stride of values
    ModP m;
    uint32_t p0;
    int N2;
    int np;
    int pi;             // prime index
    int pair_shift;     // statistics record = pair >> pair_shift
    int force_residue;  // inner transforms: always write residues
    int64_t pair0;
};

enum { OUT_ARGMAX = 0, OUT_VALUES = 1 };

template <int LOG1>
constexpr size_t pass3_smem()
{
    return (size_t)(1 << LOG1) * kPad * 4 + (size_t)Sched<LOG1>::TW_DIT * 8;
}

template <int LOG1, int OUT>
__global__ void __launch_bounds__(kThreads, 1) k_pass3(const __grid_constant__ Pass3Args a)
{
    constexpr int N1 = 1 << LOG1;
    using SC = Sched<LOG1>;
    constexpr int R0 = SC::rd(0), RAD0 = 1 << R0, NG0 = N1 >> R0;
    constexpr int RL = SC::rd(SC::NG - 1), S0L = SC::s0d(SC::NG - 1), RADL = 1 << RL;
    extern __shared__ __align__(16) uint32_t smem[];
    uint2* sti = reinterpret_cast<uint2*>(smem + N1 * kPad);

    const int64_t pl = blockIdx.y, pair = a.pair0 + pl;
    const bool cs = (a.np > 1) && cs_single(a.stats, pair >> a.pair_shift, a.p0);
    if (a.pi > 0 && cs) return;
    const bool final_out = !a.force_residue && ((a.np == 1) || cs);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int N2 = a.N2;
    const int col = blockIdx.x * 32 + lane;
    const ModP m = a.m;
    const int64_t P = (int64_t)N1 * N2;
    const uint32_t* Zc = a.Z + pl * P + col;

    // Fused argmax of a single-prime lift: every output carries + half
    // (added once per column at the DC input below), so the canonical residue
    // k = (c + half) mod p is already a monotone key of the centred value c
    // (|c| <= half): no per-element lift, compare keys, subtract half at the end.
    const uint32_t half = (m.p - 1) / 2;
    const uint32_t bias = (OUT == OUT_ARGMAX && final_out) ? half : 0u;
    stage_table(sti, a.gtwi, SC::TW_DIT);
    __syncthreads();
    // first DIT group from global (positions g*RAD0 + k, lane = column),
    // next group's loads in flight
    {
        using Buf = RegBuf<uint32_t, RAD0>;
        prefetched_loop<Buf>(
            warp, NG0, kWarps,
            [&](Buf& b, int g) {
#pragma unroll
                for (int kk = 0; kk < RAD0; ++kk) b.v[kk] = __ldg(&Zc[(g * RAD0 + kk) * N2]);
            },
            [&](const Buf& b, int g) {
                uint32_t x[RAD0];
#pragma unroll
                for (int kk = 0; kk < RAD0; ++kk) x[kk] = b.v[kk];
                // position 0 is the column's DC term: + bias there adds bias to
                // every output of the column (inputs stay below 4p: < 2p + p/2)
                if (g == 0) x[0] += bias;
                dit_regs<LOG1, 0>(x, 0, sti, m);
                uint32_t* p = smem + g * RAD0 * kPad + lane;
#pragma unroll
                for (int kk = 0; kk < RAD0; ++kk) p[kk * kPad] = x[kk];
            });
    }
    __syncthreads();
    dit_middle<LOG1, 1>(smem, sti, m);
    // last DIT group: natural-order n1 = j0 + (k << S0L), t = n1*N2 + col.
    uint32_t* Rout = a.R + (pl * a.np + a.pi) * P;
    if (!final_out || OUT == OUT_VALUES) {
#pragma unroll 1
        for (int g = warp; g < (1 << S0L); g += kWarps) {
            uint32_t x[RADL];
            const uint32_t* p = smem + g * kPad + lane;
#pragma unroll
            for (int kk = 0; kk < RADL; ++kk) x[kk] = p[(kk << S0L) * kPad];
            dit_regs<LOG1, SC::NG - 1>(x, g, sti, m);
            const int t0 = g * N2 + col;
#pragma unroll
            for (int kk = 0; kk < RADL; ++kk) {
                const int t = t0 + (kk << S0L) * N2;
                const uint32_t r = redp(red2p(x[kk], m.p2), m.p);
                if (!final_out) Rout[t] = r;
                else if (t < a.nout) a.values[pair * a.vld + t] = (int)r - (r > half ? (int)m.p : 0);
            }
        }
        return;
    }
    if constexpr (OUT == OUT_ARGMAX) {
        // Keys of a single-prime result are < 2^30 and t < 2^25, so the peak
        // bookkeeping is 32-bit.  The warp shares one running best key wm; a
        // group of 2^RL keys per lane costs a max tree and one vote unless some
        // lane reaches wm (about ln(#groups) times per warp), and only then are
        // the group's keys scanned for the count and the smallest t at wm.
        const int tmin = blockIdx.x * 32, tmax = (N1 - 1) * N2 + blockIdx.x * 32 + 31;
        const bool inside = a.am.t_lo <= tmin && a.am.t_hi >= tmax && tmax < a.nout;
        const int tlo = (int)max(a.am.t_lo, (int64_t)0), thi = (int)min(min(a.am.t_hi, a.nout - 1), P - 1);
        uint32_t wm = 0;
        int bc = 0, bt = INT_MAX;
#pragma unroll 1
        for (int g = warp; g < (1 << S0L); g += kWarps) {
            uint32_t x[RADL];
            const uint32_t* p = smem + g * kPad + lane;
#pragma unroll
            for (int kk = 0; kk < RADL; ++kk) x[kk] = p[(kk << S0L) * kPad];
            dit_regs<LOG1, SC::NG - 1>(x, g, sti, m);
            const int t0 = g * N2 + col;
#pragma unroll
            for (int kk = 0; kk < RADL; ++kk) x[kk] = redp(red2p(x[kk], m.p2), m.p);
            if (!inside) {
                // window edge (or the unused last point of P): this CTA's keys are
                // k + 1, and 0 marks an out-of-window element (it never equals wm >= 1)
#pragma unroll
                for (int kk = 0; kk < RADL; ++kk) {
                    const int t = t0 + (kk << S0L) * N2;
                    x[kk] = (t < tlo || t > thi) ? 0u : x[kk] + 1u;
                }
            }
            uint32_t mx = x[0];
#pragma unroll
            for (int kk = 1; kk + 1 < RADL; kk += 2) mx = __vimax3_u32(mx, x[kk], x[kk + 1]);
            if constexpr (RADL % 2 == 0) mx = max(mx, x[RADL - 1]);
            if (!__any_sync(0xffffffffu, mx >= wm)) continue;
            const uint32_t wn = __reduce_max_sync(0xffffffffu, mx);
            if (!inside && wn == 0) continue;  // nothing in the window yet
            if (wn > wm) {
                wm = wn;
                bc = 0;
                bt = INT_MAX;
            }
            int kb = RADL;
#pragma unroll
            for (int kk = RADL - 1; kk >= 0; --kk) {
                if (x[kk] == wm) {
                    ++bc;
                    kb = kk;
                }
            }
            if (kb < RADL) bt = min(bt, t0 + (kb << S0L) * N2);
        }
        // warp record -> CTA record -> one partial per CTA (merged per pair by
        // k_merge_partials: no ticket, so no CTA waits on a fence and an atomic
        // round trip while it holds the SM)
        __shared__ uint32_t sk[kWarps];
        __shared__ int st[kWarps], sc[kWarps];
        const int wc = __reduce_add_sync(0xffffffffu, bc);
        const int wt = __reduce_min_sync(0xffffffffu, bt);
        if (lane == 0) {
            sk[warp] = wc ? wm + 1 : 0;  // 0: no valid element in this warp's share
            st[warp] = wt;
            sc[warp] = wc;
        }
        __syncthreads();
        if (warp == 0) {
            const uint32_t k1 = lane < kWarps ? sk[lane] : 0u;
            const uint32_t kmax = __reduce_max_sync(0xffffffffu, k1);
            const bool on = lane < kWarps && k1 == kmax && kmax > 0;
            const int c = __reduce_add_sync(0xffffffffu, on ? sc[lane] : 0);
            const int t = __reduce_min_sync(0xffffffffu, on ? st[lane] : INT_MAX);
            if (lane == 0) {
                long long* pp = a.am.partials + (pair * a.am.pstride + blockIdx.x) * 3;
                const Best b = kmax ? Best{(long long)(kmax - 1) - (inside ? 0 : 1) - (long long)half, t, c}
                                    : best_init();
                pp[0] = b.v;
                pp[1] = b.t;
                pp[2] = b.c;
            }
        }
    }
}

// per-pair merge of the per-CTA argmax partials of k_pass3 (one warp per pair)
struct MergeArgs {
    ArgmaxOut am;
    const unsigned long long* stats;
    int64_t pair0, nb;
    uint32_t p0;
    int nblk, np;
};

__global__ void __launch_bounds__(256) k_merge_partials(const __grid_constant__ MergeArgs a)
{
    const int lane = threadIdx.x & 31;
    const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= a.nb) return;
    const int64_t pair = a.pair0 + w;
    // multi-prime launches: pairs that need the CRT are finished by k_combine
    if (a.np > 1 && !cs_single(a.stats, pair, a.p0)) return;
    Best r = best_init();
    const long long* pp = a.am.partials + pair * a.am.pstride * 3;
    for (int i = lane; i < a.nblk; i += 32) best_merge(r, Best{pp[3 * i], pp[3 * i + 1], pp[3 * i + 2]});
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        Best o2{__shfl_xor_sync(0xffffffffu, r.v, o), __shfl_xor_sync(0xffffffffu, r.t, o),
                __shfl_xor_sync(0xffffffffu, r.c, o)};
        best_merge(r, o2);
    }
    if (lane == 0)
        write_result(reinterpret_cast<long long*>(a.am.results) + pair * 8, r, a.am.first_lag, a.stats + pair * 8);
}

// ----------------------------------------------------- multi-prime combine

struct CombineArgs {
    const uint32_t* R;
    const unsigned long long* stats;
    ArgmaxOut am;
    int64_t* values;
    int64_t nout, vld, P;
    uint32_t p[3];
    uint64_t ginv[3];
    uint32_t p0;
    int np;
    int64_t pair0;
};

template <int OUT>
__global__ void __launch_bounds__(256) k_combine(const __grid_constant__ CombineArgs a)
{
    const int64_t pl = blockIdx.y, pair = a.pair0 + pl;
    if (cs_single(a.stats, pair, a.p0)) return;
    const uint32_t* R = a.R + pl * a.np * a.P;
    // centred lift of the mixed-radix (Garner) reconstruction
    unsigned __int128 M = a.p[0];
    for (int i = 1; i < a.np; ++i) M *= a.p[i];
    const unsigned __int128 Mh = M / 2;
    Best b = best_init();
    int64_t lo = 0, hi = a.nout - 1;
    if (OUT == OUT_ARGMAX) { lo = a.am.t_lo; hi = a.am.t_hi; }
    for (int64_t t = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= hi;
         t += (int64_t)gridDim.x * blockDim.x) {
        unsigned __int128 x = R[t];
        unsigned __int128 Mi = a.p[0];
        for (int i = 1; i < a.np; ++i) {
            const uint64_t pi = a.p[i];
            const uint64_t xm = (uint64_t)(x % pi);
            const uint64_t ri = R[(int64_t)i * a.P + t];
            const uint64_t di = (ri + pi - xm) % pi;
            const uint64_t ai = (di * a.ginv[i]) % pi;
            x += (unsigned __int128)ai * Mi;
            Mi *= pi;
        }
        const long long v = x > Mh ? -(long long)(uint64_t)(M - x) : (long long)(uint64_t)x;
        if (OUT == OUT_VALUES) a.values[pair * a.vld + t] = v;
        else best_add(b, v, t);
    }
    if (OUT == OUT_ARGMAX) argmax_finish<kWarps>(b, a.am, a.stats, pair, gridDim.x, blockIdx.x);
}

// ------------------------------------------- large transforms (P > 2^19)
//
// P = M * Q with Q = 2^lq (<= 2^19, the four-step passes above) and
// M = 2^logm: element n at (i = n / Q, j = n % Q).
//   outer forward: per column j, M-point DIF over i (+ quantise), then
//                  x omega_P^(j*k1) -> rows [pos][j] = M independent Q-point
//                  sub-transforms (the inner passes 1-3, residue mode)
//   outer inverse: per column j, x omega_P^(-j*k1)/M, M-point DIT -> natural
//                  i, t = i*Q + j -> lift -> argmax / values / residues
// The per-element twiddle omega_P^e (e = j*k1 mod P) is the Montgomery
// product of two small tables, tl[e & 8191] * th[e >> 13].

struct OuterArgs {
    OperandDesc op[2];       // forward: the two signals
    uint32_t* out;           // forward: [op][pair][pos][Q]
    const uint32_t* rin;     // inverse: inner residues [pair*M + pos][np][Q]
    uint32_t* rout;          // inverse, multi-prime: [pair][np][P] for k_combine
    const uint2* rtw;        // omega_M^(+-t), t < M/2 (Shoup pairs): fwd rf / inv ri
    const uint32_t* tl;      // two-level twiddles (Montgomery form; inv: * 1/M)
    const uint32_t* th;
    const uint32_t* tlf;     // inverse: the forward two-level tables (omega_P^-j = omega_P^(P-j))
    const uint32_t* thf;
    const uint2* tc;         // per-thread factor of the column twiddles [r][tid] (OuterTables::tcf / tci)
    const uint2* uc;         // per-tile factor [tile][r] (OuterTables::ucf / uci)
    unsigned long long* stats;
    ArgmaxOut am;
    int64_t* values;
    int64_t nout, vld, batch;
    ModP m;
    uint32_t p0;
    int lq, np, pi, skip_cs, zero_upper;
    int64_t pair0;
};

__device__ __forceinline__ uint32_t tw_2level(const uint32_t* __restrict__ tl, const uint32_t* __restrict__ th,
                                              uint32_t e, const ModP& m)
{
    return redp(montmul(__ldg(&tl[e & 8191u]), __ldg(&th[e >> 13]), m.p, m.pinv), m.p);
}

// Outer M-point transforms of the large-P path, one thread per column j of
// the M x Q layout (element n = row * Q + j): the column's M <= 128
// residues stay in registers for the whole radix-2 transform, so there is no
// shared-memory exchange and no barrier; a warp's row accesses are 32
// consecutive words.  Stage twiddles omega_M^t come from a 64-entry table.
constexpr int kOuterThreads = 256;

// natural -> bit-reversed DIF (Gentleman-Sande); values in [0, 2p).  One
// template step per stage keeps every trip count a compile-time constant,
// so the whole column stays in registers.
template <int LOGM, int ST = 0>
__device__ __forceinline__ void dif_full(uint32_t (&x)[1 << LOGM], const uint2* tw, const ModP& m)
{
    if constexpr (ST < LOGM) {
        constexpr int M = 1 << LOGM, half = M >> (ST + 1);
#pragma unroll
        for (int b0 = 0; b0 < M; b0 += 2 * half)
#pragma unroll
            for (int i = 0; i < half; ++i) {
                uint32_t& u = x[b0 + i];
                uint32_t& v = x[b0 + i + half];
                if (i == 0) {
                    const uint32_t sm = u + v + m.zero, df = u - v + m.p2;
                    u = red2p(sm, m.p2);
                    v = red2p(df, m.p2);
                } else {
                    bfly_dif(u, v, tw[i << ST], m);
                }
            }
        dif_full<LOGM, ST + 1>(x, tw, m);
    }
}

// bit-reversed -> natural DIT (Cooley-Tukey); values in [0, 4p)
template <int LOGM, int ST = 0>
__device__ __forceinline__ void dit_full(uint32_t (&x)[1 << LOGM], const uint2* tw, const ModP& m)
{
    if constexpr (ST < LOGM) {
        constexpr int M = 1 << LOGM, half = 1 << ST;
#pragma unroll
        for (int b0 = 0; b0 < M; b0 += 2 * half)
#pragma unroll
            for (int i = 0; i < half; ++i) {
                uint32_t& u = x[b0 + i];
                uint32_t& v = x[b0 + i + half];
                if (i == 0) {
                    const uint32_t a0 = red2p(u, m.p2), t = red2p(v, m.p2);
                    u = a0 + t + m.zero;
                    v = a0 - t + m.p2;
                } else {
                    bfly_dit(u, v, tw[i << (LOGM - 1 - ST)], m);
                }
            }
        dit_full<LOGM, ST + 1>(x, tw, m);
    }
}

// Constant-geometry (Pease) forms of dif_full / dit_full with identical
// outputs: every stage pairs positions j and j + M/2 (DIF) or 2j and 2j + 1
// (DIT) and writes the other array, so one unrolled two-stage body serves
// every stage pair in a runtime loop.  The fully unrolled forms above are
// ~M/2 * log2(M) butterflies of straight-line code per kernel (the C4
// k_outer_fwd instance was 6.9K SASS instructions, instruction-fetch bound:
// no_instruction stalls); these are one loop body of 2 * M/2 butterflies.
// Stage s twiddle exponents: DIF (j >> s) << s, DIT (j >> (L-1-s)) << (L-1-s)
// (both checked against the standard forms in tools/ntt_model.py).
template <int LOGM>
__device__ __forceinline__ void dif_cg_stage(const uint32_t (&x)[1 << LOGM], uint32_t (&y)[1 << LOGM], int s,
                                             const uint2* tw, const ModP& m)
{
    constexpr int H = 1 << (LOGM - 1);
#pragma unroll
    for (int j = 0; j < H; ++j) {
        uint32_t u = x[j], v = x[j + H];
        bfly_dif(u, v, tw[(j >> s) << s], m);
        y[2 * j] = u;
        y[2 * j + 1] = v;
    }
}

template <int LOGM>
__device__ __forceinline__ void dit_cg_stage(const uint32_t (&x)[1 << LOGM], uint32_t (&y)[1 << LOGM], int s,
                                             const uint2* tw, const ModP& m)
{
    constexpr int H = 1 << (LOGM - 1);
    const int sh = LOGM - 1 - s;
#pragma unroll
    for (int j = 0; j < H; ++j) {
        uint32_t u = x[2 * j], v = x[2 * j + 1];
        bfly_dit(u, v, tw[(j >> sh) << sh], m);
        y[j] = u;
        y[j + H] = v;
    }
}

// natural -> bit-reversed DIF, values in [0, 2p); result in x
template <int LOGM>
__device__ __forceinline__ void dif_cg(uint32_t (&x)[1 << LOGM], const uint2* tw, const ModP& m)
{
    uint32_t y[1 << LOGM];
#pragma unroll 1
    for (int s = 0; s + 1 < LOGM; s += 2) {
        dif_cg_stage<LOGM>(x, y, s, tw, m);
        dif_cg_stage<LOGM>(y, x, s + 1, tw, m);
    }
    if constexpr (LOGM & 1) {
        dif_cg_stage<LOGM>(x, y, LOGM - 1, tw, m);
#pragma unroll
        for (int i = 0; i < (1 << LOGM); ++i) x[i] = y[i];
    }
}

// dif_cg for inputs whose upper half is zero (x[j + M/2] == 0): stage 0
// is a copy and one product per pair, the remaining stages as dif_cg
template <int LOGM>
__device__ __forceinline__ void dif_cg_zu(uint32_t (&x)[1 << LOGM], const uint2* tw, const ModP& m)
{
    constexpr int H = 1 << (LOGM - 1);
    uint32_t y[1 << LOGM];
#pragma unroll
    for (int j = 0; j < H; ++j) {  // (u, 0) -> (u, u * omega^j); inputs in [0, p)
        const uint2 w = tw[j];
        y[2 * j] = x[j];
        y[2 * j + 1] = shoup(x[j], w.x, w.y, m.p);
    }
#pragma unroll 1
    for (int s = 1; s + 1 < LOGM; s += 2) {
        dif_cg_stage<LOGM>(y, x, s, tw, m);
        dif_cg_stage<LOGM>(x, y, s + 1, tw, m);
    }
    if constexpr ((LOGM - 1) & 1) {
        dif_cg_stage<LOGM>(y, x, LOGM - 1, tw, m);
    } else {
#pragma unroll
        for (int i = 0; i < (1 << LOGM); ++i) x[i] = y[i];
    }
}

// bit-reversed -> natural DIT, values in [0, 4p); result in x
template <int LOGM>
__device__ __forceinline__ void dit_cg(uint32_t (&x)[1 << LOGM], const uint2* tw, const ModP& m)
{
    uint32_t y[1 << LOGM];
#pragma unroll 1
    for (int s = 0; s + 1 < LOGM; s += 2) {
        dit_cg_stage<LOGM>(x, y, s, tw, m);
        dit_cg_stage<LOGM>(y, x, s + 1, tw, m);
    }
    if constexpr (LOGM & 1) {
        dit_cg_stage<LOGM>(x, y, LOGM - 1, tw, m);
#pragma unroll
        for (int i = 0; i < (1 << LOGM); ++i) x[i] = y[i];
    }
}

constexpr int brev_c(int r, int bits)
{
    int o = 0;
    for (int i = 0; i < bits; ++i) o |= ((r >> i) & 1) << (bits - 1 - i);
    return o;
}

// Column j's four-step twiddles omega_P^(+-j k1), k1 = bitrev(r), r = 0..M-1.
// With j = j0 + tid (j0 = 256 tile, the tile's first column) the twiddle is
// U[tile][r] * T[r][tid]: two host-built tables of Shoup pairs.  U (times M^-1
// on the inverse; 1 MB at Q = 2^19, M = 64) is copied to shared memory per
// tile, T is a fixed M x 256 table (128 KB at M = 64, L1/L2 resident, read
// coalesced).  Two Shoup products per element (2 IMAD.HI) replace the running
// Montgomery product's two general products (4 IMAD.HI).
template <int LOGM>
__device__ __forceinline__ void apply_column_twiddles(uint32_t (&x)[1 << LOGM], const uint2* su,
                                                      const uint2* __restrict__ tc, const ModP& m)
{
    constexpr int M = 1 << LOGM, CH = 8;
    const uint2* t = tc + threadIdx.x;
    // the table reads go out CH at a time, the next batch under this batch's
    // products (all M at once cost 2M registers and half the occupancy)
    uint2 T[2][CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) T[0][i] = __ldg(t + i * kOuterThreads);
#pragma unroll
    for (int c = 0; c < M / CH; ++c) {
        if (c + 1 < M / CH) {
#pragma unroll
            for (int i = 0; i < CH; ++i) T[(c + 1) & 1][i] = __ldg(t + ((c + 1) * CH + i) * kOuterThreads);
        }
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            const int r = c * CH + i;
            const uint2 U = su[r];
            x[r] = shoup(shoup(x[r], T[c & 1][i].x, T[c & 1][i].y, m.p), U.x, U.y, m.p);
        }
    }
}

template <int LOGM, typename T, int QM, bool ZU>
__global__ void __launch_bounds__(kOuterThreads, (LOGM <= 6 && (sizeof(T) == 4 || ZU)) ? 2 : 1) k_outer_fwd(const __grid_constant__ OuterArgs a)
{
    constexpr int M = 1 << LOGM;
    constexpr int ROWS = ZU ? M / 2 : M;  // rows that can hold samples (ZU: the upper half is zero)
    constexpr int CH = 16;                // rows loaded ahead per batch
    constexpr int NCH = ROWS < CH ? 1 : ROWS / CH, CW = ROWS < CH ? ROWS : CH;
    __shared__ uint2 stw[M / 2];
    __shared__ uint2 su[M];
    __shared__ T sthr[kMaxThr];
    const int op = blockIdx.y;
    const int64_t pl = blockIdx.z, pair = a.pair0 + pl;
    if (a.skip_cs && cs_single(a.stats, pair, a.p0)) return;
    const OperandDesc& d = a.op[op];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < M / 2; i += kOuterThreads) stw[i] = a.rtw[i];
    for (int i = threadIdx.x; i < d.q.tsize; i += kOuterThreads) sthr[i] = (T)d.q.thr[i];
    const ModP m = a.m;
    const int Q = 1 << a.lq;
    if (threadIdx.x < M) su[threadIdx.x] = __ldg(&a.uc[(int64_t)blockIdx.x * M + threadIdx.x]);
    __syncthreads();
    const T t0 = sthr[0], t1 = sthr[1], inv_step = (T)d.q.inv_step;
    const int k = d.q.k, tbits = d.q.tbits;
    const int j = blockIdx.x * kOuterThreads + threadIdx.x;
    const int64_t n = d.n;
    // element r*Q + j of the (possibly reversed) row: base pointer + signed
    // stride; rows r < nrows exist (idx < n), the upper half is zero when
    // the host says so
    const T* src = reinterpret_cast<const T*>(d.data) + pair * d.ld + (d.reverse ? n - 1 - j : j);
    const int64_t stride = d.reverse ? -(int64_t)Q : (int64_t)Q;
    const int nrows = j < n ? (int)min((n - j + Q - 1) / Q, (int64_t)ROWS) : 0;
    unsigned ssq = 0, nnz = 0, flags = 0;
    uint32_t x[M];
    if constexpr (ZU) {
#pragma unroll
        for (int r = ROWS; r < M; ++r) x[r] = 0;
    }
    const T* rp = src;  // row pointer, advanced by `stride` per row
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        // all loads of the batch first (independent, coalesced across the warp)
        T v[CW];
        bool live[CW];
#pragma unroll
        for (int i = 0; i < CW; ++i) {
            const int r = ch * CW + i;
            live[i] = r < nrows;
            v[i] = live[i] ? __ldg(rp) : T(0);
            rp += stride;
        }
        int c[CW];
        if constexpr (QM == QM_UNIFORM && sizeof(T) == 4) {
            bool bad = false;
#pragma unroll
            for (int i = 0; i < CW; ++i) c[i] = level_uniform_nb((float)v[i], k, (float)inv_step, bad);
            if (__builtin_expect(bad, 0)) {
#pragma unroll
                for (int i = 0; i < CW; ++i) {
                    if (v[i] != v[i]) flags |= SF_NONFINITE;
                    c[i] = quant_level<T, QM>(v[i], sthr, k, tbits, inv_step, t0, t1);
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < CW; ++i) {
                if constexpr (QM == QM_CODES) {
                    const long long cc = (long long)v[i];
                    if (cc > k || cc < -k) flags |= SF_CODE_RANGE;
                    c[i] = (int)cc;
                } else {
                    if (v[i] != v[i]) flags |= SF_NONFINITE;
                    c[i] = quant_level<T, QM>(v[i], sthr, k, tbits, inv_step, t0, t1);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < CW; ++i) {
            const int cc = live[i] ? c[i] : 0;
            ssq += (unsigned)(cc * cc);
            nnz += (cc != 0);
            x[ch * CW + i] = cc < 0 ? (uint32_t)(cc + (int)m.p) : (uint32_t)cc;
        }
    }
    if constexpr (ZU) dif_cg_zu<LOGM>(x, stw, m);
    else dif_cg<LOGM>(x, stw, m);
    // register r holds frequency k1 = bitrev(r): x omega_P^(j k1) -> row r
    apply_column_twiddles<LOGM>(x, su, a.tc, m);
    uint32_t* out = a.out + ((int64_t)op * a.batch + pl) * ((int64_t)M << a.lq) + j;  // a.batch: chunk size
#pragma unroll
    for (int r = 0; r < M; ++r, out += Q) *out = x[r];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
        flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if (lane == 0 && a.p0 == m.p) {
        unsigned long long* st = a.stats + (pair * 2 + op) * 4;
        if (ssq) atomicAdd(st + 0, (unsigned long long)ssq);
        if (nnz) atomicAdd(st + 1, (unsigned long long)nnz);
        if (flags) atomicOr(st + 2, (unsigned long long)flags);
    }
}

template <int LOGM, int OUT>
__global__ void __launch_bounds__(kOuterThreads, LOGM <= 6 ? 2 : 1) k_outer_inv(const __grid_constant__ OuterArgs a)
{
    constexpr int M = 1 << LOGM;
    __shared__ uint2 stw[M / 2];
    __shared__ uint2 su[2][M];  // this tile's U and the next one's (copied a tile ahead)
    const int64_t pl = blockIdx.y, pair = a.pair0 + pl;
    const bool cs = (a.np > 1) && cs_single(a.stats, pair, a.p0);
    if (a.pi > 0 && cs) return;
    const bool final_out = (a.np == 1) || cs;
    for (int i = threadIdx.x; i < M / 2; i += kOuterThreads) stw[i] = a.rtw[i];
    if (threadIdx.x < M && (int)blockIdx.x < (1 << a.lq) / kOuterThreads)
        su[0][threadIdx.x] = __ldg(&a.uc[(int64_t)blockIdx.x * M + threadIdx.x]);
    int cur = 0;
    const int Q = 1 << a.lq;
    const ModP m = a.m;
    const uint32_t half = (m.p - 1) / 2;
    const int64_t P = (int64_t)M << a.lq;
    // window in t (t = r*Q + j < P <= 2^26 and |value| < 2^29: 32-bit scan)
    const int tlo = (int)max(a.am.t_lo, (int64_t)0), thi = (int)min(a.am.t_hi, P - 1);
    // Fused argmax as in k_pass3: + half at the column's DC input makes every
    // output c + half, whose canonical residue is a monotone key of c; the warp
    // shares one running best key wm, kept as key + 1 (0: nothing in the window
    // yet); bc / bt are this lane's count and smallest index at wm.
    const uint32_t bias = (OUT == OUT_ARGMAX && final_out) ? half : 0u;
    uint32_t wm = 0;
    int bt = INT_MAX, bc = 0;
    // column tiles strided over the (<= kMaxPartialsLarge) CTAs of this pair
#pragma unroll 1
    for (int tile = blockIdx.x; tile < Q / kOuterThreads; tile += gridDim.x) {
        const int j = tile * kOuterThreads + threadIdx.x;
        // one barrier per tile: su[cur] (and stw) are visible, and every warp is
        // done with su[cur ^ 1], which now takes the next tile's U
        __syncthreads();
        const int nxt = tile + gridDim.x;
        if (threadIdx.x < M && nxt < Q / kOuterThreads)
            su[cur ^ 1][threadIdx.x] = __ldg(&a.uc[(int64_t)nxt * M + threadIdx.x]);
        uint32_t x[M];
        const uint32_t* rin = a.rin + ((int64_t)pl * M * a.np + a.pi) * Q + j;
        const int64_t rstep = (int64_t)a.np * Q;
        if (nxt < Q / kOuterThreads) {
            // the next tile's rows (this warp's 128-byte segment of each) into L2 under this tile's work
            const uint32_t* pn = rin - (threadIdx.x & 31) + (int64_t)gridDim.x * kOuterThreads;
            for (int r = threadIdx.x & 31; r < M; r += 32) prefetch_l2(pn + r * rstep);
        }
#pragma unroll
        for (int r = 0; r < M; ++r, rin += rstep) x[r] = __ldg(rin);
        // inner results of sub-transform r are frequency k1 = bitrev(r):
        // x M^-1 omega_P^(-j k1)
        apply_column_twiddles<LOGM>(x, su[cur], a.tc, m);
        cur ^= 1;
        x[0] += bias;  // register 0 is frequency 0 (inputs stay below 4p: < 2p + p/2)
        dit_cg<LOGM>(x, stw, m);
        if (!final_out) {
            uint32_t* ro = a.rout + (pl * a.np + a.pi) * P + j;
#pragma unroll
            for (int r = 0; r < M; ++r) ro[(int64_t)r * Q] = redp(red2p(x[r], m.p2), m.p);
        } else if constexpr (OUT == OUT_VALUES) {
#pragma unroll
            for (int r = 0; r < M; ++r) {
                const int64_t t = (int64_t)r * Q + j;
                const uint32_t v = redp(red2p(x[r], m.p2), m.p);
                if (t < a.nout) a.values[pair * a.vld + t] = (long long)v - (v > half ? (long long)m.p : 0);
            }
        } else {
            // a tile inside the window holds plain keys (off = 1 maps them to the
            // key + 1 scale of wm); a tile on a window edge holds key + 1 with 0 for
            // out-of-window elements, which never equal a scan target >= 1
            const int jmin = tile * kOuterThreads;
            const bool inside = tlo <= jmin && thi >= (M - 1) * Q + jmin + kOuterThreads - 1;
            const uint32_t off = inside ? 1u : 0u;
#pragma unroll
            for (int r = 0; r < M; ++r) x[r] = redp(red2p(x[r], m.p2), m.p);
            if (!inside) {
#pragma unroll
                for (int r = 0; r < M; ++r) {
                    const int t = r * Q + j;
                    x[r] = (t < tlo || t > thi) ? 0u : x[r] + 1u;
                }
            }
            uint32_t mx = x[0];
#pragma unroll
            for (int r = 1; r + 1 < M; r += 2) mx = __vimax3_u32(mx, x[r], x[r + 1]);
            mx = max(mx, x[M - 1]);
            const uint32_t mu = mx + off;
            if (__any_sync(0xffffffffu, mu >= wm && mu > 0u)) {
                const uint32_t wn = __reduce_max_sync(0xffffffffu, mu);
                if (wn > wm) {
                    wm = wn;
                    bc = 0;
                    bt = INT_MAX;
                }
                // t increases with r inside a tile; across a thread's tiles it does not
                const uint32_t target = wm - off;
                int rb = M;
#pragma unroll
                for (int r = M - 1; r >= 0; --r) {
                    if (x[r] == target && (inside || target > 0u)) {
                        ++bc;
                        rb = r;
                    }
                }
                if (rb < M) bt = min(bt, rb * Q + j);
            }
        }
    }
    if constexpr (OUT == OUT_ARGMAX) {
        if (final_out) {
            const Best b = bc ? Best{(long long)(wm - 1u) - (long long)half, bt, bc} : best_init();
            argmax_finish<kWarps>(b, a.am, a.stats, pair, gridDim.x, blockIdx.x);
        }
    }
}

// ================================================================== host

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (unsigned __int128)a * b % p; }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t p)
{
    uint64_t r = 1;
    a %= p;
    while (e) {
        if (e & 1) r = mulmod(r, a, p);
        a = mulmod(a, a, p);
        e >>= 1;
    }
    return r;
}
static uint32_t bitrev(uint32_t x, int bits)
{
    uint32_t r = 0;
    for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
    return r;
}

// group twiddle blocks of a length-2^LOG transform (layout: Sched)
template <int LOG>
static void group_tables(uint64_t root, uint64_t p, std::vector<uint2>& dif, std::vector<uint2>& dit)
{
    using SC = Sched<LOG>;
    const uint64_t iroot = powmod(root, p - 2, p);
    auto sh = [&](uint64_t v) { return make_uint2((uint32_t)v, (uint32_t)((v << 32) / p)); };
    dif.assign(SC::TW_DIF, make_uint2(0, 0));
    dit.assign(SC::TW_DIT, make_uint2(0, 0));
    for (int i = 0; i < SC::NG; ++i) {
        const int R = SC::r(i), S0 = SC::s0(i), S = SC::L >> (S0 + R);
        for (int j0 = 0; j0 < SC::nj_dif(i); ++j0)
            for (int t = 0; t < R; ++t)
                for (int kp = 0; kp < (1 << (R - 1 - t)); ++kp) {
                    const uint64_t e = (uint64_t)(j0 + kp * S) << (S0 + t);
                    dif[SC::twoff_dif(i) + j0 * (1 << R) + (1 << R) - (1 << (R - t)) + kp] = sh(powmod(root, e, p));
                }
    }
    for (int i = 0; i < SC::NG; ++i) {
        const int R = SC::rd(i), S0 = SC::s0d(i);
        for (int j0 = 0; j0 < SC::nj_dit(i); ++j0)
            for (int t = 0; t < R; ++t)
                for (int kp = 0; kp < (1 << t); ++kp) {
                    const uint64_t e = (uint64_t)(j0 + (kp << S0)) << (LOG - S0 - t - 1);
                    dit[SC::twoff_dit(i) + j0 * (1 << R) + (1 << t) - 1 + kp] = sh(powmod(iroot, e, p));
                }
    }
}

static void group_tables_rt(int log, uint64_t root, uint64_t p, std::vector<uint2>& f, std::vector<uint2>& i)
{
    switch (log) {
    case 3: group_tables<3>(root, p, f, i); break;
    case 4: group_tables<4>(root, p, f, i); break;
    case 5: group_tables<5>(root, p, f, i); break;
    case 6: group_tables<6>(root, p, f, i); break;
    case 7: group_tables<7>(root, p, f, i); break;
    case 8: group_tables<8>(root, p, f, i); break;
    case 9: group_tables<9>(root, p, f, i); break;
    case 10: group_tables<10>(root, p, f, i); break;
    }
}

cudaError_t ntt_make_tables(uint32_t p, uint32_t g, int lp, NttTables* out, void** dev_block)
{
    const int l1 = (lp + 1) / 2, l2 = lp / 2;
    const uint64_t P = 1ull << lp, N1 = 1ull << l1, N2 = 1ull << l2;
    const uint64_t w = powmod(g, (p - 1) >> lp, p), wi = powmod(w, p - 2, p);
    const uint64_t R = (1ull << 32) % p;
    const uint64_t invP = powmod(P, p - 2, p);
    std::vector<uint2> g1f, g1i, g2f, g2i;
    group_tables_rt(l1, powmod(w, N2, p), p, g1f, g1i);
    group_tables_rt(l2, powmod(w, N1, p), p, g2f, g2i);
    // layout: g1f | g1i | g2f | g2i | twf | twi  (each table 16-byte aligned)
    auto al = [](size_t n) { return (n + 1) & ~(size_t)1; };
    const size_t nt = al(g1f.size()) + al(g1i.size()) + al(g2f.size()) + al(g2i.size());
    // factored forward four-step twiddles (N1 >= 32): position pos = lane + 32 j has
    // bitrev(pos) = bitrev5(lane) << (l1 - 5) | bitrev(j), so w^(n2 bitrev(pos)) =
    // A[n2][lane] * B[n2][j] -- per n2 the 32 A then the N1/32 B (Shoup pairs)
    const uint64_t nab = N1 >= 32 ? 32 + N1 / 32 : 0;
    // and the inverse ones of pass 2: row pos, n2 = lane + 32 j:
    // ci wi^(k1 n2) = (ci wi^(k1 lane)) * wi^(32 k1 j) -- per row 32 A then N2/32 B
    const uint64_t nib = N2 >= 32 ? 32 + N2 / 32 : 0;
    const size_t bytes = nt * sizeof(uint2) + 2 * P * sizeof(uint2) + N2 * nab * sizeof(uint2) +
                         N1 * nib * sizeof(uint2);
    std::vector<unsigned char> host(bytes, 0);
    uint2* h = reinterpret_cast<uint2*>(host.data());
    size_t o1i = al(g1f.size()), o2f = o1i + al(g1i.size()), o2i = o2f + al(g2f.size());
    memcpy(h, g1f.data(), g1f.size() * 8);
    memcpy(h + o1i, g1i.data(), g1i.size() * 8);
    memcpy(h + o2f, g2f.data(), g2f.size() * 8);
    memcpy(h + o2i, g2i.data(), g2i.size() * 8);
    uint2* hf = h + nt;
    uint2* hi = hf + P;
    auto sh = [p](uint64_t v) { return make_uint2((uint32_t)v, (uint32_t)((v << 32) / p)); };
    const uint64_t ci = mulmod(invP, R, p);  // R cancels the pointwise montmul's R^-1
    for (uint64_t pos = 0; pos < N1; ++pos) {
        const uint64_t k1 = bitrev((uint32_t)pos, l1);
        const uint64_t step_f = powmod(w, k1, p), step_i = powmod(wi, k1, p);
        uint64_t f = 1, iv = ci;  // n2 = 0
        for (uint64_t n2 = 0; n2 < N2; ++n2) {
            hf[n2 * N1 + pos] = sh(f);
            hi[pos * N2 + n2] = sh(iv);
            f = mulmod(f, step_f, p);
            iv = mulmod(iv, step_i, p);
        }
    }
    uint2* hab = hi + P;
    for (uint64_t n2 = 0; n2 < N2 && nab; ++n2) {
        for (uint64_t l = 0; l < 32; ++l) hab[n2 * nab + l] = hf[n2 * N1 + l];
        for (uint64_t j = 0; j < N1 / 32; ++j) hab[n2 * nab + 32 + j] = hf[n2 * N1 + 32 * j];
    }
    uint2* hib = hab + N2 * nab;
    for (uint64_t pos = 0; pos < N1 && nib; ++pos) {
        const uint64_t k1 = bitrev((uint32_t)pos, l1);
        for (uint64_t l = 0; l < 32; ++l) hib[pos * nib + l] = hi[pos * N2 + l];
        const uint64_t st = powmod(wi, (32 * k1) % P, p);
        uint64_t b = 1;
        for (uint64_t j = 0; j < N2 / 32; ++j, b = mulmod(b, st, p)) hib[pos * nib + 32 + j] = sh(b);
    }
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, bytes);
    if (e != cudaSuccess) return e;
    e = cudaMemcpy(d, host.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(d); return e; }
    uint2* db = reinterpret_cast<uint2*>(d);
    out->p = p;
    out->m.p = p;
    out->m.p2 = 2 * p;
    uint32_t inv = 1;  // p^-1 mod 2^32 by Newton
    for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
    out->m.pinv = inv;
    out->m.zero = 0;
    out->lp = lp;
    out->l1 = l1;
    out->l2 = l2;
    out->g1f = db;
    out->g1i = db + o1i;
    out->g2f = db + o2f;
    out->g2i = db + o2i;
    out->twf = db + nt;
    out->twi = out->twf + P;
    out->twab = nab ? out->twi + P : nullptr;
    out->twib = nib ? out->twi + P + N2 * nab : nullptr;
    *dev_block = d;
    return cudaSuccess;
}

cudaError_t ntt_make_outer_tables(uint32_t p, uint32_t g, int lp, int logm, OuterTables* out, void** dev_block)
{
    const uint64_t P = 1ull << lp, M = 1ull << logm, Q = P >> logm;
    const uint64_t w = powmod(g, (p - 1) >> lp, p), wi = powmod(w, p - 2, p);
    const uint64_t R = (1ull << 32) % p;
    const uint64_t invM = powmod(M, p - 2, p);
    std::vector<uint2> gf, gi;
    group_tables_rt(logm, powmod(w, Q, p), p, gf, gi);
    const size_t nl = 8192, nh = (size_t)(P / 8192 > 0 ? P / 8192 : 1);
    auto al = [](size_t n) { return (n + 3) & ~(size_t)3; };
    const size_t ng = al(gf.size()) + al(gi.size());  // in uint2 units
    const size_t nr = al(M / 2);                      // uint2 units, each of rf / ri
    const size_t ntc = (size_t)M * kOuterThreads;  // uint2 units, each of tcf / tci
    const size_t ntile = (size_t)(Q / kOuterThreads > 0 ? Q / kOuterThreads : 1);
    const size_t nuc = ntile * M;                  // uint2 units, each of ucf / uci
    const size_t words = 2 * ng + 2 * al(nl) + 2 * al(nh) + 4 * nr + 4 * ntc + 4 * nuc;
    std::vector<uint32_t> h(words, 0);
    memcpy(h.data(), gf.data(), gf.size() * 8);
    memcpy(h.data() + 2 * al(gf.size()), gi.data(), gi.size() * 8);
    uint32_t* tl = h.data() + 2 * ng;
    uint32_t* tli = tl + al(nl);
    uint32_t* th = tli + al(nl);
    uint32_t* thi = th + al(nh);
    const uint64_t w8k = powmod(w, 8192, p), wi8k = powmod(wi, 8192, p);
    for (uint64_t a = 0, f = R, iv = mulmod(invM, R, p); a < nl; ++a, f = mulmod(f, w, p), iv = mulmod(iv, wi, p)) {
        tl[a] = (uint32_t)f;
        tli[a] = (uint32_t)iv;
    }
    for (uint64_t b = 0, f = R, iv = R; b < nh; ++b, f = mulmod(f, w8k, p), iv = mulmod(iv, wi8k, p)) {
        th[b] = (uint32_t)f;
        thi[b] = (uint32_t)iv;
    }
    // omega_M^t and omega_M^-t, t < M/2, as Shoup pairs (w, floor(w 2^32 / p))
    uint32_t* rf = thi + al(nh);
    uint32_t* ri = rf + 2 * nr;
    const uint64_t wm = powmod(w, Q, p), wmi = powmod(wm, p - 2, p);
    for (uint64_t t = 0, f = 1, iv = 1; t < M / 2; ++t, f = mulmod(f, wm, p), iv = mulmod(iv, wmi, p)) {
        rf[2 * t] = (uint32_t)f;
        rf[2 * t + 1] = (uint32_t)((f << 32) / p);
        ri[2 * t] = (uint32_t)iv;
        ri[2 * t + 1] = (uint32_t)((iv << 32) / p);
    }
    // per-thread factors of the column twiddles: omega_P^(+-tid k1), k1 = bitrev(r)
    uint32_t* tcf = ri + 2 * nr;
    uint32_t* tci = tcf + 2 * ntc;
    for (uint64_t r = 0; r < M; ++r) {
        const uint64_t k1 = bitrev((uint32_t)r, logm);
        const uint64_t sf = powmod(w, k1, p), si = powmod(wi, k1, p);
        for (uint64_t t = 0, f = 1, iv = 1; t < (uint64_t)kOuterThreads; ++t, f = mulmod(f, sf, p), iv = mulmod(iv, si, p)) {
            const size_t o = 2 * (r * kOuterThreads + t);
            tcf[o] = (uint32_t)f;
            tcf[o + 1] = (uint32_t)((f << 32) / p);
            tci[o] = (uint32_t)iv;
            tci[o + 1] = (uint32_t)((iv << 32) / p);
        }
    }
    // per-tile factors: omega_P^(+-256 tile k1), the inverse one times M^-1
    uint32_t* ucf = tci + 2 * ntc;
    uint32_t* uci = ucf + 2 * nuc;
    for (uint64_t r = 0; r < M; ++r) {
        const uint64_t k1 = bitrev((uint32_t)r, logm);
        const uint64_t sf = powmod(w, (k1 * kOuterThreads) % P, p), si = powmod(wi, (k1 * kOuterThreads) % P, p);
        for (uint64_t t = 0, f = 1, iv = invM; t < ntile; ++t, f = mulmod(f, sf, p), iv = mulmod(iv, si, p)) {
            const size_t o = 2 * (t * M + r);
            ucf[o] = (uint32_t)f;
            ucf[o + 1] = (uint32_t)((f << 32) / p);
            uci[o] = (uint32_t)iv;
            uci[o + 1] = (uint32_t)((iv << 32) / p);
        }
    }
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, words * 4);
    if (e != cudaSuccess) return e;
    e = cudaMemcpy(d, h.data(), words * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(d); return e; }
    const uint32_t* dw = reinterpret_cast<const uint32_t*>(d);
    out->ucf = reinterpret_cast<const uint2*>(dw + (ucf - h.data()));
    out->uci = reinterpret_cast<const uint2*>(dw + (uci - h.data()));
    out->tcf = reinterpret_cast<const uint2*>(dw + (tcf - h.data()));
    out->tci = reinterpret_cast<const uint2*>(dw + (tci - h.data()));
    out->rf = reinterpret_cast<const uint2*>(dw + (rf - h.data()));
    out->ri = reinterpret_cast<const uint2*>(dw + (ri - h.data()));
    out->gf = reinterpret_cast<const uint2*>(dw);
    out->gi = reinterpret_cast<const uint2*>(dw + 2 * al(gf.size()));
    out->tl = dw + 2 * ng;
    out->tli = out->tl + al(nl);
    out->th = out->tli + al(nl);
    out->thi = out->th + al(nh);
    *dev_block = d;
    return cudaSuccess;
}

// ---- kernel dispatch tables

template <int LOG1, typename T, int QM, bool ZU>
static cudaError_t launch_p1(const Pass1Args& a, dim3 grid, cudaStream_t s)
{
    const size_t smem = pass1_smem<LOG1>(sizeof(T));
    if (cudaError_t e = set_max_smem((const void*)k_pass1<LOG1, T, QM, ZU>, smem); e != cudaSuccess) return e;
    k_pass1<LOG1, T, QM, ZU><<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int LOG1, bool ZU>
static cudaError_t dispatch_p1_zu(const Pass1Args& a, int dtype, int qm, dim3 grid, cudaStream_t s)
{
#ifdef QX_NTT_DEV  // fast A/B builds (tools/build_variant.sh): float32 K1/uniform and residues only
    if (dtype == DT_U32) return launch_p1<LOG1, uint32_t, QM_RESIDUE, ZU>(a, grid, s);
    if (dtype == DT_F32 && qm == QM_K1) return launch_p1<LOG1, float, QM_K1, ZU>(a, grid, s);
    if (dtype == DT_F32 && qm == QM_UNIFORM) return launch_p1<LOG1, float, QM_UNIFORM, ZU>(a, grid, s);
    return cudaErrorInvalidValue;
#else
    if (dtype == DT_U32) return launch_p1<LOG1, uint32_t, QM_RESIDUE, ZU>(a, grid, s);
    if (dtype == DT_I64) return launch_p1<LOG1, long long, QM_CODES, ZU>(a, grid, s);
    if (dtype == DT_F32) {
        if (qm == QM_K1) return launch_p1<LOG1, float, QM_K1, ZU>(a, grid, s);
        if (qm == QM_UNIFORM) return launch_p1<LOG1, float, QM_UNIFORM, ZU>(a, grid, s);
        return launch_p1<LOG1, float, QM_BSEARCH, ZU>(a, grid, s);
    }
    if (qm == QM_K1) return launch_p1<LOG1, double, QM_K1, ZU>(a, grid, s);
    if (qm == QM_UNIFORM) return launch_p1<LOG1, double, QM_UNIFORM, ZU>(a, grid, s);
    return launch_p1<LOG1, double, QM_BSEARCH, ZU>(a, grid, s);
#endif
}

template <int LOG1>
static cudaError_t dispatch_p1_mode(const Pass1Args& a, int dtype, int qm, dim3 grid, cudaStream_t s)
{
    return a.zero_upper ? dispatch_p1_zu<LOG1, true>(a, dtype, qm, grid, s)
                        : dispatch_p1_zu<LOG1, false>(a, dtype, qm, grid, s);
}

static cudaError_t dispatch_p1(int log1, const Pass1Args& a, int dtype, int qm, dim3 grid, cudaStream_t s)
{
    switch (log1) {
#ifndef QX_NTT_DEV
    case 5: return dispatch_p1_mode<5>(a, dtype, qm, grid, s);
    case 6: return dispatch_p1_mode<6>(a, dtype, qm, grid, s);
    case 7: return dispatch_p1_mode<7>(a, dtype, qm, grid, s);
    case 8: return dispatch_p1_mode<8>(a, dtype, qm, grid, s);
    case 9: return dispatch_p1_mode<9>(a, dtype, qm, grid, s);
#endif
    case 10: return dispatch_p1_mode<10>(a, dtype, qm, grid, s);
    }
    return cudaErrorInvalidValue;
}

template <int LOG2>
static cudaError_t launch_p2(const Pass2Args& a, dim3 grid, cudaStream_t s)
{
    const size_t smem = pass2_smem<LOG2>();
    if (cudaError_t e = set_max_smem((const void*)k_pass2<LOG2>, smem); e != cudaSuccess) return e;
    k_pass2<LOG2><<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

static cudaError_t dispatch_p2(int log2, const Pass2Args& a, dim3 grid, cudaStream_t s)
{
    switch (log2) {
#ifndef QX_NTT_DEV
    case 5: return launch_p2<5>(a, grid, s);
    case 6: return launch_p2<6>(a, grid, s);
    case 7: return launch_p2<7>(a, grid, s);
    case 8: return launch_p2<8>(a, grid, s);
#endif
    case 9: return launch_p2<9>(a, grid, s);
    }
    return cudaErrorInvalidValue;
}

template <int LOG1, int OUT>
static cudaError_t launch_p3(const Pass3Args& a, dim3 grid, cudaStream_t s)
{
    const size_t smem = pass3_smem<LOG1>();
    if (cudaError_t e = set_max_smem((const void*)k_pass3<LOG1, OUT>, smem); e != cudaSuccess) return e;
    k_pass3<LOG1, OUT><<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int OUT>
static cudaError_t dispatch_p3_out(int log1, const Pass3Args& a, dim3 grid, cudaStream_t s)
{
    switch (log1) {
#ifndef QX_NTT_DEV
    case 5: return launch_p3<5, OUT>(a, grid, s);
    case 6: return launch_p3<6, OUT>(a, grid, s);
    case 7: return launch_p3<7, OUT>(a, grid, s);
    case 8: return launch_p3<8, OUT>(a, grid, s);
    case 9: return launch_p3<9, OUT>(a, grid, s);
#endif
    case 10: return launch_p3<10, OUT>(a, grid, s);
    }
    return cudaErrorInvalidValue;
}

void Profiler::pre(int kind, cudaStream_t s)
{
    if (!on) return;
    ++launches;
    ++count[kind];
    if (!timed) return;
    if (nrec == cap) {
        int ncap = cap ? 2 * cap : 256;
        Rec* n = new Rec[ncap];
        for (int i = 0; i < nrec; ++i) n[i] = recs[i];
        for (int i = nrec; i < ncap; ++i) {
            n[i].a = n[i].b = nullptr;
        }
        delete[] recs;
        recs = n;
        cap = ncap;
    }
    Rec& r = recs[nrec];
    if (!r.a) {
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
    }
    r.kind = kind;
    cudaEventRecord(r.a, s);
}

void Profiler::post(int kind, cudaStream_t s)
{
    if (!on || !timed) return;
    (void)kind;
    cudaEventRecord(recs[nrec].b, s);
    ++nrec;
}

template <int LOGM, typename T, int QM>
static cudaError_t launch_ofwd(const OuterArgs& a, dim3 grid, cudaStream_t s)
{
    if (a.zero_upper) k_outer_fwd<LOGM, T, QM, true><<<grid, kOuterThreads, 0, s>>>(a);
    else k_outer_fwd<LOGM, T, QM, false><<<grid, kOuterThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int LOGM>
static cudaError_t dispatch_ofwd_m(const OuterArgs& a, int dtype, int qm, dim3 grid, cudaStream_t s)
{
    if (dtype == DT_I64) return launch_ofwd<LOGM, long long, QM_CODES>(a, grid, s);
    if (dtype == DT_F32) {
        if (qm == QM_K1) return launch_ofwd<LOGM, float, QM_K1>(a, grid, s);
        if (qm == QM_UNIFORM) return launch_ofwd<LOGM, float, QM_UNIFORM>(a, grid, s);
        return launch_ofwd<LOGM, float, QM_BSEARCH>(a, grid, s);
    }
    if (qm == QM_K1) return launch_ofwd<LOGM, double, QM_K1>(a, grid, s);
    if (qm == QM_UNIFORM) return launch_ofwd<LOGM, double, QM_UNIFORM>(a, grid, s);
    return launch_ofwd<LOGM, double, QM_BSEARCH>(a, grid, s);
}

static cudaError_t dispatch_ofwd(int logm, const OuterArgs& a, int dtype, int qm, dim3 grid, cudaStream_t s)
{
    switch (logm) {
#ifndef QX_NTT_DEV
    case 3: return dispatch_ofwd_m<3>(a, dtype, qm, grid, s);
    case 4: return dispatch_ofwd_m<4>(a, dtype, qm, grid, s);
    case 5: return dispatch_ofwd_m<5>(a, dtype, qm, grid, s);
#endif
    case 6: return dispatch_ofwd_m<6>(a, dtype, qm, grid, s);
    case 7: return dispatch_ofwd_m<7>(a, dtype, qm, grid, s);
    }
    return cudaErrorInvalidValue;
}

template <int LOGM, int OUT>
static cudaError_t launch_oinv(const OuterArgs& a, dim3 grid, cudaStream_t s)
{
    k_outer_inv<LOGM, OUT><<<grid, kOuterThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int OUT>
static cudaError_t dispatch_oinv(int logm, const OuterArgs& a, dim3 grid, cudaStream_t s)
{
    switch (logm) {
#ifndef QX_NTT_DEV
    case 3: return launch_oinv<3, OUT>(a, grid, s);
    case 4: return launch_oinv<4, OUT>(a, grid, s);
    case 5: return launch_oinv<5, OUT>(a, grid, s);
#endif
    case 6: return launch_oinv<6, OUT>(a, grid, s);
    case 7: return launch_oinv<7, OUT>(a, grid, s);
    }
    return cudaErrorInvalidValue;
}

// P = 2^(logm + lq) > 2^19: outer forward pass (quantise + M-point DIF + twiddle)
// per operand, the three four-step passes on the chunk*M inner sub-transforms
// (residue mode), the outer inverse pass (twiddle + M-point DIT + lift +
// argmax/values), and the CRT combine for pairs that need more primes.
static cudaError_t ntt_run_large(const NttCall& c, cudaStream_t s)
{
    const int logm = c.logm, lq = c.lq, M = 1 << logm, Q = 1 << lq;
    const int64_t P = (int64_t)M * Q;
    const NttTables& t0 = c.tab[0];
    const int l1 = t0.l1, l2 = t0.l2, N1 = 1 << l1, N2 = 1 << l2;
    const bool argmax = c.am.results != nullptr;
    cudaError_t e;
    for (int64_t p0 = 0; p0 < c.batch; p0 += c.chunk) {
        const int64_t nb = (c.batch - p0 < c.chunk) ? c.batch - p0 : c.chunk;
        const int64_t nin = nb * M;  // inner sub-transforms in this chunk
        for (int pi = 0; pi < c.np; ++pi) {
            const NttTables& T = c.tab[pi];
            const OuterTables& O = c.otab[pi];
            OuterArgs oa;
            memset(&oa, 0, sizeof(oa));
            oa.op[0] = c.op[0];
            oa.op[1] = c.op[1];
            oa.out = c.OUT;
            oa.rtw = O.rf;
            oa.tl = O.tl;
            oa.th = O.th;
            oa.tc = O.tcf;
            oa.uc = O.ucf;
            oa.stats = c.stats;
            oa.batch = nb;
            oa.m = T.m;
            oa.p0 = t0.p;
            oa.lq = lq;
            oa.np = c.np;
            oa.pi = pi;
            oa.skip_cs = pi > 0;
            oa.zero_upper = c.zero_upper;
            oa.pair0 = p0;
            if (c.op[0].dtype != c.op[1].dtype || c.op[0].q.mode != c.op[1].q.mode) return cudaErrorInvalidValue;
            if (c.prof) c.prof->pre(KK_OTHER, s);
            e = dispatch_ofwd(logm, oa, c.op[0].dtype, c.op[0].q.mode, dim3(Q / kOuterThreads, 2, (unsigned)nb), s);
            if (c.prof) c.prof->post(KK_OTHER, s);
            if (e != cudaSuccess) return e;
            // inner forward (residues in), product, inverse -> residues
            Pass1Args a1;
            memset(&a1, 0, sizeof(a1));
            for (int op = 0; op < 2; ++op) {
                a1.op[op].data = c.OUT + (int64_t)op * nb * P;
                a1.op[op].ld = Q;
                a1.op[op].n = Q;
                a1.op[op].reverse = 0;
                a1.op[op].dtype = DT_U32;
                a1.op[op].q.mode = QM_RESIDUE;
            }
            a1.Y = c.Y;
            a1.gtw = T.g1f;
            a1.twf = T.twf;
            a1.twab = T.twab;
            a1.stats = c.stats;
            a1.m = T.m;
            a1.p0 = t0.p;
            a1.N2 = N2;
            a1.skip_cs = pi > 0;
            a1.pair_shift = logm;
            a1.pair0 = p0 * M;
            a1.row0 = p0 * M;
            if (c.prof) c.prof->pre(KK_PASS1, s);
            e = dispatch_p1(l1, a1, DT_U32, QM_RESIDUE, dim3(N2 / 32, 2, (unsigned)nin), s);
            if (c.prof) c.prof->post(KK_PASS1, s);
            if (e != cudaSuccess) return e;
            Pass2Args a2;
            memset(&a2, 0, sizeof(a2));
            a2.Y = c.Y;
            a2.Z = c.Z;
            a2.gtwf = T.g2f;
            a2.gtwi = T.g2i;
            a2.twinv = T.twi;
            a2.twib = T.twib;
            a2.stats = c.stats;
            a2.m = T.m;
            a2.p0 = t0.p;
            a2.N1 = N1;
            a2.skip_cs = pi > 0;
            a2.pair_shift = logm;
            a2.pair0 = p0 * M;
            if (c.prof) c.prof->pre(KK_PASS2, s);
            e = dispatch_p2(l2, a2, dim3(N1 / 32, (unsigned)nin), s);
            if (c.prof) c.prof->post(KK_PASS2, s);
            if (e != cudaSuccess) return e;
            Pass3Args a3;
            memset(&a3, 0, sizeof(a3));
            a3.Z = c.Z;
            a3.R = c.RI;
            a3.gtwi = T.g1i;
            a3.stats = c.stats;
            a3.am = c.am;
            a3.nout = Q;
            a3.m = T.m;
            a3.p0 = t0.p;
            a3.N2 = N2;
            a3.np = c.np;
            a3.pi = pi;
            a3.pair_shift = logm;
            a3.force_residue = 1;
            a3.pair0 = p0 * M;
            if (c.prof) c.prof->pre(KK_PASS3, s);
            e = dispatch_p3_out<OUT_VALUES>(l1, a3, dim3(N2 / 32, (unsigned)nin), s);
            if (c.prof) c.prof->post(KK_PASS3, s);
            if (e != cudaSuccess) return e;
            // outer inverse
            OuterArgs ob = oa;
            ob.rin = c.RI;
            ob.rout = c.R;
            ob.rtw = O.ri;
            ob.tlf = O.tl;
            ob.thf = O.th;
            ob.tl = O.tli;
            ob.th = O.thi;
            ob.tc = O.tci;
            ob.uc = O.uci;
            ob.am = c.am;
            ob.values = c.values;
            ob.nout = c.nout;
            ob.vld = c.nout;
            const int nblk = (Q / kOuterThreads) < kMaxPartialsLarge ? (Q / kOuterThreads) : kMaxPartialsLarge;
            if (c.prof) c.prof->pre(KK_OTHER, s);
            e = argmax ? dispatch_oinv<OUT_ARGMAX>(logm, ob, dim3(nblk, (unsigned)nb), s)
                       : dispatch_oinv<OUT_VALUES>(logm, ob, dim3(nblk, (unsigned)nb), s);
            if (c.prof) c.prof->post(KK_OTHER, s);
            if (e != cudaSuccess) return e;
        }
        if (c.np > 1) {
            CombineArgs ca;
            memset(&ca, 0, sizeof(ca));
            ca.R = c.R;
            ca.stats = c.stats;
            ca.am = c.am;
            ca.values = c.values;
            ca.nout = c.nout;
            ca.vld = c.nout;
            ca.P = P;
            for (int i = 0; i < c.np; ++i) {
                ca.p[i] = c.tab[i].p;
                ca.ginv[i] = c.garner_inv[i];
            }
            ca.p0 = t0.p;
            ca.np = c.np;
            ca.pair0 = p0;
            if (c.prof) c.prof->pre(KK_COMBINE, s);
            if (argmax) k_combine<OUT_ARGMAX><<<dim3(kMaxPartials, (unsigned)nb), 256, 0, s>>>(ca);
            else k_combine<OUT_VALUES><<<dim3(kMaxPartials, (unsigned)nb), 256, 0, s>>>(ca);
            e = cudaGetLastError();
            if (c.prof) c.prof->post(KK_COMBINE, s);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

cudaError_t ntt_run(const NttCall& c, cudaStream_t s)
{
    if (c.large) return ntt_run_large(c, s);
    const NttTables& t0 = c.tab[0];
    const int l1 = t0.l1, l2 = t0.l2;
    const int N1 = 1 << l1, N2 = 1 << l2;
    const int64_t P = (int64_t)N1 * N2;
    const bool argmax = c.am.results != nullptr;
    cudaError_t e;
    for (int64_t p0 = 0; p0 < c.batch; p0 += c.chunk) {
        const int64_t nb = (c.batch - p0 < c.chunk) ? c.batch - p0 : c.chunk;
        for (int pi = 0; pi < c.np; ++pi) {
            const NttTables& T = c.tab[pi];
            Pass1Args a1;
            memset(&a1, 0, sizeof(a1));
            a1.op[0] = c.op[0];
            a1.op[1] = c.op[1];
            a1.Y = c.Y;
            a1.gtw = T.g1f;
            a1.twf = T.twf;
            a1.twab = T.twab;
            a1.stats = c.stats;
            a1.m = T.m;
            a1.p0 = t0.p;
            a1.N2 = N2;
            a1.zero_upper = c.zero_upper;
            a1.skip_cs = pi > 0;
            a1.pair0 = p0;
            // both operands must use the same kernel instantiation (grid.y = 2)
            const int dt = c.op[0].dtype, qm = c.op[0].q.mode;
            if (c.op[1].dtype == dt && c.op[1].q.mode == qm) {
                if (c.prof) c.prof->pre(KK_PASS1, s);
                e = dispatch_p1(l1, a1, dt, qm, dim3(N2 / 32, 2, (unsigned)nb), s);
                if (c.prof) c.prof->post(KK_PASS1, s);
                if (e != cudaSuccess) return e;
            } else {
                // mixed quantiser modes: one launch per operand (grid.y = 1)
                for (int op = 0; op < 2; ++op) {
                    Pass1Args b1 = a1;
                    b1.op[0] = c.op[op];
                    b1.op[1] = c.op[op];
                    b1.op_base = op;
                    const int dto = c.op[op].dtype, qmo = c.op[op].q.mode;
                    if (c.prof) c.prof->pre(KK_PASS1, s);
                    e = dispatch_p1(l1, b1, dto, qmo, dim3(N2 / 32, 1, (unsigned)nb), s);
                    if (c.prof) c.prof->post(KK_PASS1, s);
                    if (e != cudaSuccess) return e;
                }
            }
            Pass2Args a2;
            memset(&a2, 0, sizeof(a2));
            a2.Y = c.Y;
            a2.Z = c.Z;
            a2.gtwf = T.g2f;
            a2.gtwi = T.g2i;
            a2.twinv = T.twi;
            a2.twib = T.twib;
            a2.stats = c.stats;
            a2.m = T.m;
            a2.p0 = t0.p;
            a2.N1 = N1;
            a2.skip_cs = pi > 0;
            a2.pair0 = p0;
            if (c.prof) c.prof->pre(KK_PASS2, s);
            e = dispatch_p2(l2, a2, dim3(N1 / 32, (unsigned)nb), s);
            if (c.prof) c.prof->post(KK_PASS2, s);
            if (e != cudaSuccess) return e;
            Pass3Args a3;
            memset(&a3, 0, sizeof(a3));
            a3.Z = c.Z;
            a3.R = c.R;
            a3.gtwi = T.g1i;
            a3.stats = c.stats;
            a3.am = c.am;
            a3.values = c.values;
            a3.nout = c.nout;
            a3.vld = c.nout;
            a3.m = T.m;
            a3.p0 = t0.p;
            a3.N2 = N2;
            a3.np = c.np;
            a3.pi = pi;
            a3.pair0 = p0;
            if (c.prof) c.prof->pre(KK_PASS3, s);
            e = argmax ? dispatch_p3_out<OUT_ARGMAX>(l1, a3, dim3(N2 / 32, (unsigned)nb), s)
                       : dispatch_p3_out<OUT_VALUES>(l1, a3, dim3(N2 / 32, (unsigned)nb), s);
            if (c.prof) c.prof->post(KK_PASS3, s);
            if (e != cudaSuccess) return e;
            if (argmax && pi == 0) {
                MergeArgs ma;
                memset(&ma, 0, sizeof(ma));
                ma.am = c.am;
                ma.stats = c.stats;
                ma.pair0 = p0;
                ma.nb = nb;
                ma.p0 = t0.p;
                ma.nblk = N2 / 32;
                ma.np = c.np;
                if (c.prof) c.prof->pre(KK_PASS3, s);
                k_merge_partials<<<(unsigned)((nb + 7) / 8), 256, 0, s>>>(ma);
                e = cudaGetLastError();
                if (c.prof) c.prof->post(KK_PASS3, s);
                if (e != cudaSuccess) return e;
            }
        }
        if (c.np > 1) {
            CombineArgs ca;
            memset(&ca, 0, sizeof(ca));
            ca.R = c.R;
            ca.stats = c.stats;
            ca.am = c.am;
            ca.values = c.values;
            ca.nout = c.nout;
            ca.vld = c.nout;
            ca.P = P;
            for (int i = 0; i < c.np; ++i) {
                ca.p[i] = c.tab[i].p;
                ca.ginv[i] = c.garner_inv[i];
            }
            ca.p0 = t0.p;
            ca.np = c.np;
            ca.pair0 = p0;
            int64_t span = argmax ? (c.am.t_hi - c.am.t_lo + 1) : c.nout;
            int nblk = (int)((span + 256 * 8 - 1) / (256 * 8));
            if (nblk > kMaxPartials) nblk = kMaxPartials;
            if (nblk < 1) nblk = 1;
            if (c.prof) c.prof->pre(KK_COMBINE, s);
            if (argmax) k_combine<OUT_ARGMAX><<<dim3(nblk, (unsigned)nb), 256, 0, s>>>(ca);
            else k_combine<OUT_VALUES><<<dim3(nblk, (unsigned)nb), 256, 0, s>>>(ca);
            e = cudaGetLastError();
            if (c.prof) c.prof->post(KK_COMBINE, s);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

}  // namespace qx
