// qx_tc.cu -- bounded-lag-window correlation on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, s8 x s8 -> s32 in TMEM).
//
// For a lag tile [L0, L0 + 2048): c[L0 + 16a + r] = sum_k A[a][k] * B[r][k]
// with a in [0,128) (M = 128), r in [0,16) (N = 16),
//   A[a][k] = ycode[L0 + 16a + k]          (Hankel rows, stride 16 bytes)
//   B[r][k] = xcode[k - r]                 (16 byte-shifted copies of x)
// k in [0, K), K = nx + 15 rounded up to 32.  A is read straight from the
// linear y-code buffer in shared memory: the K-major no-swizzle descriptor's
// core matrices (8 rows x 16 B) overlap (LBO = 16 B along K, SBO = 128 B
// along M), so the Hankel matrix is never materialised.  B is materialised
// once per pair: chunk (k-chunk kc, shift r) = xcode[16kc - r, +16) at
// kc*272 + (r/8)*128 + (r%8)*16 (LBO = 272 B, SBO = 128 B).
// This is the reference's brute-force correlation (intxcorr.py:96-100)
// restricted to a window (parity = the full correlogram sliced).
//
// Per CTA (persistent over pairs, one CTA per SM, 16 warps): smem operands
// and TMEM accumulators are double buffered.  Warp 0 issues each pair's MMA
// chain from one thread (completion: tcgen05.commit -> mbarrier); warps 4-7
// drain the previous pair's accumulator (tcgen05.ld -> argmax) behind a
// named barrier; every warp quantises and builds the next pair meanwhile,
// with that pair's float4 loads already in flight.
#include <climits>
#include <cstring>
#include <type_traits>

#include "qx_internal.h"

namespace qx {

constexpr int kTcThreads = 512;                 // builder threads (warps 0-15)
constexpr int kTcMmaWarp = 16;                   // MMA issuer
constexpr int kTcTotalThreads = 24 * 32;         // + warp 16 (MMA), warps 20-23 (epilogue)
constexpr int kTcLags = 2048;      // lags per tile: M=128 rows x N=16
constexpr int kTcMaxK = 4608;      // nx + 15 <= kTcMaxK (B buffer 16*K bytes)
constexpr int kTcMaxTiles = 2;     // lag tiles per pair
constexpr int kTcYBytes = kTcMaxTiles * kTcLags + kTcMaxK + 64;
// B layout: K-chunk stride 272 B (= 256 + 16): 16-byte stores of 32
// consecutive chunks then hit 8 distinct bank groups (4 wavefronts, no
// conflicts); the descriptor's LBO carries the stride
constexpr int kTcBLbo = 272;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// bounded wait: a commit that never arrives traps (error) instead of hanging
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase)
{
    uint32_t done = 0;
    for (uint32_t spin = 0; !done; ++spin) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
        if (spin > (1u << 26)) __trap();
    }
}

// 64-bit shared-memory matrix descriptor, K-major, no swizzle (sm_100 v1)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// instruction descriptor: kind::i8, D = s32, A = B = s8, K-major, N = 16, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct TcArgs {
    OperandDesc op[2];       // x (template side, B), y (A)
    unsigned long long* stats;
    ArgmaxOut am;            // window on t, results
    int64_t L0;              // first lag of tile 0, relative: t = L0 + (nx - 1) + ...
    int ntiles;
    int K;                   // padded K (multiple of 32)
    int fast;                // float32, n <= 4096, aligned rows, L0 % 4 == 0
    int64_t batch;
};

struct TcSmem {
    alignas(128) int8_t b[2][kTcBLbo * (kTcMaxK / 16)];   // shifted x copies
    alignas(128) int8_t y[2][kTcYBytes];      // y codes from lag L0 on
    alignas(16) int8_t xl[2][kTcMaxK + 64];   // linear x codes, 16 zero bytes in front
    double thr[2][kMaxThr];
    uint64_t bar[2];    // MMA chain of slot s complete (tcgen05.commit)
    uint64_t tfree[2];  // epilogue finished reading TMEM slot s (128 arrivals)
    uint32_t tmem_base;
    int best[kTcThreads / 32][3];
};

template <typename T, int QM>
__device__ __forceinline__ int tc_level(T v, const T* thr, int k, int tbits, T inv_step, unsigned& flags)
{
    if (v != v) flags |= SF_NONFINITE;
    if constexpr (QM == QM_K1) return level_k1(v, thr[0], thr[1]);
    else if constexpr (QM == QM_UNIFORM) return level_uniform(v, thr, k, inv_step);
    else return level_bsearch(v, thr, tbits) - k;
}

// quantise pair `pair` into smem slot s: x -> xl (linear) -> b (shifted
// copies), y window -> y; accumulate statistics over the whole signals
template <typename T, int QM>
__device__ void tc_build(const TcArgs& a, TcSmem& S, int s, int64_t pair)
{
    const T* thrx = reinterpret_cast<const T*>(S.thr[0]);
    const T* thry = reinterpret_cast<const T*>(S.thr[1]);
    const OperandDesc& dx = a.op[0];
    const OperandDesc& dy = a.op[1];
    const T* xs = reinterpret_cast<const T*>(dx.data) + pair * dx.ld;
    const T* ys = reinterpret_cast<const T*>(dy.data) + pair * dy.ld;
    const int nx = (int)dx.n, ny = (int)dy.n, K = a.K;
    unsigned ssx = 0, nzx = 0, ssy = 0, nzy = 0, fl = 0;
    // linear x codes: xl[16 + m] = q(x[m]) (zero padding around)
    int8_t* xl = S.xl[s];
    for (int i = threadIdx.x; i < K + 48; i += kTcThreads) {
        const int m = i - 16;
        int c = 0;
        if (m >= 0 && m < nx) {
            c = tc_level<T, QM>(__ldg(&xs[m]), thrx, dx.q.k, dx.q.tbits, (T)dx.q.inv_step, fl);
            ssx += (unsigned)(c * c);
            nzx += c != 0;
        }
        xl[i] = (int8_t)c;
    }
    // y codes of the lag window: y[s][i] = q(y[L0 + (nx-1) + i]); lag
    // L0 + 16a + r pairs x[m] with y[m + lag], so row a starts at y index
    // lag_base + 16a with lag_base = L0 (x starts at k - r = m)
    int8_t* yb = S.y[s];
    const int ylen = a.ntiles * kTcLags + K;
    const int64_t y0 = a.L0;
    for (int i = threadIdx.x; i < ylen; i += kTcThreads) {
        const int64_t j = y0 + i;
        int c = 0;
        if (j >= 0 && j < ny) {
            c = tc_level<T, QM>(__ldg(&ys[j]), thry, dy.q.k, dy.q.tbits, (T)dy.q.inv_step, fl);
            ssy += (unsigned)(c * c);
            nzy += c != 0;
        }
        yb[i] = (int8_t)c;
    }
    // y samples outside the window still count for the statistics
    for (int64_t j = threadIdx.x; j < ny; j += kTcThreads) {
        if (j >= y0 && j < y0 + ylen) continue;
        const int c = tc_level<T, QM>(__ldg(&ys[j]), thry, dy.q.k, dy.q.tbits, (T)dy.q.inv_step, fl);
        ssy += (unsigned)(c * c);
        nzy += c != 0;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");  // builders only
    // shifted copies: chunk (kc, r) = xl[16kc + 16 - r, +16)
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(xl);
    uint4* b4 = reinterpret_cast<uint4*>(S.b[s]);
    const int nchunk = K / 16;
    for (int i = threadIdx.x; i < nchunk * 16; i += kTcThreads) {
        const int kc = i >> 4, r = i & 15;
        const int o = 16 * kc + 16 - r;
        const int w0 = o >> 2, sh = (o & 3) * 8;
        const uint32_t a0 = xw[w0], a1 = xw[w0 + 1], a2 = xw[w0 + 2], a3 = xw[w0 + 3], a4 = xw[w0 + 4];
        uint4 v;
        v.x = __funnelshift_r(a0, a1, sh);
        v.y = __funnelshift_r(a1, a2, sh);
        v.z = __funnelshift_r(a2, a3, sh);
        v.w = __funnelshift_r(a3, a4, sh);
        b4[kc * (kTcBLbo / 16) + (r >> 3) * 8 + (r & 7)] = v;
    }
    // statistics (one atomic per warp)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ssx += __shfl_xor_sync(0xffffffffu, ssx, o);
        nzx += __shfl_xor_sync(0xffffffffu, nzx, o);
        ssy += __shfl_xor_sync(0xffffffffu, ssy, o);
        nzy += __shfl_xor_sync(0xffffffffu, nzy, o);
        fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* st = a.stats + pair * 8;
        if (ssx) atomicAdd(st + 0, (unsigned long long)ssx);
        if (nzx) atomicAdd(st + 1, (unsigned long long)nzx);
        if (ssy) atomicAdd(st + 4, (unsigned long long)ssy);
        if (nzy) atomicAdd(st + 5, (unsigned long long)nzy);
        if (fl) atomicOr(st + 2, (unsigned long long)fl);
    }
}

// ---- fast build: float32 rows, nx, ny <= kTcFastN, 16-B aligned rows,
// L0 % 4 == 0.  Each thread owns float4 #t and #t + kTcThreads of x and y;
// the next pair's float4s are loaded into registers before the current pair
// is built (one pair of loads always in flight).
constexpr int kTcFastN = 4 * 2 * kTcThreads;  // 4096 with 512 threads

struct TcRegs {
    float4 x[2], y[2];
};

__device__ __forceinline__ void tc_fetch(const TcArgs& a, int64_t pair, TcRegs& r)
{
    const float4* xs = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.op[0].data) + pair * a.op[0].ld);
    const float4* ys = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.op[1].data) + pair * a.op[1].ld);
    const int nx4 = (int)(a.op[0].n >> 2), ny4 = (int)(a.op[1].n >> 2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = threadIdx.x + h * kTcThreads;
        r.x[h] = i < nx4 ? __ldg(&xs[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
        r.y[h] = i < ny4 ? __ldg(&ys[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

template <int QM>
__device__ __forceinline__ int tc_q(float v, const float* thr, int k, float inv_step, unsigned& flags, int tbits = 8)
{
    if (v != v) flags |= SF_NONFINITE;
    if constexpr (QM == QM_K1) return level_k1(v, thr[0], thr[1]);
    else if constexpr (QM == QM_UNIFORM) return level_uniform_magic(v, thr, k, inv_step);
    else return level_bsearch(v, thr, tbits) - k;
}

// quantise 4 samples -> packed int8 word, statistics
template <int QM>
__device__ __forceinline__ uint32_t tc_q4(float4 v, const float* thr, int k, float inv_step, int tbits,
                                          unsigned& ss, unsigned& nz, unsigned& fl)
{
    const int c0 = tc_q<QM>(v.x, thr, k, inv_step, fl, tbits), c1 = tc_q<QM>(v.y, thr, k, inv_step, fl, tbits);
    const int c2 = tc_q<QM>(v.z, thr, k, inv_step, fl, tbits), c3 = tc_q<QM>(v.w, thr, k, inv_step, fl, tbits);
    ss += (unsigned)(c0 * c0 + c1 * c1 + c2 * c2 + c3 * c3);
    nz += (c0 != 0) + (c1 != 0) + (c2 != 0) + (c3 != 0);
    return (uint32_t)(c0 & 0xff) | ((uint32_t)(c1 & 0xff) << 8) | ((uint32_t)(c2 & 0xff) << 16) |
           ((uint32_t)c3 << 24);
}

template <int QM>
__device__ void tc_build_fast(const TcArgs& a, TcSmem& S, int s, int64_t pair, const TcRegs& r)
{
    const float* thrx = reinterpret_cast<const float*>(S.thr[0]);
    const float* thry = reinterpret_cast<const float*>(S.thr[1]);
    const int kx = a.op[0].q.k, ky = a.op[1].q.k;
    const float ix = (float)a.op[0].q.inv_step, iy = (float)a.op[1].q.inv_step;
    const int nx4 = (int)(a.op[0].n >> 2), ny4 = (int)(a.op[1].n >> 2), K = a.K;
    const int ylen = a.ntiles * kTcLags + K;
    uint32_t* xw = reinterpret_cast<uint32_t*>(S.xl[s]);
    uint32_t* yw = reinterpret_cast<uint32_t*>(S.y[s]);
    // zero the margins: x words outside [4, 4 + nx4), y words outside the signal
    const int yoff = (int)(-a.L0) >> 2;  // word index of y[0] in the window (may be < 0)
    for (int i = threadIdx.x; i < (K + 64) / 4; i += kTcThreads)
        if (i < 4 || i >= 4 + nx4) xw[i] = 0;
    for (int i = threadIdx.x; i < (ylen + 3) / 4; i += kTcThreads)
        if (i < yoff || i >= yoff + ny4) yw[i] = 0;
    unsigned ssx = 0, nzx = 0, ssy = 0, nzy = 0, fl = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = threadIdx.x + h * kTcThreads;
        if (i < nx4) xw[4 + i] = tc_q4<QM>(r.x[h], thrx, kx, ix, a.op[0].q.tbits, ssx, nzx, fl);
        if (i < ny4) {
            const uint32_t w = tc_q4<QM>(r.y[h], thry, ky, iy, a.op[1].q.tbits, ssy, nzy, fl);
            const int wi = yoff + i;
            if (wi >= 0 && wi < (ylen + 3) / 4) yw[wi] = w;
        }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");  // builders only
    // shifted copies: item -> (chunk position kc, half h) with h uniform per
    // warp; the thread emits shifts r = 8h .. 8h+7 of chunk kc
    const uint4* xq = reinterpret_cast<const uint4*>(S.xl[s]);
    uint4* b4 = reinterpret_cast<uint4*>(S.b[s]);
    const int nchunk = K / 16;
    const int nitems = 64 * ((nchunk + 31) / 32);
    for (int i = threadIdx.x; i < nitems; i += kTcThreads) {
        const int kc = (i & 31) + 32 * (i >> 6), h = (i >> 5) & 1;
        if (kc >= nchunk) continue;
        // bytes [16kc, 16kc + 32) of xl (= x[16kc - 16 .. 16kc + 16))
        const uint4 lo = xq[kc], hi = xq[kc + 1];
        const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        uint4* dst = b4 + kc * (kTcBLbo / 16) + h * 8;
        if (h == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // r = j: bytes [16 - j, 32 - j)
                const int o = 16 - j, wq = o >> 2, sh = (o & 3) * 8;
                uint4 v;
                v.x = __funnelshift_r(w[wq], w[wq + 1], sh);
                v.y = __funnelshift_r(w[wq + 1], w[wq + 2], sh);
                v.z = __funnelshift_r(w[wq + 2], w[wq + 3], sh);
                v.w = __funnelshift_r(w[wq + 3], (wq + 4 < 8) ? w[wq + 4] : 0u, sh);
                dst[j] = v;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // r = 8 + j: bytes [8 - j, 24 - j)
                const int o = 8 - j, wq = o >> 2, sh = (o & 3) * 8;
                uint4 v;
                v.x = __funnelshift_r(w[wq], w[wq + 1], sh);
                v.y = __funnelshift_r(w[wq + 1], w[wq + 2], sh);
                v.z = __funnelshift_r(w[wq + 2], w[wq + 3], sh);
                v.w = __funnelshift_r(w[wq + 3], w[wq + 4], sh);
                dst[j] = v;
            }
        }
    }
    ssx = __reduce_add_sync(0xffffffffu, ssx);
    nzx = __reduce_add_sync(0xffffffffu, nzx);
    ssy = __reduce_add_sync(0xffffffffu, ssy);
    nzy = __reduce_add_sync(0xffffffffu, nzy);
    fl = __reduce_or_sync(0xffffffffu, fl);
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* st = a.stats + pair * 8;
        if (ssx) atomicAdd(st + 0, (unsigned long long)ssx);
        if (nzx) atomicAdd(st + 1, (unsigned long long)nzx);
        if (ssy) atomicAdd(st + 4, (unsigned long long)ssy);
        if (nzy) atomicAdd(st + 5, (unsigned long long)nzy);
        if (fl) atomicOr(st + 2, (unsigned long long)fl);
    }
}

// argmax epilogue of pair `pair` from TMEM slot s, run by warps 4..7 only
// (warp w reads TMEM lanes 32*(w%4) .. +31 = accumulator rows), reduced with
// a 128-thread named barrier so the other warps keep building.
constexpr int kEpiWarp0 = 20;

__device__ void tc_epilogue(const TcArgs& a, TcSmem& S, int s, int64_t pair)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp - kEpiWarp0;  // 0..3 = TMEM lane quarter
    long long bv = LLONG_MIN, bt = LLONG_MAX, bc = 0;
    const int64_t nx = a.op[0].n;
    for (int tile = 0; tile < a.ntiles; ++tile) {
        int v[16];
        const uint32_t taddr = S.tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(s * 32 + tile * 16);
        tmem_ld16(taddr, v);
        const int row = q * 32 + lane;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            // lag = L0 + tile*2048 + 16*row + r; correlogram index t = lag + nx - 1
            const long long t = a.L0 + tile * kTcLags + 16 * row + r + nx - 1;
            if (t < a.am.t_lo || t > a.am.t_hi) continue;
            const long long val = v[r];
            if (val > bv) { bv = val; bt = t; bc = 1; }
            else if (val == bv) { bt = min(bt, t); ++bc; }
        }
    }
    // TMEM reads are complete (wait::ld) before the next MMA into this slot
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const long long ov = __shfl_xor_sync(0xffffffffu, bv, o), ot = __shfl_xor_sync(0xffffffffu, bt, o),
                        oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (ov > bv) { bv = ov; bt = ot; bc = oc; }
        else if (ov == bv) { bt = min(bt, ot); bc += oc; }
    }
    asm volatile("bar.sync 4, 128;" ::: "memory");  // previous pair's S.best reads done
    if (lane == 0) {
        S.best[q][0] = (int)(bv == LLONG_MIN ? INT_MIN : bv);
        S.best[q][1] = (int)(bt == LLONG_MAX ? INT_MAX : bt);
        S.best[q][2] = (int)bc;
    }
    asm volatile("bar.sync 4, 128;" ::: "memory");
    if (q == 0 && lane == 0) {
        long long v0 = LLONG_MIN, t0 = LLONG_MAX, c0 = 0;
        for (int w = 0; w < 4; ++w) {
            if (S.best[w][2] == 0) continue;
            const long long ov = S.best[w][0], ot = S.best[w][1], oc = S.best[w][2];
            if (ov > v0) { v0 = ov; t0 = ot; c0 = oc; }
            else if (ov == v0) { t0 = min(t0, ot); c0 += oc; }
        }
        // qx_result record; the statistics atomics of this pair were issued by
        // this CTA before the barrier that preceded its MMA chain
        long long* res = reinterpret_cast<long long*>(a.am.results) + pair * 8;
        const unsigned long long* sp = a.stats + pair * 8;
        __threadfence();
        unsigned long long st[8];
        for (int i = 0; i < 8; ++i) st[i] = __ldcg(sp + i);  // atomics live in L2
        const long long nzx = (long long)st[1], nzy = (long long)st[5];
        const unsigned f = (unsigned)(st[2] | st[6]);
        int flags = 0;
        if (nzx == 0) flags |= 1;
        if (nzy == 0) flags |= 2;
        if (f & SF_NONFINITE) flags |= 4;
        int status = (flags & 4) ? 9 : ((flags & 3) ? 2 : 0);
        res[0] = v0;
        res[1] = a.am.first_lag + t0;
        res[2] = c0;
        res[3] = (long long)st[0];
        res[4] = (long long)st[4];
        res[5] = nzx;
        res[6] = nzy;
        res[7] = ((long long)status << 32) | (unsigned)flags;
    }
}

// completion of the MMA chain of loop iteration j (slot j & 1): the slot's
// mbarrier completes once per use, so use number j >> 1 has parity (j>>1)&1
__device__ __forceinline__ void tc_wait_iter(TcSmem& S, int j)
{
    mbar_wait(&S.bar[j & 1], (uint32_t)((j >> 1) & 1));
}

template <typename T, int QM>
__global__ void __launch_bounds__(kTcTotalThreads, 1) k_tc_window(const __grid_constant__ TcArgs a)
{
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    TcSmem& S = *reinterpret_cast<TcSmem*>(tc_smem_raw);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kMaxThr; i += kTcTotalThreads) {
        reinterpret_cast<T*>(S.thr[0])[i] = (T)a.op[0].q.thr[i];
        reinterpret_cast<T*>(S.thr[1])[i] = (T)a.op[1].q.thr[i];
    }
    if (threadIdx.x == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
        mbar_init(&S.tfree[0], 128);
        mbar_init(&S.tfree[1], 128);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&S.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    const int64_t npairs = a.batch > blockIdx.x ? (a.batch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (warp < kTcThreads / 32) {
        // ---- builders: quantise + operands of iteration it into slot it & 1
        auto handoff = [&](int it) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> async proxy
            // alternating barrier ids keep consecutive iterations apart
            if (it & 1) asm volatile("bar.arrive 3, %0;" ::"n"(kTcThreads + 32) : "memory");
            else asm volatile("bar.arrive 2, %0;" ::"n"(kTcThreads + 32) : "memory");
        };
        bool fast = false;
        if constexpr (std::is_same<T, float>::value) fast = a.fast;
        if (fast) {
            if constexpr (std::is_same<T, float>::value) {
                TcRegs cur, nxt;
                if (npairs) tc_fetch(a, blockIdx.x, cur);
                for (int it = 0; it < npairs; ++it) {
                    const int64_t pair = blockIdx.x + (int64_t)it * gridDim.x;
                    if (it + 1 < npairs) tc_fetch(a, pair + gridDim.x, nxt);
                    if (it >= 2) tc_wait_iter(S, it - 2);  // slot no longer read by MMAs
                    tc_build_fast<QM>(a, S, it & 1, pair, cur);
                    handoff(it);
                    cur = nxt;
                }
            }
        } else {
            for (int it = 0; it < npairs; ++it) {
                const int64_t pair = blockIdx.x + (int64_t)it * gridDim.x;
                if (it >= 2) tc_wait_iter(S, it - 2);
                tc_build<T, QM>(a, S, it & 1, pair);
                handoff(it);
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ---- MMA issuer: one thread drives the tensor core
        const int nk = a.K / 32;
        for (int it = 0; it < npairs; ++it) {
            const int s = it & 1;
            if (it & 1) asm volatile("bar.sync 3, %0;" ::"n"(kTcThreads + 32) : "memory");
            else asm volatile("bar.sync 2, %0;" ::"n"(kTcThreads + 32) : "memory");
            if (it >= 2) mbar_wait(&S.tfree[s], (uint32_t)(((it - 2) >> 1) & 1));  // TMEM slot drained
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if ((threadIdx.x & 31) == 0) {
                const uint32_t ya = smem_u32(S.y[s]), ba = smem_u32(S.b[s]);
                const uint64_t bd0 = smem_desc(ba, kTcBLbo, 128);
                for (int tile = 0; tile < a.ntiles; ++tile) {
                    const uint32_t d = S.tmem_base + (uint32_t)(s * 32 + tile * 16);
                    uint64_t ad = smem_desc(ya + tile * kTcLags, 16, 128), bd = bd0;
                    for (int kk = 0; kk < nk; ++kk) {
                        mma_i8(d, ad, bd, kk > 0);
                        ad += 32 >> 4;             // next 32 k-bytes of A
                        bd += (2 * kTcBLbo) >> 4;  // next two k-chunks of B
                    }
                }
                mma_commit(&S.bar[s]);
            }
            __syncwarp();
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ---- epilogue: TMEM -> argmax -> qx_result, then free the TMEM slot
        for (int it = 0; it < npairs; ++it) {
            const int64_t pair = blockIdx.x + (int64_t)it * gridDim.x;
            tc_wait_iter(S, it);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            tc_epilogue(a, S, it & 1, pair);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.tfree[it & 1])) : "memory");
        }
    }
    // every MMA was waited on by the epilogue before TMEM is released
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(S.tmem_base));
}

// eligibility: window of at most kTcMaxTiles*2048 lags, nx + 15 <= kTcMaxK,
// |values| < 2^31 (nx * Kx * Ky), same input dtype and quantiser mode (float)
bool tc_window_eligible(const NttCall& c, int64_t nx, int64_t ny)
{
    (void)ny;
    const int64_t W = c.am.t_hi - c.am.t_lo + 1;
    if (W > (int64_t)kTcMaxTiles * kTcLags) return false;
    if (nx + 15 > kTcMaxK) return false;
    if (c.op[0].dtype != c.op[1].dtype || c.op[0].dtype == DT_I64) return false;
    if (c.op[0].q.mode != c.op[1].q.mode) return false;
    if (c.op[0].q.k > 127 || c.op[1].q.k > 127) return false;
    if ((double)nx * c.op[0].q.k * c.op[1].q.k >= 2147483647.0) return false;
    return true;
}

template <typename T, int QM>
static cudaError_t launch_tc(const TcArgs& a, cudaStream_t s, int sms)
{
    static bool attr = false;
    const size_t smem = sizeof(TcSmem);
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_tc_window<T, QM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int grid = (int)(a.batch < sms ? a.batch : sms);
    k_tc_window<T, QM><<<grid, kTcTotalThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t tc_window_run(const NttCall& c, int64_t nx, cudaStream_t s)
{
    TcArgs a;
    memset(&a, 0, sizeof(a));
    a.op[0] = c.op[0];
    a.op[1] = c.op[1];
    a.stats = c.stats;
    a.am = c.am;
    a.batch = c.batch;
    // tile 0 starts at the window's first lag (relative lag = t - (nx - 1))
    a.L0 = c.am.t_lo - (nx - 1);
    const int64_t W = c.am.t_hi - c.am.t_lo + 1;
    a.ntiles = (int)((W + kTcLags - 1) / kTcLags);
    a.K = (int)(((nx + 15) + 31) / 32 * 32);
    const int64_t ny = c.op[1].n;
    a.fast = c.op[0].dtype == DT_F32 && nx <= kTcFastN && ny <= kTcFastN && nx % 4 == 0 && ny % 4 == 0 &&
             (c.batch == 1 || (c.op[0].ld % 4 == 0 && c.op[1].ld % 4 == 0)) &&
             ((uintptr_t)c.op[0].data % 16 == 0) && ((uintptr_t)c.op[1].data % 16 == 0) && (a.L0 % 4 == 0);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (c.prof) c.prof->pre(KK_DIRECT, s);
    cudaError_t e;
    const int qm = c.op[0].q.mode;
    if (c.op[0].dtype == DT_F32) {
        if (qm == QM_K1) e = launch_tc<float, QM_K1>(a, s, sms);
        else if (qm == QM_UNIFORM) e = launch_tc<float, QM_UNIFORM>(a, s, sms);
        else e = launch_tc<float, QM_BSEARCH>(a, s, sms);
    } else {
        if (qm == QM_K1) e = launch_tc<double, QM_K1>(a, s, sms);
        else if (qm == QM_UNIFORM) e = launch_tc<double, QM_UNIFORM>(a, s, sms);
        else e = launch_tc<double, QM_BSEARCH>(a, s, sms);
    }
    if (c.prof) c.prof->post(KK_DIRECT, s);
    return e;
}

}  // namespace qx
