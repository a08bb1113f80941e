// qx_tc_i8.cu -- bounded-lag-window correlation on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, s8 x s8 -> s32 in TMEM): the int8 modes
// (per-pair B, BASELINE config 3; shared template with k > 4 codes).
// Reached through qx_tc.cu tc_window_run, which keeps the fp4 modes; the two
// kernels differ in their role layout -- here 3 lag warps and the merge in
// the first epilogue warp, whose hand-off timing an int8 pair needs (the fp4
// kernel's dedicated merge warp measured 14 % slower on config 3, b = 4).
//
// For a lag tile [L0, L0 + 16M): c[L0 + 16a + r] = sum_k A[a][k] * B[r][k]
// with a in [0,M) (M = 64 or 128), r in [0,16) (N = 16),
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
// Cost model (tools/tc_rate.cu, measured on B200): an i8 MMA with both
// operands in shared memory takes max(~(32*M + 32*N) / 128 B/clk, M*N/256)
// cycles when issued from a converged warp -- 25.8 cycles at M=64, 39 at
// M=128 (N=16) -- so the tile shape follows the window: M=64 when the window
// fits 1024 lags (+16), else M=128.  The symmetric windows callers use have
// 2h+1 lags; up to 16 lags past the tiles are summed on the CUDA cores
// (dp4a) by the epilogue warps instead of a second tile.
//
// Per CTA (persistent over pairs, one CTA per SM): shared-memory operands
// are double buffered (data slot = it & 1), TMEM accumulators and the
// per-pair statistics / extra-lag sums quadruple buffered (aux slot =
// it & 3).  Warps 0-15 quantise and build the next pair (its float4 loads
// already in flight), sum the extra lags and reduce the statistics into
// shared memory; warp 16 issues the MMA chain (converged, elect.sync;
// completion: tcgen05.commit -> mdone[aux]); warps 20-23 drain an
// accumulator (tcgen05.ld -> argmax), write the qx_result and release the
// aux slot (tfree[aux]).  A data slot is reused as soon as its MMA chain
// completes, so the epilogue is off the builders' critical path.
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "qx_internal.h"

namespace qx {
namespace i8 {

constexpr int kTcThreads = 512;                 // builder threads (warps 0-15)
constexpr int kTcMmaWarp = 16;                   // MMA issuer
constexpr int kTcLagWarp0 = 17, kTcLagWarps = 3;  // extra-lag dot products (warps 17-19)
// builders + MMA warp + lag warps meet at the per-pair hand-off barrier
constexpr int kTcHandoff = kTcThreads + 32 + 32 * kTcLagWarps;
constexpr int kTcTotalThreads = 24 * 32;         // + warp 16 (MMA), warps 20-23 (epilogue)
constexpr int kTcLags = 2048;      // lags per M=128 tile (M=64: 1024)
constexpr int kTcMaxK = 4608;      // nx + 15 <= kTcMaxK (B buffer 16*K bytes)
constexpr int kTcMaxTiles = 2;     // lag tiles per pair
constexpr int kTcMaxExtra = 16;    // lags past the tiles, summed on CUDA cores
constexpr int kTcYBytes = kTcMaxTiles * kTcLags + kTcMaxExtra + kTcMaxK + 64;
constexpr int kTcYStride = (kTcYBytes + 1023) / 1024 * 1024;  // 1024-B aligned slots (SW32 rows)
constexpr int kTcXPad = 32;  // zero bytes in front of the linear x codes (>= the Hankel pitch)
// B layout: K-chunk stride 272 B (= 256 + 16): 16-byte stores of 32
// consecutive chunks then hit 8 distinct bank groups (4 wavefronts, no
// conflicts); the descriptor's LBO carries the stride
constexpr int kTcBLbo = 272;
// shared-template mode (pitch 32): 32 copies, K-chunk stride 528 B = 33
// 16-B units (odd: conflict-free like 272); one buffer, built once
constexpr int kTcBLbo32 = 528;
constexpr int kTcBSlot = kTcBLbo * (kTcMaxK / 16);
constexpr int kTcBBytes = 2 * kTcBSlot;
static_assert(kTcBLbo32 * (kTcMaxK / 16) <= kTcBBytes, "pitch-32 B must fit the two pitch-16 slots");

// y code word wi of a slot: pitch 32 stores the buffer through the 32-byte
// swizzle (byte bit 4 ^= bit 7, i.e. word bit 2 ^= bit 5) so that a SW32
// K-major descriptor reads it back as a linear buffer: Hankel rows 32 B
// apart at any 32-B-aligned start (verified by tools/tc_swz.cu)
template <int PITCH>
__device__ __forceinline__ int ysw(int wi)
{
    if constexpr (PITCH == 32) return wi ^ (((wi >> 5) & 1) << 2);
    else return wi;
}

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

// instruction descriptor: kind::i8, D = s32, A = B = s8, K-major
constexpr uint32_t tc_idesc(int M, int N)
{
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Issued by a whole converged warp: elect.sync picks the issuing lane inside
// the asm, so ptxas emits no per-instruction divergence loop around UTCIMMA
// (single-lane issue under `if (lane == 0)` costs ~52 cycles per MMA).
__device__ __forceinline__ void mma_i8_warp(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Four MMAs on consecutive K steps under one elect.sync.  Descriptors are
// passed as 32-bit low words (start address >> 4, which never carries into
// the LBO field) and a shared high word; A advances 32 B (+2), B two
// 272-B K-chunks (+34) per step.
template <int BINC>  // B descriptor step per K step (16-B units)
__device__ __forceinline__ void mma_i8_warp4(uint32_t tmem_d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                             uint32_t idesc)
{
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b64 a0, a1, a2, a3, b0, b1, b2, b3;\n\t.reg .b32 t;\n\t"
        "mov.b64 a0, {%1, %2};\n\tadd.u32 t, %1, 2;\n\tmov.b64 a1, {t, %2};\n\t"
        "add.u32 t, %1, 4;\n\tmov.b64 a2, {t, %2};\n\tadd.u32 t, %1, 6;\n\tmov.b64 a3, {t, %2};\n\t"
        "mov.b64 b0, {%3, %4};\n\tadd.u32 t, %3, %6;\n\tmov.b64 b1, {t, %4};\n\t"
        "add.u32 t, %3, %7;\n\tmov.b64 b2, {t, %4};\n\tadd.u32 t, %3, %8;\n\tmov.b64 b3, {t, %4};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a0, b0, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a2, b2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a3, b3, %5, 1;\n}" ::"r"(tmem_d),
        "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "n"(BINC), "n"(2 * BINC), "n"(3 * BINC));
}

__device__ __forceinline__ void mma_commit_warp(uint64_t* bar)
{
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
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
    int M;                   // MMA rows per tile (64 or 128); a tile holds 16*M lags
    int ntiles;
    int extra;               // lags after the tiles (<= kTcMaxExtra), CUDA cores
    int ylen;                // y-code window bytes: ntiles*16*M + extra + K
    uint32_t idesc;
    int K;                   // padded K (multiple of 32)
    int fast;                // float32, n <= 4096, aligned rows, L0 % 4 == 0
    int shared_x;            // fast path with x row stride 0 (template search): x built once per CTA
    int pitch;               // Hankel row pitch / N: 16 (per-pair B), 32 (shared template, SW32 A)
    int debug;               // QX_TC_TIMING builds only: 1 = skip MMAs, 2 = skip builds
    int64_t batch;
};

constexpr int kTcAux = 4;  // TMEM accumulator / statistics slots

struct TcSmem {
    alignas(1024) int8_t b[kTcBBytes];        // shifted x copies: 2 pitch-16 slots or 1 pitch-32 buffer
    alignas(1024) int8_t y[2][kTcYStride];    // y codes from lag L0 on (pitch 32: swizzled)
    alignas(16) int8_t xl[2][kTcMaxK + 96];   // linear x codes after kTcXPad zero bytes
    double thr[2][kMaxThr];
    uint64_t mdone[kTcAux];  // MMA chain of aux slot complete (tcgen05.commit)
    uint64_t tfree[kTcAux];  // epilogue finished with aux slot (128 arrivals)
    // per-builder-warp partials (no atomics): ssx, nzx, ssy, nzy, flags
    unsigned long long wst[kTcAux][kTcThreads / 32][5];
    int wxs[kTcAux][kTcLagWarps][kTcMaxExtra];     // extra-lag sums, one record per lag warp
    uint64_t xdone[kTcAux];  // lag warps finished with the pair of aux slot (96 arrivals)
    unsigned xst[3];      // shared-x mode: template ssx, nzx, flags (built once)
    uint32_t tmem_base;
    int best[kTcAux][4][3];                 // per epilogue warp (value, j, count), per aux slot
    unsigned long long fst[kTcAux][5];      // final statistics of the pair (lag warps)
#ifdef QX_TC_TIMING
    unsigned long long tm[16];
#endif
};

// Each aux barrier completes once per use of its slot (every 4th
// iteration), so iteration j's completion has parity (j >> 2) & 1.  Every
// waiter is at most one use behind (see the dependency notes in the kernel),
// so parity waits are unambiguous.
__device__ __forceinline__ void tc_wait_mdone(TcSmem& S, int j)
{
    mbar_wait(&S.mdone[j & 3], (uint32_t)((j >> 2) & 1));
}
__device__ __forceinline__ void tc_wait_tfree(TcSmem& S, int j)
{
    mbar_wait(&S.tfree[j & 3], (uint32_t)((j >> 2) & 1));
}
__device__ __forceinline__ void tc_wait_xdone(TcSmem& S, int j)
{
    mbar_wait(&S.xdone[j & 3], (uint32_t)((j >> 2) & 1));
}

// builder-side extra lags and statistics of the pair in data slot s, aux
// slot u: warp-reduced, one record per builder warp (summed by the epilogue)
// SM: statistics mode.  0: generic (64-bit y sums); 1: per-pair fast path
// (<= 8 samples per thread and operand: per warp, sum of squares < 2^23 and
// count < 2^9, so each operand's pair packs into one 32-bit REDUX); 2:
// shared template (x statistics are already final, in thread 0 only)
template <int SM>
__device__ void tc_aux_finish(TcSmem& S, int u, unsigned ssx, unsigned nzx, unsigned long long ssy,
                              unsigned long long nzy, unsigned fl)
{
    const int lane = threadIdx.x & 31;
    if (__any_sync(0xffffffffu, fl)) fl = __reduce_or_sync(0xffffffffu, fl);  // NaN: rare
    if constexpr (SM == 1) {
        const unsigned px = __reduce_add_sync(0xffffffffu, ssx | (nzx << 23));
        const unsigned py = __reduce_add_sync(0xffffffffu, (unsigned)ssy | ((unsigned)nzy << 23));
        ssx = px & 0x7fffffu;
        nzx = px >> 23;
        ssy = py & 0x7fffffu;
        nzy = py >> 23;
    } else if constexpr (SM == 2) {
        ssy = __reduce_add_sync(0xffffffffu, (unsigned)ssy);
        nzy = __reduce_add_sync(0xffffffffu, (unsigned)nzy);
    } else {
        ssx = __reduce_add_sync(0xffffffffu, ssx);
        nzx = __reduce_add_sync(0xffffffffu, nzx);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            ssy += __shfl_xor_sync(0xffffffffu, ssy, o);
            nzy += __shfl_xor_sync(0xffffffffu, nzy, o);
        }
    }
    if (lane == 0) {
        unsigned long long* st = S.wst[u][threadIdx.x >> 5];
        st[0] = ssx;
        st[1] = nzx;
        st[2] = ssy;
        st[3] = nzy;
        st[4] = fl;
    }
}


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
__device__ void tc_build(const TcArgs& a, TcSmem& S, int s, int u, int64_t pair)
{
    const T* thrx = reinterpret_cast<const T*>(S.thr[0]);
    const T* thry = reinterpret_cast<const T*>(S.thr[1]);
    const OperandDesc& dx = a.op[0];
    const OperandDesc& dy = a.op[1];
    const T* xs = reinterpret_cast<const T*>(dx.data) + pair * dx.ld;
    const T* ys = reinterpret_cast<const T*>(dy.data) + pair * dy.ld;
    const int nx = (int)dx.n, K = a.K;
    const int64_t ny = dy.n;
    unsigned ssx = 0, nzx = 0, fl = 0;
    unsigned long long ssy = 0, nzy = 0;
    // linear x codes: xl[kTcXPad + m] = q(x[m]) (zero padding around)
    int8_t* xl = S.xl[s];
    for (int i = threadIdx.x; i < K + 64; i += kTcThreads) {
        const int m = i - kTcXPad;
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
    const int ylen = a.ylen;
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
    // shifted copies: chunk (kc, r) = xl[16kc + kTcXPad - r, +16)
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(xl);
    uint4* b4 = reinterpret_cast<uint4*>(S.b + s * kTcBSlot);
    const int nchunk = K / 16;
    for (int i = threadIdx.x; i < nchunk * 16; i += kTcThreads) {
        const int kc = i >> 4, r = i & 15;
        const int o = 16 * kc + kTcXPad - r;
        const int w0 = o >> 2, sh = (o & 3) * 8;
        const uint32_t a0 = xw[w0], a1 = xw[w0 + 1], a2 = xw[w0 + 2], a3 = xw[w0 + 3], a4 = xw[w0 + 4];
        uint4 v;
        v.x = __funnelshift_r(a0, a1, sh);
        v.y = __funnelshift_r(a1, a2, sh);
        v.z = __funnelshift_r(a2, a3, sh);
        v.w = __funnelshift_r(a3, a4, sh);
        b4[kc * (kTcBLbo / 16) + (r >> 3) * 8 + (r & 7)] = v;
    }
    tc_aux_finish<0>(S, u, ssx, nzx, ssy, nzy, fl);
}

// ---- fast build: float32 rows, nx, ny <= kTcFastN, 16-B aligned rows,
// L0 % 4 == 0.  Each thread owns float4 #t and #t + kTcThreads of x and y;
// the next pair's float4s are loaded into registers before the current pair
// is built (one pair of loads always in flight).
constexpr int kTcFastN = 4 * 2 * kTcThreads;   // 4096 with 512 threads
constexpr int kTcFastNY = 4 * 4 * kTcThreads;  // shared-x mode: y rows up to 8192

// per-thread float4s of one pair (loaded one pair ahead): both rows, or in
// shared-x mode only the y row (the template is built once per CTA)
template <bool SX>
struct TcRegs {
    float4 x[2], y[2];
};
template <>
struct TcRegs<true> {
    float4 y[4];
};

// float4 #i of a row of n floats (the tail float4 of an n % 4 != 0 row by
// scalar loads, zero-padded: a zero sample quantises to code 0)
__device__ __forceinline__ float4 tc_ld4(const float* row, int i, int n)
{
    if (4 * i + 4 <= n) return __ldg(reinterpret_cast<const float4*>(row) + i);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * i < n) {
        v.x = __ldg(row + 4 * i);
        if (4 * i + 1 < n) v.y = __ldg(row + 4 * i + 1);
        if (4 * i + 2 < n) v.z = __ldg(row + 4 * i + 2);
    }
    return v;
}

template <bool SX>
__device__ __forceinline__ void tc_fetch(const TcArgs& a, int64_t pair, TcRegs<SX>& r)
{
    const float* ys = reinterpret_cast<const float*>(a.op[1].data) + pair * a.op[1].ld;
    const int ny = (int)a.op[1].n;
    if constexpr (SX) {
#pragma unroll
        for (int h = 0; h < 4; ++h) r.y[h] = tc_ld4(ys, threadIdx.x + h * kTcThreads, ny);
    } else {
        // n % 4 == 0 here: whole float4s only
        const float4* xs4 = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.op[0].data) +
                                                            pair * a.op[0].ld);
        const float4* ys4 = reinterpret_cast<const float4*>(ys);
        const int nx4 = (int)(a.op[0].n >> 2), ny4 = ny >> 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = threadIdx.x + h * kTcThreads;
            r.x[h] = i < nx4 ? __ldg(&xs4[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
            r.y[h] = i < ny4 ? __ldg(&ys4[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

// Bulk L2 prefetch (TMA engine) of the float rows of a pair kTcPrefetch
// pairs ahead: the builders hold only the next pair in registers (80
// registers per thread leave no room for a deeper register prefetch, and the
// shifted-copy buffers leave no shared memory for a float ring), so the
// pair after that is pulled into L2 and its register loads then wait on L2
// latency instead of HBM latency (ncu r01: long_scoreboard was the top
// builder stall).  One instruction per row, issued by one lane.
#ifndef QX_TC_PREFETCH
#define QX_TC_PREFETCH 2
#endif
constexpr int kTcPrefetch = QX_TC_PREFETCH;
template <bool SX>
__device__ __forceinline__ void tc_prefetch_l2(const TcArgs& a, int64_t pair)
{
    if (threadIdx.x == 0) {
        const float* ys = reinterpret_cast<const float*>(a.op[1].data) + pair * a.op[1].ld;
        const uint32_t by = (uint32_t)(a.op[1].n * 4) & ~15u;
        if (by) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ys), "r"(by) : "memory");
    } else if (!SX && threadIdx.x == 32) {
        const float* xs = reinterpret_cast<const float*>(a.op[0].data) + pair * a.op[0].ld;
        const uint32_t bx = (uint32_t)(a.op[0].n * 4) & ~15u;
        if (bx) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(xs), "r"(bx) : "memory");
    }
}

// level_uniform_nb (qx_common.cuh) as a scalar, with the NaN test folded into its
// rare exact branch: a NaN makes d NaN, fails `>= 2^-14` and lands there
// (so does +-inf, which the exact compares then map to +-k)
__device__ __forceinline__ int tc_level_uniform(float v, const float* s, int k, float inv_step, unsigned& flags)
{
    const float a = fabsf(v);
    const float t = fmaf(a, inv_step, 12582912.0f);
    int lv = __float_as_int(t) - 0x4B400000;
    const float d = fmaf(a, inv_step, -(t - 12582912.0f));
    lv = min(lv, k);
    if (__builtin_expect(!(fabsf(fabsf(d) - 0.5f) >= 0x1p-14f), 0)) {
        if (v != v) {
            flags |= SF_NONFINITE;
            return 0;
        }
        int l2 = v < 0.f ? -lv : lv;
        if (l2 < k && v >= s[l2 + k]) ++l2;
        if (l2 > -k && !(v >= s[l2 + k - 1])) --l2;
        return l2;
    }
    return v < 0.f ? -lv : lv;
}

template <int QM>
__device__ __forceinline__ int tc_q(float v, const float* thr, int k, float inv_step, unsigned& flags, int tbits = 8)
{
    if constexpr (QM == QM_UNIFORM) return tc_level_uniform(v, thr, k, inv_step, flags);
    if (v != v) flags |= SF_NONFINITE;
    if constexpr (QM == QM_K1) return level_k1(v, thr[0], thr[1]);
    else return level_bsearch(v, thr, tbits) - k;
}

// quantise 4 samples exactly -> packed int8 word (statistics are taken
// from the packed word by tc_word_stats)
template <int QM>
__device__ __forceinline__ uint32_t tc_q4(float4 v, const float* thr, int k, float inv_step, int tbits,
                                          unsigned& ss, unsigned& nz, unsigned& fl)
{
    const int c0 = tc_q<QM>(v.x, thr, k, inv_step, fl, tbits), c1 = tc_q<QM>(v.y, thr, k, inv_step, fl, tbits);
    const int c2 = tc_q<QM>(v.z, thr, k, inv_step, fl, tbits), c3 = tc_q<QM>(v.w, thr, k, inv_step, fl, tbits);
    (void)ss;
    (void)nz;
    return (uint32_t)(c0 & 0xff) | ((uint32_t)(c1 & 0xff) << 8) | ((uint32_t)(c2 & 0xff) << 16) |
           ((uint32_t)c3 << 24);
}

// branch-free magic-rounding levels of 4 samples; `bad` is raised for a
// sample near a rounding half-point, or NaN/inf (all rare): the caller then
// recomputes the word exactly with tc_q4
__device__ __forceinline__ uint32_t tc_q4_uniform_fast(float4 v, int k, float inv_step, bool& bad)
{
    const float e[4] = {v.x, v.y, v.z, v.w};
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float a = fabsf(e[i]);
        const float t = fmaf(a, inv_step, 12582912.0f);
        const int lv = min(__float_as_int(t) - 0x4B400000, k);
        const float d = fmaf(a, inv_step, -(t - 12582912.0f));
        bad |= !(fabsf(fabsf(d) - 0.5f) >= 0x1p-14f);
        const int c = e[i] < 0.f ? -lv : lv;
        w |= (uint32_t)(c & 0xff) << (8 * i);
    }
    return w;
}

__device__ __forceinline__ void tc_word_stats(uint32_t w, unsigned& ss, unsigned& nz)
{
    ss += (unsigned)__dp4a((int)w, (int)w, 0);
    nz += (unsigned)__popc(__vcmpne4(w, 0u)) >> 3;
}

// NV float4s -> NV packed code words: branch-free for uniform quantisers
// (one rare exact redo of all NV words), exact compares otherwise
template <int QM, int NV>
__device__ __forceinline__ void tc_quant_words(const float4 (&v)[NV], const float* thr, int k, float inv_step,
                                               int tbits, uint32_t (&w)[NV], unsigned& fl)
{
    unsigned d0 = 0, d1 = 0;
    if constexpr (QM == QM_UNIFORM) {
        bool bad = false;
#pragma unroll
        for (int h = 0; h < NV; ++h) w[h] = tc_q4_uniform_fast(v[h], k, inv_step, bad);
        if (__builtin_expect(bad, 0)) {
#pragma unroll
            for (int h = 0; h < NV; ++h) w[h] = tc_q4<QM>(v[h], thr, k, inv_step, 8, d0, d1, fl);
        }
    } else {
#pragma unroll
        for (int h = 0; h < NV; ++h) w[h] = tc_q4<QM>(v[h], thr, k, inv_step, tbits, d0, d1, fl);
    }
}

// the PITCH byte-shifted copies of slot xs's x codes into B buffer bs
// (chunk (kc, r) = x[16kc - r, +16) at kc*LBO + (r/8)*128 + (r%8)*16):
// item -> (chunk kc, group h of 8 shifts) with h uniform per warp; the
// thread loads the 16*(PITCH/16+1) source bytes once and emits 8 shifts
template <int PITCH>
__device__ __forceinline__ void tc_build_copies(const TcArgs& a, TcSmem& S, int xs, int bs)
{
    constexpr int NH = PITCH / 8, NW = 4 * (PITCH / 16 + 1), LBO = PITCH == 32 ? kTcBLbo32 : kTcBLbo;
    const uint4* xq = reinterpret_cast<const uint4*>(S.xl[xs]);
    uint4* b4 = reinterpret_cast<uint4*>(S.b + bs * kTcBSlot);
    const int nchunk = a.K / 16;
    const int nitems = 32 * NH * ((nchunk + 31) / 32);
    for (int i = threadIdx.x; i < nitems; i += kTcThreads) {
        const int kc = (i & 31) + 32 * (i / (32 * NH)), h = (i >> 5) % NH;
        if (kc >= nchunk) continue;
        // xl bytes [16kc + kTcXPad - PITCH, +NW*4) = x[16kc - PITCH, 16kc + 16)
        uint32_t w[NW + 1];
#pragma unroll
        for (int q = 0; q < NW / 4; ++q) {
            const uint4 v = xq[kc + (kTcXPad - PITCH) / 16 + q];
            w[4 * q] = v.x;
            w[4 * q + 1] = v.y;
            w[4 * q + 2] = v.z;
            w[4 * q + 3] = v.w;
        }
        w[NW] = 0u;
        uint4* dst = b4 + kc * (LBO / 16) + h * 8;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
            if (hh != h) continue;  // warp-uniform
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // r = 8hh + j: window bytes [PITCH - r, PITCH - r + 16)
                const int o = PITCH - (8 * hh + j), wq = o >> 2, sh = (o & 3) * 8;
                uint4 v;
                v.x = __funnelshift_r(w[wq], w[wq + 1], sh);
                v.y = __funnelshift_r(w[wq + 1], w[wq + 2], sh);
                v.z = __funnelshift_r(w[wq + 2], w[wq + 3], sh);
                v.w = __funnelshift_r(w[wq + 3], w[wq + 4 <= NW ? wq + 4 : NW], sh);
                dst[j] = v;
            }
        }
    }
}

// zero the margins of the code buffers: x words outside [XP, XP + nx4) of
// slot xs (nx4 < 0: leave x alone), y words of slot s outside the signal
// (front [0, yf), back [yb, Y))
template <int PITCH = 16>
__device__ __forceinline__ void tc_zero_margins(const TcArgs& a, TcSmem& S, int xs, int nx4, int s, int ny4)
{
    constexpr int XP = kTcXPad / 4;
    uint32_t* xw = reinterpret_cast<uint32_t*>(S.xl[xs]);
    uint32_t* yw = reinterpret_cast<uint32_t*>(S.y[s]);
    const int yoff = (int)(-a.L0) >> 2;  // word index of y[0] in the window (may be < 0)
    const int X = (a.K + 96) / 4, Y = (a.ylen + 3) / 4;
    const int yf = min(max(yoff, 0), Y), yb = min(max(yoff + ny4, yf), Y);
    const int nxz = nx4 < 0 ? 0 : X - nx4, nyz = yf + (Y - yb);
    for (int i = threadIdx.x; i < nxz + nyz; i += kTcThreads) {
        if (i < nxz) xw[i < XP ? i : nx4 + i] = 0;
        else {
            const int j = i - nxz;
            yw[ysw<PITCH>(j < yf ? j : yb + (j - yf))] = 0;
        }
    }
}

// shared-x mode prologue: the template's codes (slot 0), its 16 shifted
// copies (B slot 0) and statistics (S.xst), once per CTA
template <int QM>
__device__ void tc_build_template(const TcArgs& a, TcSmem& S)
{
    const float* thrx = reinterpret_cast<const float*>(S.thr[0]);
    const float* xs = reinterpret_cast<const float*>(a.op[0].data);
    const int nx = (int)a.op[0].n, nx4 = (nx + 3) >> 2;
    if (threadIdx.x < 3) S.xst[threadIdx.x] = 0;
    float4 v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) v[h] = tc_ld4(xs, threadIdx.x + h * kTcThreads, nx);
    uint32_t w[2];
    unsigned fl = 0, ss = 0, nz = 0;
    tc_quant_words<QM, 2>(v, thrx, a.op[0].q.k, (float)a.op[0].q.inv_step, a.op[0].q.tbits, w, fl);
    uint32_t* xw = reinterpret_cast<uint32_t*>(S.xl[0]);
    constexpr int XP = kTcXPad / 4;
    const int X = (a.K + 96) / 4;
    for (int i = threadIdx.x; i < X; i += kTcThreads)
        if (i < XP || i >= XP + nx4) xw[i] = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = threadIdx.x + h * kTcThreads;
        tc_word_stats(w[h], ss, nz);
        if (i < nx4) xw[XP + i] = w[h];
    }
    ss = __reduce_add_sync(0xffffffffu, ss);
    nz = __reduce_add_sync(0xffffffffu, nz);
    fl = __reduce_or_sync(0xffffffffu, fl);
    asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");  // codes + zeroed xst visible
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&S.xst[0], ss);
        atomicAdd(&S.xst[1], nz);
        atomicOr(&S.xst[2], fl);
    }
    tc_build_copies<32>(a, S, 0, 0);
    asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");  // xst complete
}

// shared-x mode, one pair: only the y row (<= 8192 samples, 4 float4 per
// thread) into the swizzled pitch-32 buffer; the template statistics ride in
// builder warp 0's record
template <int QM>
__device__ void tc_build_tmpl(const TcArgs& a, TcSmem& S, int s, int u, const TcRegs<true>& r, bool first)
{
    const float* thry = reinterpret_cast<const float*>(S.thr[1]);
    const int ny = (int)a.op[1].n, ny4 = (ny + 3) >> 2;
    if (first) tc_zero_margins<32>(a, S, 0, -1, s, ny4);  // margins are the same for every pair
    uint32_t w[4];
    unsigned fl = 0, ssy = 0, nzy = 0;
    tc_quant_words<QM, 4>(r.y, thry, a.op[1].q.k, (float)a.op[1].q.inv_step, a.op[1].q.tbits, w, fl);
    uint32_t* yw = reinterpret_cast<uint32_t*>(S.y[s]);
    const int yoff = (int)(-a.L0) >> 2, Y = (a.ylen + 3) / 4;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int i = threadIdx.x + h * kTcThreads;
        tc_word_stats(w[h], ssy, nzy);
        const int wi = yoff + i;
        if (i < ny4 && wi >= 0 && wi < Y) yw[ysw<32>(wi)] = w[h];
    }
    const bool w0 = threadIdx.x == 0;
    tc_aux_finish<2>(S, u, w0 ? S.xst[0] : 0u, w0 ? S.xst[1] : 0u, ssy, nzy, fl | (w0 ? S.xst[2] : 0u));
}

template <int QM>
__device__ void tc_build_fast(const TcArgs& a, TcSmem& S, int s, int u, const TcRegs<false>& r, bool first)
{
    const float* thrx = reinterpret_cast<const float*>(S.thr[0]);
    const float* thry = reinterpret_cast<const float*>(S.thr[1]);
    const int nx4 = (int)(a.op[0].n >> 2), ny4 = (int)(a.op[1].n >> 2);
#ifdef QX_TC_TIMING
    long long _m = clock64();
#define TC_MARK(i) if (threadIdx.x == 0) { const long long _n = clock64(); atomicAdd(&S.tm[i], (unsigned long long)(_n - _m)); _m = _n; }
#else
#define TC_MARK(i)
#endif
    if (first) tc_zero_margins(a, S, s, nx4, s, ny4);  // margins are the same for every pair
    TC_MARK(8);
    // samples past n were fetched as zeros: code 0, no statistics
    unsigned ssx = 0, nzx = 0, ssy = 0, nzy = 0, fl = 0;
    uint32_t wx[2], wy[2];
    tc_quant_words<QM, 2>(r.x, thrx, a.op[0].q.k, (float)a.op[0].q.inv_step, a.op[0].q.tbits, wx, fl);
    tc_quant_words<QM, 2>(r.y, thry, a.op[1].q.k, (float)a.op[1].q.inv_step, a.op[1].q.tbits, wy, fl);
    uint32_t* xw = reinterpret_cast<uint32_t*>(S.xl[s]);
    uint32_t* yw = reinterpret_cast<uint32_t*>(S.y[s]);
    const int yoff = (int)(-a.L0) >> 2, Y = (a.ylen + 3) / 4;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = threadIdx.x + h * kTcThreads;
        tc_word_stats(wx[h], ssx, nzx);
        tc_word_stats(wy[h], ssy, nzy);
        if (i < nx4) xw[kTcXPad / 4 + i] = wx[h];
        const int wi = yoff + i;
        if (i < ny4 && wi >= 0 && wi < Y) yw[wi] = wy[h];
    }
    TC_MARK(9);
    asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");  // builders only
    TC_MARK(10);
    tc_build_copies<16>(a, S, s, s);
    TC_MARK(11);
    tc_aux_finish<1>(S, u, ssx, nzx, ssy, nzy, fl);
    TC_MARK(12);
}

// Extra lags of the pair in data slot s (aux slot u), run by the lag warps
// after the hand-off barrier: j = ntiles*pitch*M + e, sum_m x[m] *
// ycode[L0 + j + m] over packed words (dp4a), one record per lag warp.
template <int PITCH>
__device__ void tc_extra_lags(const TcArgs& a, TcSmem& S, int s, int u, int xs)
{
    const int lane = threadIdx.x & 31, lw = (threadIdx.x >> 5) - kTcLagWarp0;
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(S.xl[xs]) + kTcXPad / 4;  // x codes from m = 0
    const uint32_t* yw = reinterpret_cast<const uint32_t*>(S.y[s]);
    const int nw = (int)((a.op[0].n + 3) >> 2);
    const int j0 = a.ntiles * a.pitch * a.M;
    for (int e = 0; e < a.extra; ++e) {
        const int j = j0 + e, jw = j >> 2, sh = (j & 3) * 8;
        int acc = 0;
        for (int w = lw * 32 + lane; w < nw; w += 32 * kTcLagWarps)
            acc = __dp4a((int)xw[w], (int)__funnelshift_r(yw[ysw<PITCH>(w + jw)], yw[ysw<PITCH>(w + jw + 1)], sh),
                         acc);
        acc = __reduce_add_sync(0xffffffffu, acc);
        if (lane == 0) S.wxs[u][lw][e] = acc;
    }
}

// final statistics of the pair in aux slot u from the builder warps'
// records (lane w < 16 holds warp w's), by one lag warp after the hand-off
__device__ void tc_final_stats(const TcArgs& a, TcSmem& S, int u)
{
    constexpr int kW = kTcThreads / 32;
    const int lane = threadIdx.x & 31;
    unsigned long long r[5];
    if (a.fast) {
        // per-pair totals fit 32 bits (n <= 8192, k <= 127): one REDUX per field
        unsigned v[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) v[i] = lane < kW ? (unsigned)S.wst[u][lane][i] : 0u;
        r[0] = __reduce_add_sync(0xffffffffu, v[0]);
        r[1] = __reduce_add_sync(0xffffffffu, v[1]);
        r[2] = __reduce_add_sync(0xffffffffu, v[2]);
        r[3] = __reduce_add_sync(0xffffffffu, v[3]);
        r[4] = __reduce_or_sync(0xffffffffu, v[4]);
    } else {
        unsigned long long sum = 0;
        if (lane < 5)
            for (int w = 0; w < kW; ++w) {
                const unsigned long long x = S.wst[u][w][lane];
                sum = lane == 4 ? (sum | x) : sum + x;
            }
#pragma unroll
        for (int i = 0; i < 5; ++i) r[i] = __shfl_sync(0xffffffffu, sum, i);
    }
    if (lane < 5) S.fst[u][lane] = lane == 0 ? r[0] : lane == 1 ? r[1] : lane == 2 ? r[2] : lane == 3 ? r[3] : r[4];
}

// argmax epilogue of the pair in aux slot u, run by warps 20..23 only (warp
// w reads TMEM lane quarter w%4; M=128: lane = row, M=64: rows 16q..16q+15
// sit in lanes 32q..32q+15), reduced behind a 128-thread named barrier so
// the builders keep going; merges the builders' extra-lag sums and writes
// the qx_result with the statistics from shared memory.
constexpr int kEpiWarp0 = 20;

__device__ __forceinline__ void best_add(long long& bv, long long& bt, long long& bc, long long v, long long t,
                                         long long c)
{
    if (v > bv) { bv = v; bt = t; bc = c; }
    else if (v == bv) { bt = min(bt, t); bc += c; }
}

template <int PITCH>
__device__ void tc_epilogue(const TcArgs& a, TcSmem& S, int u, int64_t pair)
{
    const int lane = threadIdx.x & 31;
    const int q = (threadIdx.x >> 5) - kEpiWarp0;  // 0..3 = TMEM lane quarter
    const int tl = PITCH * a.M;
    const int row = a.M == 128 ? q * 32 + lane : q * 16 + lane;
    const bool live = a.M == 128 || lane < 16;
    // window in tile-relative lag index j = lag - L0 (t = L0 + j + nx - 1)
    const int64_t tbase = a.L0 + a.op[0].n - 1;
    const int jlo = (int)(a.am.t_lo - tbase), jhi = (int)(a.am.t_hi - tbase);
    // 32-bit branch-free scan: |value| < 2^31 - 1 (eligibility), so INT_MIN
    // marks out-of-window entries and INT_MIN + 1 is below every value; j
    // increases along the scan, so the first maximum is the smallest lag
    int bv = INT_MIN + 1, bj = INT_MAX, bc = 0;
#ifdef QX_TC_TIMING
    long long _e = clock64();
#define TC_EMARK(i) if (threadIdx.x == kEpiWarp0 * 32) { const long long _n = clock64(); atomicAdd(&S.tm[i], (unsigned long long)(_n - _e)); _e = _n; }
#else
#define TC_EMARK(i)
#endif
    for (int tile = 0; tile < a.ntiles; ++tile) {
#pragma unroll
        for (int c0 = 0; c0 < PITCH; c0 += 16) {
            int v[16];
            const uint32_t taddr =
                S.tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(u * 32 + tile * PITCH + c0);
            tmem_ld16(taddr, v);
            const int j0 = tile * tl + PITCH * row + c0;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int j = j0 + r;
                const int val = (live && j >= jlo && j <= jhi) ? v[r] : INT_MIN;
                const bool gt = val > bv, eq = val == bv;
                bj = gt ? j : bj;
                bc = gt ? 1 : bc + (int)eq;
                bv = gt ? val : bv;
            }
        }
    }
    // TMEM reads are complete (wait::ld) before the slot is released
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    TC_EMARK(13);
    // warp (value, smallest j, count) by REDUX: the max, then the min j and
    // the summed count of the lanes holding it (empty lanes: INT_MIN + 1, 0)
    {
        const int mv = __reduce_max_sync(0xffffffffu, bv);
        const bool at = bv == mv;
        bj = __reduce_min_sync(0xffffffffu, at ? bj : INT_MAX);
        bc = __reduce_add_sync(0xffffffffu, at ? bc : 0);
        bv = mv;
    }
    TC_EMARK(14);
    // per-aux-slot records: the epilogue warps are never a pair apart (the
    // barrier below), so the slot written here is not being read
    if (lane == 0) {
        S.best[u][q][0] = bv;
        S.best[u][q][1] = bj;
        S.best[u][q][2] = bc;
    }
    asm volatile("bar.sync 4, 128;" ::: "memory");
    if (q == 0) {
        const unsigned long long* fs = S.fst[u];  // summed by the lag warps
        const unsigned long long ssx = fs[0], nzx = fs[1], ssy = fs[2], nzy = fs[3], fls = fs[4];
        // the four warp records by REDUX (lanes 0..3)
        const int wv = lane < 4 ? S.best[u][lane][0] : INT_MIN;
        const int mv = __reduce_max_sync(0xffffffffu, wv);
        const bool at = lane < 4 && wv == mv;
        const int mj = __reduce_min_sync(0xffffffffu, at ? S.best[u][lane][1] : INT_MAX);
        const int mc = __reduce_add_sync(0xffffffffu, at ? S.best[u][lane][2] : 0);
        long long v0 = LLONG_MIN, t0 = LLONG_MAX, c0 = 0;
        if (mc) best_add(v0, t0, c0, mv, tbase + mj, mc);

        for (int e = 0; e < a.extra; ++e) {
            const int xs = __reduce_add_sync(0xffffffffu, lane < kTcLagWarps ? S.wxs[u][lane][e] : 0);
            const int j = a.ntiles * tl + e;
            if (j < jlo || j > jhi) continue;
            best_add(v0, t0, c0, xs, tbase + j, 1);
        }
        int flags = 0;
        if (nzx == 0) flags |= 1;
        if (nzy == 0) flags |= 2;
        if (fls & SF_NONFINITE) flags |= 4;
        const int status = (flags & 4) ? 9 : ((flags & 3) ? 2 : 0);
        long long f = ((long long)status << 32) | (unsigned)flags;
        f = lane == 0 ? v0 : lane == 1 ? a.am.first_lag + t0 : lane == 2 ? c0 : lane == 3 ? (long long)ssx
          : lane == 4 ? (long long)ssy : lane == 5 ? (long long)nzx : lane == 6 ? (long long)nzy : f;
        if (lane < 8) reinterpret_cast<long long*>(a.am.results)[pair * 8 + lane] = f;
    }
    TC_EMARK(15);
}

#ifdef QX_TC_TIMING
#define TC_T0() const long long _t0 = clock64()
#define TC_ACC(i) atomicAdd(&S.tm[i], (unsigned long long)(clock64() - _t0))
#else
#define TC_T0() ((void)0)
#define TC_ACC(i) ((void)0)
#endif

template <typename T, int QM, bool SX>
__global__ void __launch_bounds__(kTcTotalThreads, 1) k_tc_window(const __grid_constant__ TcArgs a)
{
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    TcSmem& S = *reinterpret_cast<TcSmem*>(tc_smem_raw);
    // warp index through a shuffle: provably warp-uniform, so the role
    // branches keep descriptor arithmetic in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kMaxThr; i += kTcTotalThreads) {
        reinterpret_cast<T*>(S.thr[0])[i] = (T)a.op[0].q.thr[i];
        reinterpret_cast<T*>(S.thr[1])[i] = (T)a.op[1].q.thr[i];
    }
    if (threadIdx.x < kTcAux) {
        mbar_init(&S.mdone[threadIdx.x], 1);
        mbar_init(&S.tfree[threadIdx.x], 128);
        mbar_init(&S.xdone[threadIdx.x], 32 * kTcLagWarps);
    }
#ifdef QX_TC_TIMING
    if (threadIdx.x < 16) S.tm[threadIdx.x] = 0;
#endif
    if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&S.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // Dependencies (iteration it: data slot it & 1, aux slot it & 3):
    //   build(it)    after MMA(it-2) [data slot] and epilogue(it-4) [aux slot]
    //   MMA(it)      after build(it) [named barrier] and epilogue(it-4) [TMEM]
    //   epilogue(it) after MMA(it)
    const int64_t npairs = a.batch > blockIdx.x ? (a.batch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (warp < kTcThreads / 32) {
        // ---- builders
        auto acquire = [&](int it) {
            TC_T0();
            if (it >= 2) tc_wait_mdone(S, it - 2);
            if (it >= 2) tc_wait_xdone(S, it - 2);  // lag warps done reading the data slot
            if (it >= 4) tc_wait_tfree(S, it - 4);
            if (threadIdx.x == 0) TC_ACC(0);
        };
        auto handoff = [&](int it) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> async proxy
            // alternating barrier ids keep consecutive iterations apart
            if (it & 1) asm volatile("bar.arrive 3, %0;" ::"n"(kTcHandoff) : "memory");
            else asm volatile("bar.arrive 2, %0;" ::"n"(kTcHandoff) : "memory");
        };
        bool fast = false;
        if constexpr (std::is_same<T, float>::value) fast = a.fast;
        if (fast) {
            if constexpr (std::is_same<T, float>::value) {
                TcRegs<SX> cur, nxt;
                if (npairs) tc_fetch<SX>(a, blockIdx.x, cur);
                if constexpr (SX) {
                    if (npairs) tc_build_template<QM>(a, S);
                }
                for (int p = 1; p < kTcPrefetch && p < npairs; ++p)
                    tc_prefetch_l2<SX>(a, blockIdx.x + (int64_t)p * gridDim.x);
                for (int it = 0; it < npairs; ++it) {
                    const int64_t pair = blockIdx.x + (int64_t)it * gridDim.x;
                    if (it + kTcPrefetch < npairs) tc_prefetch_l2<SX>(a, pair + (int64_t)kTcPrefetch * gridDim.x);
                    if (it + 1 < npairs) tc_fetch<SX>(a, pair + gridDim.x, nxt);
                    acquire(it);
                    TC_T0();
#ifdef QX_TC_TIMING
                    if (!(a.debug & 2))
#endif
                    {
                        if constexpr (SX) tc_build_tmpl<QM>(a, S, it & 1, it & 3, cur, it < 2);
                        else tc_build_fast<QM>(a, S, it & 1, it & 3, cur, it < 2);
                    }
                    if (threadIdx.x == 0) TC_ACC(1);
                    handoff(it);
                    cur = nxt;
                }
            }
        } else {
            for (int it = 0; it < npairs; ++it) {
                const int64_t pair = blockIdx.x + (int64_t)it * gridDim.x;
                acquire(it);
                tc_build<T, QM>(a, S, it & 1, it & 3, pair);
                handoff(it);
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ---- MMA issuer: the whole warp runs the loop, one elected lane issues
        const int nk = a.K / 32;
        for (int it = 0; it < npairs; ++it) {
            const int s = it & 1, u = it & 3;
            {
                TC_T0();
                if (it & 1) asm volatile("bar.sync 3, %0;" ::"n"(kTcHandoff) : "memory");
                else asm volatile("bar.sync 2, %0;" ::"n"(kTcHandoff) : "memory");
                if (lane == 0) TC_ACC(2);
            }
            {
                TC_T0();
                if (it >= 4) tc_wait_tfree(S, it - 4);  // TMEM slot drained
                if (lane == 0) TC_ACC(4);
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            TC_T0();
            // pitch 32 (shared template): one B buffer built once, SW32 A rows
            constexpr int PITCH = SX ? 32 : 16, LBO = SX ? kTcBLbo32 : kTcBLbo, BINC = 2 * LBO / 16;
            const uint32_t ya = smem_u32(S.y[s]), ba = smem_u32(S.b + (SX ? 0 : s) * kTcBSlot);
            const uint64_t bd0 = smem_desc(ba, LBO, 128);
            const uint32_t tbase = __shfl_sync(0xffffffffu, S.tmem_base, 0);
            for (int tile = 0; tile < a.ntiles; ++tile) {
#ifdef QX_TC_TIMING
                if (a.debug & 1) break;
#endif
                const uint32_t d = tbase + (uint32_t)(u * 32 + tile * PITCH);
                const uint64_t ad0 = smem_desc(ya + tile * PITCH * a.M, 16, 8 * PITCH) |
                                     (PITCH == 32 ? (6ull << 61) : 0ull);  // layout SWIZZLE_32B
                const uint32_t ahi = (uint32_t)(ad0 >> 32), bhi = (uint32_t)(bd0 >> 32);
                uint32_t alo = (uint32_t)ad0, blo = (uint32_t)bd0;
                mma_i8_warp(d, ad0, bd0, a.idesc, 0);
                int kk = 1;
                for (; kk + 4 <= nk; kk += 4) {
                    mma_i8_warp4<BINC>(d, alo + 2, ahi, blo + BINC, bhi, a.idesc);
                    alo += 8;
                    blo += 4 * BINC;
                }
                for (; kk < nk; ++kk) {
                    alo += 32 >> 4;  // next 32 k-bytes of A
                    blo += BINC;     // next two k-chunks of B
                    mma_i8_warp(d, ((uint64_t)ahi << 32) | alo, ((uint64_t)bhi << 32) | blo, a.idesc, 1);
                }
            }
            mma_commit_warp(&S.mdone[u]);
            __syncwarp();
            if (lane == 0) TC_ACC(5);
        }
    } else if (warp >= kTcLagWarp0 && warp < kTcLagWarp0 + kTcLagWarps) {
        // ---- lag warps: the extra lags of each pair from its code buffers
        for (int it = 0; it < npairs; ++it) {
            if (it & 1) asm volatile("bar.sync 3, %0;" ::"n"(kTcHandoff) : "memory");
            else asm volatile("bar.sync 2, %0;" ::"n"(kTcHandoff) : "memory");
            if (it >= 4) tc_wait_tfree(S, it - 4);  // epilogue done with this aux slot's records
            if (a.extra) tc_extra_lags<SX ? 32 : 16>(a, S, it & 1, it & 3, SX ? 0 : (it & 1));
            if (warp == kTcLagWarp0) tc_final_stats(a, S, it & 3);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.xdone[it & 3])) : "memory");
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ---- epilogue: TMEM -> argmax -> qx_result, then free the aux slot
        for (int it = 0; it < npairs; ++it) {
            const int64_t pair = blockIdx.x + (int64_t)it * gridDim.x;
            TC_T0();
            tc_wait_mdone(S, it);
            tc_wait_xdone(S, it);  // extra-lag records written
            if (threadIdx.x == kEpiWarp0 * 32) TC_ACC(3);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            {
                TC_T0();
                tc_epilogue<SX ? 32 : 16>(a, S, it & 3, pair);
                if (threadIdx.x == kEpiWarp0 * 32) TC_ACC(6);
            }
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.tfree[it & 3])) : "memory");
        }
    }
    // every MMA was waited on by the epilogue before TMEM is released
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef QX_TC_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("tc timing block0 npairs=%lld debug=%d (cycles/pair): build-wait %llu build %llu | mma: wait-handoff %llu "
               "wait-tfree %llu issue %llu | epi: wait %llu run %llu\n",
               (long long)npairs, a.debug, S.tm[0] / npairs, S.tm[1] / npairs, S.tm[2] / npairs, S.tm[4] / npairs,
               S.tm[5] / npairs, S.tm[3] / npairs, S.tm[6] / npairs);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("  build phases (cycles/pair): zero %llu quant %llu bar %llu copies %llu aux %llu | epi: tmem+scan %llu "
               "shfl %llu bars+merge %llu\n", S.tm[8] / npairs, S.tm[9] / npairs, S.tm[10] / npairs,
               S.tm[11] / npairs, S.tm[12] / npairs, S.tm[13] / npairs, S.tm[14] / npairs, S.tm[15] / npairs);
#endif
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(S.tmem_base));
}

// eligibility: window of at most kTcMaxTiles*2048 lags, nx + 15 <= kTcMaxK,
// |values| < 2^31 (nx * Kx * Ky), same input dtype and quantiser mode (float)
bool tc_i8_window_eligible(const NttCall& c, int64_t nx, int64_t ny)
{
    (void)ny;
    const int64_t W = c.am.t_hi - c.am.t_lo + 1;
    if (W > (int64_t)kTcMaxTiles * kTcLags + kTcMaxExtra) return false;
    if (nx + 15 > kTcMaxK) return false;
    if (c.op[0].dtype != c.op[1].dtype || c.op[0].dtype == DT_I64) return false;
    if (c.op[0].q.mode != c.op[1].q.mode) return false;
    if (c.op[0].q.k > 127 || c.op[1].q.k > 127) return false;
    if ((double)nx * c.op[0].q.k * c.op[1].q.k >= 2147483647.0) return false;
    return true;
}

template <typename T, int QM, bool SX = false>
static cudaError_t launch_tc(const TcArgs& a, cudaStream_t s, int sms)
{
    const size_t smem = sizeof(TcSmem);
    if (cudaError_t e = set_max_smem((const void*)k_tc_window<T, QM, SX>, smem); e != cudaSuccess) return e;
    const int grid = (int)(a.batch < sms ? a.batch : sms);
    k_tc_window<T, QM, SX><<<grid, kTcTotalThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t tc_i8_window_run(const NttCall& c, int64_t nx, cudaStream_t s)
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
    a.K = (int)(((nx + 15) + 31) / 32 * 32);
    const int64_t ny = c.op[1].n;
    const bool aligned = ((uintptr_t)c.op[0].data % 16 == 0) && ((uintptr_t)c.op[1].data % 16 == 0) &&
                         (a.L0 % 4 == 0) && (c.batch == 1 || c.op[1].ld % 4 == 0);
    // shared x (template search: every pair's x is the same row): the
    // template's 32 shifted copies are built once per CTA (pitch 32, one
    // M=128 tile of 4096 lags, y rows up to 8192 samples); otherwise per-pair
    // copies with pitch 16
    a.shared_x = c.op[0].dtype == DT_F32 && c.batch > 1 && c.op[0].ld == 0 && nx <= kTcFastN && nx % 4 == 0 &&
                 ny <= kTcFastNY && aligned && W <= 4096 + kTcMaxExtra;
    a.fast = a.shared_x || (c.op[0].dtype == DT_F32 && nx <= kTcFastN && ny <= kTcFastN && nx % 4 == 0 &&
                            ny % 4 == 0 && aligned && (c.batch == 1 || c.op[0].ld % 4 == 0));
    a.pitch = a.shared_x ? 32 : 16;
    // B copy r holds x at k = m + r: K covers nx + pitch - 1 (pitch 32 needs
    // more than the pitch-16 default for templates with nx % 32 outside 1..17)
    if (a.pitch == 32) a.K = (int)((nx + 31 + 31) / 32 * 32);
    // shape: pitch 16: one M=64 tile (1024 lags) when it covers the window up
    // to the extra lags, else M=128 tiles (2048 lags each); pitch 32: M=128
    a.M = (a.pitch == 16 && W <= 1024 + kTcMaxExtra) ? 64 : 128;
    const int tl = a.pitch * a.M;
    a.ntiles = (int)((W - kTcMaxExtra + tl - 1) / tl);
    if (a.ntiles < 1) a.ntiles = 1;
    a.extra = (int)(W > (int64_t)a.ntiles * tl ? W - (int64_t)a.ntiles * tl : 0);
    a.idesc = tc_idesc(a.M, a.pitch);
    a.ylen = a.ntiles * tl + kTcMaxExtra + a.K;
#ifdef QX_TC_TIMING
    if (const char* ev = getenv("QX_TC_DEBUG")) a.debug = atoi(ev);
#endif
    const int sms = device_sms();
    if (c.prof) c.prof->pre(KK_DIRECT, s);
    cudaError_t e;
    const int qm = c.op[0].q.mode;
    if (c.op[0].dtype == DT_F32 && a.shared_x) {
        if (qm == QM_K1) e = launch_tc<float, QM_K1, true>(a, s, sms);
        else if (qm == QM_UNIFORM) e = launch_tc<float, QM_UNIFORM, true>(a, s, sms);
        else e = launch_tc<float, QM_BSEARCH, true>(a, s, sms);
    } else if (c.op[0].dtype == DT_F32) {
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

}  // namespace i8
}  // namespace qx
