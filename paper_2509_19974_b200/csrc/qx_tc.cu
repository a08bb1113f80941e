// qx_tc.cu -- bounded-lag-window correlation on the 5th-generation tensor
// cores: the template-search fp4 modes (kind::mxf4 e2m1 x e2m1 -> exact f32,
// mode 2 on one SM, mode 3 on a CTA pair) and the block merge of
// qx_template_search.  tc_window_run sends the int8 modes (kind::i8, s8 x s8
// -> s32; modes 0 and 1 below) to qx_tc_i8.cu, whose role layout they are
// tuned for; the int8 paths of this kernel template are not instantiated.
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
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "qx_internal.h"

namespace qx {

constexpr int kTcThreads = 512;                 // builder threads (warps 0-15)
constexpr int kTcMmaWarp = 16;                   // MMA issuer
// lag warps (extra-lag dot products, final statistics) from warp 17: three in
// the int8 modes (whose per-pair hand-off they are part of), two in the fp4
// modes, where warp 19 is a dedicated merge warp (an fp4 pair's epilogue is
// long; an int8 pair's first epilogue warp merges instead)
constexpr int kTcLagWarp0 = 17, kTcLagWarps = 3;
template <int MODE>
struct TcRoles {
    static constexpr int NLAG = MODE >= 2 ? 2 : 3;
    static constexpr bool MERGE_WARP = MODE >= 2;
    // builders + MMA warp + lag warps (+ the mode-4 stager warps) meet at the hand-off
    static constexpr int HANDOFF = kTcThreads + 32 + 32 * NLAG + (MODE == 4 ? 128 : 0);
};
// mode 4: fp4 with the Hankel A operand in TMEM.  Stager warps 24-27 (one per
// TMEM lane quarter) copy each row's next 4 K-steps (32 words) from the y slot
// into TMEM with one 32-column tcgen05.st; A chunks of 16 K-steps alternate in
// a two-chunk TMEM ring with full/free mbarriers (tools/tc_fp4_tmema.cu: 32.5
// cycles per M128 N64 K64 MMA with A in TMEM vs 68 from shared memory)
constexpr int kT4StageWarp0 = 24;
constexpr int kT4Chunk = 16;    // K-steps per A chunk (8 TMEM columns each)
constexpr int kT4ACol = 128;    // TMEM columns 128..383: the two A chunks
constexpr int kT4Sf = 384;      // scale factors (2 accumulator slots x 64 columns below)
constexpr int tc_threads(int mode) { return mode == 4 ? 28 * 32 : 24 * 32; }
// builders + MMA warp + lag warps meet at the per-pair hand-off barrier

constexpr int kTcMergeWarp = 19;                 // per-pair merge + result record
// 24 warps = 6 per SM sub-partition: an 80-register budget (25 warps: 72)
constexpr int kTcTotalThreads = 24 * 32;         // + warp 16 (MMA), 19 (merge), 20-23 (epilogue)
constexpr int kTcLags = 2048;      // lags per M=128 tile (M=64: 1024)
constexpr int kTcMaxK = 4608;      // nx + 15 <= kTcMaxK (B buffer 16*K bytes)
constexpr int kTcMaxTiles = 2;     // lag tiles per pair
constexpr int kTcMaxExtra = 16;    // lags past the tiles, summed on CUDA cores
// 2-SM fp4 mode (cta_group::2, M = 256 = 128 Hankel rows per CTA): pitch
// 128 samples (64-B SW64 rows) = N = 128 template copies, 64 per CTA; one
// pair-block is 32768 lags, 16384 per CTA (tools/tc_fp4_2sm.cu: exact, 64-69
// cycles per M256 N128 K64 instruction = the fp4 peak, 2.1x the 1-SM mode)
constexpr int kF2Pitch = 128;
constexpr int kF2CtaLags = 128 * kF2Pitch;      // 16384
constexpr int kF2Lags = 2 * kF2CtaLags;         // 32768
constexpr int kF2Pad = 128;                     // template nibble front padding (samples)
constexpr int kF2Sf = 256;                      // TMEM scale-factor column (2 aux slots x 128 columns)
constexpr int kTcYBytesI8 = kTcMaxTiles * kTcLags + kTcMaxExtra + kTcMaxK + 64;
constexpr int kTcYBytesF2 = (kF2CtaLags + kTcMaxK + 2 * kF2Pad) / 2;
constexpr int kTcYBytes = kTcYBytesI8 > kTcYBytesF2 ? kTcYBytesI8 : kTcYBytesF2;
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
// shared-template fp4 mode (kind::mxf4, e2m1 codes, every scale 2^0): codes
// |c| <= 4 are exact e2m1 values and every partial sum is an integer below
// 2^24, so the f32 accumulator holds the exact correlation (tools/tc_fp4.cu:
// 0 mismatches, 68 cycles per M128 N64 K64 MMA vs 40 for the i8 M128 N32
// K32 one: 2.35x the lags x samples per cycle).  Samples are nibbles (sample
// 2i in the low nibble of byte i), so the 32-B SW32 Hankel row pitch is 64
// samples: 64 template copies (N = 64), one M=128 tile = 8192 lags.
constexpr int kF4Pitch = 64;
constexpr int kF4Lbo = 1040;                    // B K-chunk (32 samples = 16 B) stride: 65 16-B units (odd)
constexpr int kF4Lags = 128 * kF4Pitch;         // 8192
constexpr int kF4MaxCode = 4;                   // |code| bound of the e2m1 mode
constexpr int kF4Sf = 256;                      // TMEM column of the (constant) scale factors
constexpr int kTcFastNY4 = 8 * 3 * kTcThreads;  // fp4 mode: y rows up to 12288 samples (3 x 8 per thread)
static_assert(kF4Lbo * (kTcMaxK / 32 + 2) <= kTcBBytes, "fp4 B must fit the B buffer");

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
// CLUSTER: acquire at cluster scope (arrivals from the peer CTA of a pair)
template <bool CLUSTER = false>
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase)
{
    uint32_t done = 0;
    for (uint32_t spin = 0; !done; ++spin) {
        if constexpr (CLUSTER)
            asm volatile(
                "{\n\t.reg .pred P1;\n\t"
                "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, P1;\n}"
                : "=r"(done)
                : "r"(smem_u32(bar)), "r"(phase)
                : "memory");
        else
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

// arrive (release, cluster scope) on the same mbarrier of CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank)
{
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// instruction descriptor: kind::mxf4 block32, A = B = E2M1 (1), scale UE8M0 (bit 23), K = 64
constexpr uint32_t tc_idesc_f4(int M, int N)
{
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

// CG: cta_group (2: issued by the pair's leader CTA, operands and D split
// across the two CTAs of the cluster)
template <int CG = 1>
__device__ __forceinline__ void mma_f4_warp(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate, uint32_t sf)
{
    if constexpr (CG == 2)
        asm volatile(
            "{\n\t.reg .pred e, p;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n}" ::"r"(
                tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(sf));
    else
        asm volatile(
            "{\n\t.reg .pred e, p;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n}" ::"r"(
                tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(sf));
}

// fp4 MMA with the A operand in TMEM (mode 4)
__device__ __forceinline__ void mma_f4t_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                             uint32_t accumulate, uint32_t sf)
{
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n}" ::"r"(
            tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate), "r"(sf));
}

// four fp4 MMAs on consecutive K steps (64 samples = 32 B of A, two B chunks)
#define QX_F4_MMA4(CGS)                                                                                              \
    asm volatile(                                                                                                    \
        "{\n\t.reg .pred e;\n\t.reg .b64 a0, a1, a2, a3, b0, b1, b2, b3;\n\t.reg .b32 t;\n\t"                              \
        "mov.b64 a0, {%1, %2};\n\tadd.u32 t, %1, 2;\n\tmov.b64 a1, {t, %2};\n\t"                                       \
        "add.u32 t, %1, 4;\n\tmov.b64 a2, {t, %2};\n\tadd.u32 t, %1, 6;\n\tmov.b64 a3, {t, %2};\n\t"                   \
        "mov.b64 b0, {%3, %4};\n\tadd.u32 t, %3, %7;\n\tmov.b64 b1, {t, %4};\n\t"                                      \
        "add.u32 t, %3, %8;\n\tmov.b64 b2, {t, %4};\n\tadd.u32 t, %3, %9;\n\tmov.b64 b3, {t, %4};\n\t"                  \
        "elect.sync _|e, 0xffffffff;\n\t"                                                                            \
        "@e tcgen05.mma.cta_group::" CGS ".kind::mxf4.block_scale.block32 [%0], a0, b0, %5, [%6], [%6], 1;\n\t"         \
        "@e tcgen05.mma.cta_group::" CGS ".kind::mxf4.block_scale.block32 [%0], a1, b1, %5, [%6], [%6], 1;\n\t"         \
        "@e tcgen05.mma.cta_group::" CGS ".kind::mxf4.block_scale.block32 [%0], a2, b2, %5, [%6], [%6], 1;\n\t"         \
        "@e tcgen05.mma.cta_group::" CGS ".kind::mxf4.block_scale.block32 [%0], a3, b3, %5, [%6], [%6], 1;\n}" ::"r"(     \
            tmem_d),                                                                                                 \
        "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(sf), "n"(BINC), "n"(2 * BINC), "n"(3 * BINC))

template <int BINC, int CG = 1>
__device__ __forceinline__ void mma_f4_warp4(uint32_t tmem_d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                             uint32_t idesc, uint32_t sf)
{
    if constexpr (CG == 2) QX_F4_MMA4("2");
    else QX_F4_MMA4("1");
}
#undef QX_F4_MMA4

// 2-SM completion: arrives on the same mbarrier of both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar)
{
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(
            smem_u32(bar)),
        "h"((unsigned short)3)
        : "memory");
}

// eight samples of a 1-level quantiser (k = 1: thresholds t0 < t1, codes
// -1 / 0 / +1 = e2m1 0xA / 0 / 0x2) straight to a nibble word (sample i at
// bits 4i); nz += nonzero codes (= their sum of squares), NaN -> flags
__device__ __forceinline__ uint32_t tc_nib8_k1(const float4& a, const float4& b, float t0, float t1, unsigned& nz,
                                               unsigned& fl)
{
    const float e[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t w = 0;
    bool nan = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        w |= (e[i] >= t1 ? 0x2u : (e[i] >= t0 ? 0u : 0xAu)) << (4 * i);
        nan |= e[i] != e[i];
    }
    if (nan) {
        fl |= SF_NONFINITE;
        // a NaN sample is code 0 (the call fails on the flag)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (e[i] != e[i]) w &= ~(0xFu << (4 * i));
    }
    nz += __popc(w & 0x22222222u);
    return w;
}

// four int8 codes in [-4, 4] (bytes of w) -> four e2m1 nibbles (16 bits,
// code i at bits 4i): |c| -> {0, 2, 4, 5, 6} = |c| <= 2 ? 2|c| : |c| + 2,
// sign -> bit 3; byte-SIMD, no per-sample branches
__device__ __forceinline__ uint32_t tc_nib4(uint32_t w)
{
    const uint32_t a = __vabs4(w);
    const uint32_t big = __vcmpgtu4(a, 0x02020202u);
    const uint32_t m = (big & (a + 0x02020202u)) | (~big & (a << 1));
    const uint32_t n = m | ((w & 0x80808080u) >> 4);
    return __byte_perm(n | (n >> 4), 0u, 0x4420);
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

// 32 accumulator columns of this warp's lane quarter; completion by tmem_wait_ld()
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int* v)
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

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
    int pitch;               // Hankel row pitch / N: 16 (per-pair B), 32 (shared template, SW32 A),
                             // 64 (shared template, fp4 nibbles, SW32 A)
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
    uint64_t tfree[kTcAux];  // aux slot free again: TMEM drained, records read (merge warp, 32 arrivals)
    uint64_t edone[kTcAux];  // epilogue warps' records of the aux slot written (4 arrivals)
    // per-builder-warp partials (no atomics): ssx, nzx, ssy, nzy, flags
    unsigned long long wst[kTcAux][kTcThreads / 32][5];
    int wxs[kTcAux][kTcLagWarps][kTcMaxExtra];     // extra-lag sums, one record per lag warp
    uint64_t xdone[kTcAux];  // lag warps finished with the pair of aux slot (96 arrivals)
    uint64_t pready[2];      // 2-SM mode, leader CTA: the peer's data slot is built (1 remote arrival)
    uint64_t afull[2], afree[2];  // mode 4: A chunk staged in TMEM (4 stager warps) / consumed (commit)
    unsigned xst[3];      // shared-x mode: template ssx, nzx, flags (built once)
    uint32_t tmem_base;
    int best[kTcAux][4][3];                 // per epilogue warp (value, j, count), per aux slot
    unsigned long long fst[kTcAux][5];      // final statistics of the pair (lag warps)
#ifdef QX_TC_TIMING
    unsigned long long tm[20];
#endif
};

// Each aux barrier completes once per use of its slot (every AUX-th
// iteration; AUX = 4, or 2 in the 2-SM mode whose 128-column accumulators
// fill TMEM faster), so iteration j's completion has parity (j / AUX) & 1.
// Every waiter is at most one use behind (see the dependency notes in the
// kernel), so parity waits are unambiguous.
template <int AUX = 4, bool CLUSTER = false>
__device__ __forceinline__ void tc_wait_mdone(TcSmem& S, int j)
{
    mbar_wait<CLUSTER>(&S.mdone[j % AUX], (uint32_t)((j / AUX) & 1));
}
template <int AUX = 4, bool CLUSTER = false>
__device__ __forceinline__ void tc_wait_tfree(TcSmem& S, int j)
{
    mbar_wait<CLUSTER>(&S.tfree[j % AUX], (uint32_t)((j / AUX) & 1));
}
template <int AUX = 4>
__device__ __forceinline__ void tc_wait_edone(TcSmem& S, int j)
{
    mbar_wait(&S.edone[j % AUX], (uint32_t)((j / AUX) & 1));
}
template <int AUX = 4>
__device__ __forceinline__ void tc_wait_xdone(TcSmem& S, int j)
{
    mbar_wait(&S.xdone[j % AUX], (uint32_t)((j / AUX) & 1));
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
// MODE: 0 per-pair B, 1 shared template (i8), 2 shared template (fp4)
template <int MODE>
struct TcRegs {
    float4 x[2], y[2];
};
template <>
struct TcRegs<1> {
    float4 y[4];
};
template <>
struct TcRegs<2> {
    float4 y[6];  // samples 8(t + 512g) .. +8 in y[2g], y[2g + 1]
};
template <>
struct TcRegs<4> : TcRegs<2> {};  // mode 4 builds like mode 2
template <>
struct TcRegs<3> {
    float4 y[12];  // 2-SM: window samples y0 + 8(t + 512g) .. +8, g < 6 (one buffer, refilled after each build)
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

template <int MODE>
__device__ __forceinline__ void tc_fetch(const TcArgs& a, int64_t pair, TcRegs<MODE>& r)
{
    const float* ys = reinterpret_cast<const float*>(a.op[1].data) + pair * a.op[1].ld;
    const int ny = (int)a.op[1].n;
    if constexpr (MODE == 3) {
        const int f0 = kF2CtaLags / 4 * (int)cluster_rank();  // the CTA's window (float4s)
        const int Y = (a.ylen + 7) / 8;
#pragma unroll
        for (int g = 0; g < 6; ++g) {
            const int wi = (int)threadIdx.x + g * kTcThreads, i = f0 + 2 * wi;
            const bool in = wi < Y;
            r.y[2 * g] = in ? tc_ld4(ys, i, ny) : make_float4(0.f, 0.f, 0.f, 0.f);
            r.y[2 * g + 1] = in ? tc_ld4(ys, i + 1, ny) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    } else if constexpr (MODE == 2 || MODE == 4) {
#pragma unroll
        for (int g = 0; g < 3; ++g) {
            const int i = 2 * ((int)threadIdx.x + g * kTcThreads);
            r.y[2 * g] = tc_ld4(ys, i, ny);
            r.y[2 * g + 1] = tc_ld4(ys, i + 1, ny);
        }
    } else if constexpr (MODE == 1) {
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

// Bulk L2 prefetch (TMA engine) of a pair's y window kTcPrefetch pairs
// ahead: the builders hold at most the next pair in registers, so the one
// after it is pulled into L2 and its register loads wait on L2 rather than
// HBM latency.  One instruction, one lane.
#ifndef QX_TC_PREFETCH
#define QX_TC_PREFETCH 2
#endif
constexpr int kTcPrefetch = QX_TC_PREFETCH;
template <int MODE>
__device__ __forceinline__ void tc_prefetch_l2(const TcArgs& a, int64_t pair)
{
    if (threadIdx.x != 0) return;
    const float* ys = reinterpret_cast<const float*>(a.op[1].data) + pair * a.op[1].ld;
    int64_t s0 = 0;
    if constexpr (MODE == 3) s0 = (int64_t)kF2CtaLags * cluster_rank();
    int64_t cnt = a.ylen;
    if (s0 + cnt > a.op[1].n) cnt = a.op[1].n - s0;
    const uint32_t bytes = cnt > 0 ? (uint32_t)(cnt * 4) & ~15u : 0u;
    if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ys + s0), "r"(bytes) : "memory");
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
// fp4 modes: 64 nibble-shifted copies of the template from the linear
// nibble buffer S.xl[1] (sample m at nibble pad + m): chunk (kc, r) =
// x[32kc - (shift0 + r), +32) (16 B) at kc*kF4Lbo + (r/8)*128 + (r%8)*16
// (LBO kF4Lbo, SBO 128); shift0 = 64 * rank in the 2-SM mode
__device__ __forceinline__ void tc_build_copies_f4(const TcArgs& a, TcSmem& S, int pad, int shift0)
{
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(S.xl[1]);
    uint4* b4 = reinterpret_cast<uint4*>(S.b);
    const int nchunk = a.K / 32;
    for (int i = threadIdx.x; i < nchunk * kF4Pitch; i += kTcThreads) {
        const int r = i & (kF4Pitch - 1), kc = i / kF4Pitch;
        const int s0 = 32 * kc - (shift0 + r) + pad;  // nibble of x[32kc - shift0 - r]
        const int w0 = s0 >> 3, sh = (s0 & 7) * 4;
        const uint32_t w[5] = {xw[w0], xw[w0 + 1], xw[w0 + 2], xw[w0 + 3], xw[w0 + 4]};
        uint4 v;
        v.x = __funnelshift_r(w[0], w[1], sh);
        v.y = __funnelshift_r(w[1], w[2], sh);
        v.z = __funnelshift_r(w[2], w[3], sh);
        v.w = __funnelshift_r(w[3], w[4], sh);
        b4[kc * (kF4Lbo / 16) + (r >> 3) * 8 + (r & 7)] = v;
    }
}

// FM: 0 int8 copies (pitch 32), 1 fp4 (64 copies), 2 fp4 2-SM (this CTA's 64 of 128 copies)
template <int QM, int FM = 0>
__device__ void tc_build_template(const TcArgs& a, TcSmem& S)
{
    constexpr bool F4 = FM != 0;
    constexpr int PAD = FM == 2 ? kF2Pad : 64;  // nibble front padding >= the largest shift
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
    if constexpr (F4) {
        // nibble buffer: zero words [0, (K + PAD) / 8 + 16) (the copies read up to (K + PAD) / 8 + 4)
        uint32_t* xn = reinterpret_cast<uint32_t*>(S.xl[1]);
        for (int i = threadIdx.x; i < (a.K + PAD) / 8 + 16; i += kTcThreads) xn[i] = 0;
    }
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
    if constexpr (F4) {
        uint16_t* xh = reinterpret_cast<uint16_t*>(S.xl[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = threadIdx.x + h * kTcThreads;
            if (i < nx4) xh[PAD / 4 + i] = (uint16_t)tc_nib4(w[h]);  // samples 4i.. at nibble PAD + 4i
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");
        tc_build_copies_f4(a, S, PAD, FM == 2 ? 64 * (int)cluster_rank() : 0);
    } else {
        tc_build_copies<32>(a, S, 0, 0);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");  // xst complete
}

// fp4 mode, one pair: the y row (<= 12288 samples, 3 x 8 per thread) as
// e2m1 nibbles into the swizzled buffer (8 samples per word); the slot is
// zeroed on its first use, so samples past the row stay code 0
template <int QM>
__device__ void tc_build_tmpl4(const TcArgs& a, TcSmem& S, int s, int u, const TcRegs<2>& r, bool first)
{
    const float* thry = reinterpret_cast<const float*>(S.thr[1]);
    const int ny = (int)a.op[1].n;
    uint32_t* yw = reinterpret_cast<uint32_t*>(S.y[s]);
    if (first) {
        for (int i = threadIdx.x; i < kTcYStride / 4; i += kTcThreads) yw[i] = 0;
        asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");
    }
    uint32_t w[6];
    unsigned fl = 0, ssy = 0, nzy = 0;
    const int yoff = (int)(-a.L0) >> 3, Y = (a.ylen + 7) / 8;
    if constexpr (QM == QM_K1) {
        const float t0 = thry[0], t1 = thry[1];
#pragma unroll
        for (int g = 0; g < 3; ++g) {
            const int i = threadIdx.x + g * kTcThreads;
            const uint32_t wn = tc_nib8_k1(r.y[2 * g], r.y[2 * g + 1], t0, t1, nzy, fl);
            const int wi = yoff + i;
            if (8 * i < ny && wi >= 0 && wi < Y) yw[ysw<32>(wi)] = wn;
        }
        ssy = nzy;
        const bool w0 = threadIdx.x == 0;
        tc_aux_finish<2>(S, u, w0 ? S.xst[0] : 0u, w0 ? S.xst[1] : 0u, ssy, nzy, fl | (w0 ? S.xst[2] : 0u));
        return;
    }
    tc_quant_words<QM, 6>(r.y, thry, a.op[1].q.k, (float)a.op[1].q.inv_step, a.op[1].q.tbits, w, fl);
#pragma unroll
    for (int g = 0; g < 3; ++g) {
        const int i = threadIdx.x + g * kTcThreads;
        tc_word_stats(w[2 * g], ssy, nzy);
        tc_word_stats(w[2 * g + 1], ssy, nzy);
        const int wi = yoff + i;
        if (8 * i < ny && wi >= 0 && wi < Y) yw[ysw<32>(wi)] = tc_nib4(w[2 * g]) | (tc_nib4(w[2 * g + 1]) << 16);
    }
    const bool w0 = threadIdx.x == 0;
    tc_aux_finish<2>(S, u, w0 ? S.xst[0] : 0u, w0 ? S.xst[1] : 0u, ssy, nzy, fl | (w0 ? S.xst[2] : 0u));
}

// 2-SM fp4 mode, one pair: this CTA's y window, row samples [16384*rank,
// +16384 + K), as nibbles into the SW64-swizzled buffer (byte bits 4-5 ^=
// bits 7-8: Hankel rows 64 B apart).  Words of 8 samples: t + 512g, g < 6;
// g < 3 arrive prefetched (one pair ahead), g >= 3 are loaded here first and
// complete while the prefetched ones are quantised.  Statistics cover the
// window (the degeneracy test needs only "any nonzero"; the windows of the
// two CTAs cover the row).
__device__ __forceinline__ int ysw64(int wi) { return wi ^ (((wi >> 5) & 3) << 2); }

template <int QM>
__device__ void tc_build_tmpl2(const TcArgs& a, TcSmem& S, int s, int u, const TcRegs<3>& r, bool first)
{
    const float* thry = reinterpret_cast<const float*>(S.thr[1]);
    const int ny = (int)a.op[1].n;
    const int y0 = kF2CtaLags * (int)cluster_rank();  // first row sample of the window
    uint32_t* yw = reinterpret_cast<uint32_t*>(S.y[s]);
    if (first) {
        for (int i = threadIdx.x; i < kTcYStride / 4; i += kTcThreads) yw[i] = 0;
        asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads) : "memory");
    }
    const int Y = (a.ylen + 7) / 8;  // window words
    unsigned fl = 0, ssy = 0, nzy = 0;
    if constexpr (QM == QM_K1) {
        const float t0 = thry[0], t1 = thry[1];
#pragma unroll
        for (int g = 0; g < 6; ++g) {
            const int i = threadIdx.x + g * kTcThreads;
            const uint32_t w = tc_nib8_k1(r.y[2 * g], r.y[2 * g + 1], t0, t1, nzy, fl);
            if (i < Y && y0 + 8 * i < ny) yw[ysw64(i)] = w;
        }
        ssy = nzy;
    } else
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t w[6];
        const float4 v[6] = {r.y[6 * h], r.y[6 * h + 1], r.y[6 * h + 2], r.y[6 * h + 3], r.y[6 * h + 4], r.y[6 * h + 5]};
        tc_quant_words<QM, 6>(v, thry, a.op[1].q.k, (float)a.op[1].q.inv_step, a.op[1].q.tbits, w, fl);
#pragma unroll
        for (int g = 0; g < 3; ++g) {
            const int i = threadIdx.x + (3 * h + g) * kTcThreads;
            tc_word_stats(w[2 * g], ssy, nzy);
            tc_word_stats(w[2 * g + 1], ssy, nzy);
            if (i < Y && y0 + 8 * i < ny) yw[ysw64(i)] = tc_nib4(w[2 * g]) | (tc_nib4(w[2 * g + 1]) << 16);
        }
    }
    const bool w0 = threadIdx.x == 0;
    tc_aux_finish<2>(S, u, w0 ? S.xst[0] : 0u, w0 ? S.xst[1] : 0u, ssy, nzy, fl | (w0 ? S.xst[2] : 0u));
}

// shared-x mode, one pair: only the y row (<= 8192 samples, 4 float4 per
// thread) into the swizzled pitch-32 buffer; the template statistics ride in
// builder warp 0's record
template <int QM>
__device__ void tc_build_tmpl(const TcArgs& a, TcSmem& S, int s, int u, const TcRegs<1>& r, bool first)
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
__device__ void tc_build_fast(const TcArgs& a, TcSmem& S, int s, int u, const TcRegs<0>& r, bool first)
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
template <int PITCH, int NLAG>
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
        for (int w = lw * 32 + lane; w < nw; w += 32 * NLAG)
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

// warp (value, smallest j, count) by REDUX -- the max, then the min j and the
// summed count of the lanes holding it (empty lanes: INT_MIN + 1, 0) -- into
// the per-aux-slot record of warp q, read by the merge warp before it frees
// the slot (the next write of slot u follows mdone(it + AUX), after tfree(it))
__device__ __forceinline__ void tc_epi_record(TcSmem& S, int u, int q, int bv, int bj, int bc)
{
    // TMEM reads are complete (wait::ld) before the slot is released
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    const int mv = __reduce_max_sync(0xffffffffu, bv);
    const bool at = bv == mv;
    bj = __reduce_min_sync(0xffffffffu, at ? bj : INT_MAX);
    bc = __reduce_add_sync(0xffffffffu, at ? bc : 0);
    if ((threadIdx.x & 31) == 0) {
        S.best[u][q][0] = mv;
        S.best[u][q][1] = bj;
        S.best[u][q][2] = bc;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.edone[u])) : "memory");
    }
}

template <int PITCH, bool F4 = false>
__device__ void tc_epilogue(const TcArgs& a, TcSmem& S, int u)
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
    if constexpr (F4) {
        // f32 accumulators holding exact integers (|value| < 2^24): the same
        // scan in float (-FLT_MAX below every value, -inf out of window), one
        // conversion per thread at the end; a tile fully inside the window
        // (every full template-search block) skips the masks
        float fv = -FLT_MAX;
        const bool full = jlo <= 0 && jhi >= tl - 1;
        const uint32_t taddr = S.tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(u * kF4Pitch);
        if (full) {
            // the thread's 64 lags j = 64*row + c: max by a tree (no serial
            // compare chain), then the tie set as a 64-bit mask of c: count =
            // popc, smallest lag = first set bit
            int v[64];
            tmem_ld32(taddr, v);
            tmem_ld32(taddr + 32, v + 32);
            tmem_wait_ld();
            float m[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) m[i] = fmaxf(__int_as_float(v[i]), __int_as_float(v[i + 32]));
#pragma unroll
            for (int w = 16; w; w >>= 1)
#pragma unroll
                for (int i = 0; i < w; ++i) m[i] = fmaxf(m[i], m[i + w]);
            const float mx = m[0];
            unsigned lo = 0, hi = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                lo |= (__int_as_float(v[i]) == mx ? 1u : 0u) << i;
                hi |= (__int_as_float(v[i + 32]) == mx ? 1u : 0u) << i;
            }
            bc = __popc(lo) + __popc(hi);
            bj = PITCH * row + (lo ? __ffs(lo) - 1 : 31 + __ffs(hi));
            fv = mx;
        } else
#pragma unroll
        for (int c0 = 0; c0 < PITCH; c0 += 16) {
            int v[16];
            tmem_ld16(taddr + c0, v);
            const int j0 = PITCH * row + c0;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int j = j0 + r;
                const float val = (full || (j >= jlo && j <= jhi)) ? __int_as_float(v[r]) : -INFINITY;
                const bool gt = val > fv, eq = val == fv;
                bj = gt ? j : bj;
                bc = gt ? 1 : bc + (int)eq;
                fv = gt ? val : fv;
            }
        }
        bv = fv == -FLT_MAX ? INT_MIN + 1 : __float2int_rn(fv);
    } else
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
    TC_EMARK(13);
    tc_epi_record(S, u, q, bv, bj, bc);
    TC_EMARK(15);
}

// tcgen05.ld of 16 columns without the wait (completion: tmem_wait_ld)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, int (&v)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// 16 accumulator columns (lags j0 + c .. + 15) into the running (max,
// count, first column): chunk max by a tree, its tie mask, then one
// branch-free update (an equal chunk max adds its ties, a larger one restarts)
template <bool FULL>
__device__ __forceinline__ void f2_chunk(const int (&v)[16], int c, int j0, int jlo, int jhi, float& mx, int& cnt,
                                         int& first)
{
    float f[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        f[i] = __int_as_float(v[i]);
        if constexpr (!FULL) {
            const int j = j0 + c + i;
            f[i] = (j >= jlo && j <= jhi) ? f[i] : -INFINITY;
        }
    }
    float m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = fmaxf(f[i], f[i + 8]);
#pragma unroll
    for (int w = 4; w; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) m[i] = fmaxf(m[i], m[i + w]);
    const float lm = m[0];
    unsigned mask = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) mask |= (f[i] == lm ? 1u : 0u) << i;
    if (lm == -INFINITY) mask = 0;  // nothing in the window
    const int pc = __popc(mask);
    const bool newer = lm > mx, same = lm == mx;
    cnt = newer ? pc : cnt + (same ? pc : 0);
    first = (newer && mask) ? c + __ffs(mask) - 1 : first;
    mx = fmaxf(mx, lm);
}

// 2-SM fp4 epilogue: this CTA's 128 accumulator columns of TMEM slot u (the
// lane quarter's rows, 128 lags per thread: j = 16384*rank + 128*row + c),
// 16 columns at a time with the next load in flight; one TMEM pass
__device__ void tc_epilogue_f2(const TcArgs& a, TcSmem& S, int u)
{
    const int lane = threadIdx.x & 31;
    const int q = (threadIdx.x >> 5) - kEpiWarp0;
    const int row = q * 32 + lane;
    const int64_t tbase = a.L0 + a.op[0].n - 1;
    const int jlo = (int)(a.am.t_lo - tbase), jhi = (int)(a.am.t_hi - tbase);
    const int j0 = kF2CtaLags * (int)cluster_rank() + kF2Pitch * row;
    const bool full = __all_sync(0xffffffffu, jlo <= j0 && jhi >= j0 + kF2Pitch - 1);
    const uint32_t taddr = S.tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(u * kF2Pitch);
    float mx = -FLT_MAX;
    int cnt = 0, first = -1;
    int v0[16], v1[16];
    tmem_ld16_nw(taddr, v0);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < kF2Pitch; c += 32) {
        tmem_ld16_nw(taddr + c + 16, v1);
        if (full) f2_chunk<true>(v0, c, j0, jlo, jhi, mx, cnt, first);
        else f2_chunk<false>(v0, c, j0, jlo, jhi, mx, cnt, first);
        tmem_wait_ld();
        if (c + 32 < kF2Pitch) tmem_ld16_nw(taddr + c + 32, v0);
        if (full) f2_chunk<true>(v1, c + 16, j0, jlo, jhi, mx, cnt, first);
        else f2_chunk<false>(v1, c + 16, j0, jlo, jhi, mx, cnt, first);
        tmem_wait_ld();
    }
    const bool any = first >= 0;
    const int bv = any ? __float2int_rn(mx) : INT_MIN + 1;
    tc_epi_record(S, u, q, bv, any ? j0 + first : INT_MAX, any ? cnt : 0);
}

// merge warp: the pair's four epilogue records, the lag warps' extra-lag
// sums and statistics -> the qx_result; frees the aux slot (tfree) as soon as
// the records are in registers, so neither the epilogue warps nor the MMA
// warp wait for the merge and the result stores
// rec: the qx_result record index (pair, or 2*pair + rank in the 2-SM mode);
// notify: also free the slot in the leader CTA (2-SM peer: the leader's MMA
// writes this CTA's TMEM)
template <int PITCH, int NLAG>
__device__ void tc_merge(const TcArgs& a, TcSmem& S, int u, int64_t rec, bool notify = false, bool free_slot = true)
{
    const int lane = threadIdx.x & 31;
    const int tl = PITCH * a.M;
    const int64_t tbase = a.L0 + a.op[0].n - 1;
    const int jlo = (int)(a.am.t_lo - tbase), jhi = (int)(a.am.t_hi - tbase);
    {
        const unsigned long long* fs = S.fst[u];  // summed by the lag warps
        const unsigned long long ssx = fs[0], nzx = fs[1], ssy = fs[2], nzy = fs[3], fls = fs[4];
        // the four warp records by REDUX (lanes 0..3)
        const int wv = lane < 4 ? S.best[u][lane][0] : INT_MIN;
        const int wj = lane < 4 ? S.best[u][lane][1] : INT_MAX;
        const int wc = lane < 4 ? S.best[u][lane][2] : 0;
        int xs[kTcMaxExtra];
#pragma unroll
        for (int e = 0; e < kTcMaxExtra; ++e)
            xs[e] = e < a.extra ? __reduce_add_sync(0xffffffffu, lane < NLAG ? S.wxs[u][lane][e] : 0) : 0;
        // every record of slot u is in registers: free the slot
        if (free_slot) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.tfree[u])) : "memory");
        if (notify && lane == 0) mbar_arrive_remote(&S.tfree[u], 0);
        const int mv = __reduce_max_sync(0xffffffffu, wv);
        const bool at = lane < 4 && wv == mv;
        const int mj = __reduce_min_sync(0xffffffffu, at ? wj : INT_MAX);
        const int mc = __reduce_add_sync(0xffffffffu, at ? wc : 0);
        long long v0 = LLONG_MIN, t0 = LLONG_MAX, c0 = 0;
        if (mc) best_add(v0, t0, c0, mv, tbase + mj, mc);

#pragma unroll
        for (int e = 0; e < kTcMaxExtra; ++e) {
            const int j = a.ntiles * tl + e;
            if (e >= a.extra || j < jlo || j > jhi) continue;
            best_add(v0, t0, c0, xs[e], tbase + j, 1);
        }
        int flags = 0;
        if (nzx == 0) flags |= 1;
        if (nzy == 0) flags |= 2;
        if (fls & SF_NONFINITE) flags |= 4;
        const int status = (flags & 4) ? 9 : ((flags & 3) ? 2 : 0);
        long long f = ((long long)status << 32) | (unsigned)flags;
        f = lane == 0 ? v0 : lane == 1 ? a.am.first_lag + t0 : lane == 2 ? c0 : lane == 3 ? (long long)ssx
          : lane == 4 ? (long long)ssy : lane == 5 ? (long long)nzx : lane == 6 ? (long long)nzy : f;
        if (lane < 8) reinterpret_cast<long long*>(a.am.results)[rec * 8 + lane] = f;
    }
}

#ifdef QX_TC_TIMING
#define TC_T0() const long long _t0 = clock64()
#define TC_ACC(i) atomicAdd(&S.tm[i], (unsigned long long)(clock64() - _t0))
#else
#define TC_T0() ((void)0)
#define TC_ACC(i) ((void)0)
#endif

// MODE: 0 per-pair B (int8), 1 shared template (int8, pitch 32), 2 shared
// template (fp4, pitch 64), 3 shared template on a CTA pair (fp4, 2-SM MMA,
// pitch 128; launched as clusters of 2, rank 0 issues the MMAs)
template <typename T, int QM, int MODE>
__global__ void __launch_bounds__(tc_threads(MODE), 1) k_tc_window(const __grid_constant__ TcArgs a)
{
    static_assert(MODE == 2, "only the 1-SM fp4 mode is built (modes 3 and 4 are retired, see DESIGN.md 6)");
    constexpr bool T4 = MODE == 4;                   // fp4, A in TMEM (otherwise as mode 2)
    constexpr bool SX = MODE != 0, F4 = MODE == 2 || T4, F2 = MODE == 3, FP4 = MODE >= 2;
    constexpr int AUX = (F2 || T4) ? 2 : 4;          // accumulator / record slots
    constexpr uint32_t SFC = T4 ? kT4Sf : kF4Sf;     // TMEM column of the scale factors
    constexpr uint32_t kTmemCols = FP4 ? 512 : 128;  // fp4: accumulators + scale factors
    constexpr int PITCH = F2 ? kF2Pitch : F4 ? kF4Pitch : SX ? 32 : 16;
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    TcSmem& S = *reinterpret_cast<TcSmem*>(tc_smem_raw);
    // warp index through a shuffle: provably warp-uniform, so the role
    // branches keep descriptor arithmetic in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const uint32_t rank = F2 ? cluster_rank() : 0u;
    for (int i = threadIdx.x; i < kMaxThr; i += tc_threads(MODE)) {
        reinterpret_cast<T*>(S.thr[0])[i] = (T)a.op[0].q.thr[i];
        reinterpret_cast<T*>(S.thr[1])[i] = (T)a.op[1].q.thr[i];
    }
    if (threadIdx.x < kTcAux) {
        mbar_init(&S.mdone[threadIdx.x], 1);
        // 2-SM leader: its own merge warp + the peer's (remote) release of the slot
        // merge warp (+ the 2-SM peer's remote release); int8 modes: the 128
        // epilogue threads, after their first warp's merge
        mbar_init(&S.tfree[threadIdx.x], !TcRoles<MODE>::MERGE_WARP ? 128 : (F2 && rank == 0) ? 33 : 32);
        mbar_init(&S.edone[threadIdx.x], 4);
        mbar_init(&S.xdone[threadIdx.x], 32 * TcRoles<MODE>::NLAG);
        if (threadIdx.x < 2) mbar_init(&S.pready[threadIdx.x], 1);
        if (T4 && threadIdx.x < 2) {
            mbar_init(&S.afull[threadIdx.x], 4);
            mbar_init(&S.afree[threadIdx.x], 1);
        }
    }
#ifdef QX_TC_TIMING
    if (threadIdx.x < 20) S.tm[threadIdx.x] = 0;
    const long long k_t0 = clock64();
    unsigned long long k_g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(k_g0));
#endif
    if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (warp == 0) {
        if constexpr (F2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(&S.tmem_base)),
                         "n"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(&S.tmem_base)),
                         "n"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (FP4) {
        // scale factors: 32 columns of 0x7f bytes (ue8m0 2^0) in every lane,
        // written by the epilogue warps (warp w reaches lanes 32*(w%4)..)
        static_assert(kF4Sf == kF2Sf, "one scale-factor column for both fp4 modes");
        if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
            const uint32_t t = S.tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + SFC;
            const uint32_t v = 0x7f7f7f7fu;
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(t),
                "r"(v));
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    t + 16),
                "r"(v));
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // both CTAs of a pair: barriers initialised and TMEM allocated before any
    // remote arrive or 2-SM MMA
    if constexpr (F2) cluster_sync_all();

    // Dependencies (iteration it: data slot it & 1, aux slot it % AUX):
    //   build(it)    after MMA(it-2) [data slot] and epilogue(it-AUX) [aux slot]
    //   MMA(it)      after build(it) [named barrier; 2-SM: and the peer's, pready]
    //                and epilogue(it-AUX) [TMEM; 2-SM: of both CTAs]
    //   epilogue(it) after MMA(it)
    // 2-SM: a cluster shares its pair sequence (both CTAs build halves of it)
    const int64_t base = F2 ? (blockIdx.x >> 1) : blockIdx.x, stride = F2 ? (gridDim.x >> 1) : gridDim.x;
    const int64_t npairs = a.batch > base ? (a.batch - base + stride - 1) / stride : 0;
    if (warp < kTcThreads / 32) {
        // ---- builders
        auto acquire = [&](int it) {
            TC_T0();
            if (it >= 2) tc_wait_mdone<AUX>(S, it - 2);
            if (it >= 2) tc_wait_xdone<AUX>(S, it - 2);  // lag warps done reading the data slot
            if (it >= AUX) tc_wait_tfree<AUX>(S, it - AUX);
            if (threadIdx.x == 0) TC_ACC(0);
        };
        auto handoff = [&](int it) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> async proxy
            // alternating barrier ids keep consecutive iterations apart
            if (it & 1) asm volatile("bar.arrive 3, %0;" ::"n"(TcRoles<MODE>::HANDOFF) : "memory");
            else asm volatile("bar.arrive 2, %0;" ::"n"(TcRoles<MODE>::HANDOFF) : "memory");
        };
        bool fast = false;
        if constexpr (std::is_same<T, float>::value) fast = a.fast;
        if (fast) {
            if constexpr (std::is_same<T, float>::value) {
                TcRegs<MODE> cur;
                TcRegs<F2 ? 0 : MODE> nxt;  // 2-SM: one buffer, refilled right after its build
                if (npairs) tc_fetch<MODE>(a, base, cur);
                if constexpr (SX) {
                    if (npairs) tc_build_template<QM, F2 ? 2 : F4 ? 1 : 0>(a, S);
                }
                if constexpr (FP4) {
                    for (int p = 1; p < kTcPrefetch && p < npairs; ++p)
                        tc_prefetch_l2<MODE>(a, base + (int64_t)p * stride);
                }
                for (int it = 0; it < npairs; ++it) {
                    const int64_t pair = base + (int64_t)it * stride;
                    if constexpr (FP4) {
                        if (it + kTcPrefetch < npairs) tc_prefetch_l2<MODE>(a, pair + (int64_t)kTcPrefetch * stride);
                    }
                    if constexpr (!F2) {
                        if (it + 1 < npairs) tc_fetch<MODE>(a, pair + stride, nxt);
                    }
                    acquire(it);
                    TC_T0();
#ifdef QX_TC_TIMING
                    if (!(a.debug & 2))
#endif
                    {
                        if constexpr (F2) tc_build_tmpl2<QM>(a, S, it & 1, it % AUX, cur, it < 2);
                        else if constexpr (F4) tc_build_tmpl4<QM>(a, S, it & 1, it % AUX, cur, it < 2);
                        else if constexpr (SX) tc_build_tmpl<QM>(a, S, it & 1, it % AUX, cur, it < 2);
                        else tc_build_fast<QM>(a, S, it & 1, it % AUX, cur, it < 2);
                    }
                    if (threadIdx.x == 0) TC_ACC(1);
                    handoff(it);
                    if constexpr (F2) {
                        if (it + 1 < npairs) tc_fetch<MODE>(a, pair + stride, cur);
                    } else {
                        cur = nxt;
                    }
                }
            }
        } else {
            for (int it = 0; it < npairs; ++it) {
                const int64_t pair = base + (int64_t)it * stride;
                acquire(it);
                tc_build<T, QM>(a, S, it & 1, it % AUX, pair);
                handoff(it);
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ---- MMA issuer: the whole warp runs the loop, one elected lane issues
        const int nk = a.K / 32;
        uint32_t t4gc = 0;  // mode 4: A chunks consumed
        (void)t4gc;
        for (int it = 0; it < npairs; ++it) {
            const int s = it & 1, u = it % AUX;
            {
                TC_T0();
                if (it & 1) asm volatile("bar.sync 3, %0;" ::"n"(TcRoles<MODE>::HANDOFF) : "memory");
                else asm volatile("bar.sync 2, %0;" ::"n"(TcRoles<MODE>::HANDOFF) : "memory");
                if (lane == 0) TC_ACC(2);
            }
            if constexpr (F2) {
                if (rank != 0) {
                    // peer: its half of the pair is built; the leader issues
                    if (lane == 0) mbar_arrive_remote(&S.pready[s], 0);
                    continue;
                }
                mbar_wait<true>(&S.pready[s], (uint32_t)((it >> 1) & 1));
            }
            {
                TC_T0();
                if (it >= AUX) tc_wait_tfree<AUX, F2>(S, it - AUX);  // TMEM slot drained (2-SM: in both CTAs)
                if (lane == 0) TC_ACC(4);
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            TC_T0();
            constexpr int LBO = FP4 ? kF4Lbo : SX ? kTcBLbo32 : kTcBLbo, BINC = 2 * LBO / 16;
            const uint32_t ya = smem_u32(S.y[s]), ba = smem_u32(S.b + (SX ? 0 : s) * kTcBSlot);
            const uint64_t bd0 = smem_desc(ba, LBO, 128);
            const uint32_t tbase = __shfl_sync(0xffffffffu, S.tmem_base, 0);
            if constexpr (T4) {
                // A chunks from the stagers' TMEM ring, B from shared memory
                const uint32_t d = tbase + (uint32_t)(u * kF4Pitch), sf = tbase + SFC;
                const int nk4 = a.K / 64;
                for (int c0 = 0; c0 < nk4; c0 += kT4Chunk, ++t4gc) {
                    const int slot = t4gc & 1;
#ifdef QX_TC_TIMING
                    long long _m0 = clock64();
#endif
                    mbar_wait(&S.afull[slot], (t4gc >> 1) & 1);
#ifdef QX_TC_TIMING
                    if (lane == 0) atomicAdd(&S.tm[18], (unsigned long long)(clock64() - _m0));
#endif
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const int n = min(kT4Chunk, nk4 - c0);
                    for (int j = 0; j < n; ++j) {
                        const int k = c0 + j;
                        mma_f4t_warp(d, tbase + (uint32_t)(kT4ACol + slot * 128 + 8 * j),
                                     bd0 + (uint64_t)(k * BINC), a.idesc, k > 0 ? 1u : 0u, sf);
                    }
                    mma_commit_warp(&S.afree[slot]);  // the chunk's MMAs done: the stagers may refill it
                }
            } else if constexpr (FP4) {
                // F4: one M=128 x N=64 tile (8192 lags); F2: one M=256 x N=128
                // tile over the pair (32768 lags); K = 64 samples (32 B of A) per MMA
                constexpr int CG = F2 ? 2 : 1;
                const uint32_t d = tbase + (uint32_t)(u * PITCH), sf = tbase + SFC;
                const uint64_t ad0 = F2 ? (smem_desc(ya, 16, 512) | (4ull << 61))   // SWIZZLE_64B, 8 rows x 64 B
                                        : (smem_desc(ya, 16, 256) | (6ull << 61));  // SWIZZLE_32B, 8 rows x 32 B
                const uint32_t ahi = (uint32_t)(ad0 >> 32), bhi = (uint32_t)(bd0 >> 32);
                uint32_t alo = (uint32_t)ad0, blo = (uint32_t)bd0;
                const int nk4 = a.K / 64;
#ifdef QX_TC_TIMING
                if (!(a.debug & 1))
#endif
                {
                    mma_f4_warp<CG>(d, ad0, bd0, a.idesc, 0, sf);
                    int kk = 1;
                    for (; kk + 4 <= nk4; kk += 4) {
                        mma_f4_warp4<BINC, CG>(d, alo + 2, ahi, blo + BINC, bhi, a.idesc, sf);
                        alo += 8;
                        blo += 4 * BINC;
                    }
                    for (; kk < nk4; ++kk) {
                        alo += 2;
                        blo += BINC;
                        mma_f4_warp<CG>(d, ((uint64_t)ahi << 32) | alo, ((uint64_t)bhi << 32) | blo, a.idesc, 1, sf);
                    }
                }
            } else
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
            if constexpr (F2) mma_commit_pair(&S.mdone[u]);
            else mma_commit_warp(&S.mdone[u]);
            __syncwarp();
            if (lane == 0) TC_ACC(5);
        }
    } else if (warp >= kTcLagWarp0 && warp < kTcLagWarp0 + TcRoles<MODE>::NLAG) {
        // ---- lag warps: the extra lags of each pair from its code buffers
        for (int it = 0; it < npairs; ++it) {
            if (it & 1) asm volatile("bar.sync 3, %0;" ::"n"(TcRoles<MODE>::HANDOFF) : "memory");
            else asm volatile("bar.sync 2, %0;" ::"n"(TcRoles<MODE>::HANDOFF) : "memory");
            if (it >= AUX) tc_wait_tfree<AUX>(S, it - AUX);  // epilogue done with this aux slot's records
            if (a.extra) tc_extra_lags<SX ? 32 : 16, TcRoles<MODE>::NLAG>(a, S, it & 1, it % AUX, SX ? 0 : (it & 1));
            if (warp == kTcLagWarp0) tc_final_stats(a, S, it % AUX);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.xdone[it % AUX])) : "memory");
        }
    } else if (T4 && warp >= kT4StageWarp0 && warp < kT4StageWarp0 + 4) {
        // ---- mode 4 stagers: the pair's Hankel rows into the TMEM A ring
        if constexpr (T4) {
            const int q = warp & 3, row = q * 32 + lane;
            const uint32_t lanebase = S.tmem_base + ((uint32_t)(q * 32) << 16);
            const int nk4 = a.K / 64;
            uint32_t gc = 0;
            for (int it = 0; it < npairs; ++it) {
                if (it & 1) asm volatile("bar.sync 3, %0;" ::"n"(TcRoles<MODE>::HANDOFF) : "memory");
                else asm volatile("bar.sync 2, %0;" ::"n"(TcRoles<MODE>::HANDOFF) : "memory");
                const uint32_t* yw = reinterpret_cast<const uint32_t*>(S.y[it & 1]);
                int s0 = 0;  // next K-step to stage
                for (int c0 = 0; c0 < nk4; c0 += kT4Chunk, ++gc) {
                    const int slot = gc & 1;
#ifdef QX_TC_TIMING
                    long long _s0 = clock64();
#endif
                    if (gc >= 2) mbar_wait(&S.afree[slot], ((gc >> 1) - 1) & 1);
#ifdef QX_TC_TIMING
                    long long _s1 = clock64();
                    if (threadIdx.x == kT4StageWarp0 * 32) atomicAdd(&S.tm[16], (unsigned long long)(_s1 - _s0));
#endif
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const int n = min(kT4Chunk, nk4 - c0);
                    // groups of 4 K-steps, one 32-column tcgen05.st each; the row's
                    // 4 x 8 words are contiguous in the (SW32-swizzled) y slot: two
                    // 16-B loads per step (the swizzle swaps the halves of 32 B)
                    for (int j = 0; j < n; j += 4) {
                        uint32_t g[32];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int base = 8 * row + 8 * (s0 + k), b5 = (base >> 5) & 1;
                            const uint4 lo = *reinterpret_cast<const uint4*>(yw + base + 4 * b5);
                            const uint4 hi = *reinterpret_cast<const uint4*>(yw + base + 4 * (1 - b5));
                            g[8 * k + 0] = lo.x;
                            g[8 * k + 1] = lo.y;
                            g[8 * k + 2] = lo.z;
                            g[8 * k + 3] = lo.w;
                            g[8 * k + 4] = hi.x;
                            g[8 * k + 5] = hi.y;
                            g[8 * k + 6] = hi.z;
                            g[8 * k + 7] = hi.w;
                        }
                        asm volatile(
                            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
                                lanebase + (uint32_t)(kT4ACol + slot * 128 + 8 * j)),
                            "r"(g[0]), "r"(g[1]), "r"(g[2]), "r"(g[3]), "r"(g[4]), "r"(g[5]), "r"(g[6]), "r"(g[7]),
                            "r"(g[8]), "r"(g[9]), "r"(g[10]), "r"(g[11]), "r"(g[12]), "r"(g[13]), "r"(g[14]), "r"(g[15]),
                            "r"(g[16]), "r"(g[17]), "r"(g[18]), "r"(g[19]), "r"(g[20]), "r"(g[21]), "r"(g[22]), "r"(g[23]),
                            "r"(g[24]), "r"(g[25]), "r"(g[26]), "r"(g[27]), "r"(g[28]), "r"(g[29]), "r"(g[30]), "r"(g[31]));
                        s0 += 4;
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
#ifdef QX_TC_TIMING
                    if (threadIdx.x == kT4StageWarp0 * 32) atomicAdd(&S.tm[17], (unsigned long long)(clock64() - _s1));
#endif
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.afull[slot])) : "memory");
                    s0 = c0 + kT4Chunk;  // (the last, partial chunk ends the pair)
                }
            }
        }
    } else if (TcRoles<MODE>::MERGE_WARP && warp == kTcMergeWarp) {
        // ---- merge: records -> qx_result (2-SM: one record per CTA and pair)
        for (int it = 0; it < npairs; ++it) {
            const int64_t pair = base + (int64_t)it * stride;
            tc_wait_xdone<AUX>(S, it);  // statistics and extra-lag records written
            tc_wait_edone<AUX>(S, it);  // epilogue records written
            tc_merge<PITCH, TcRoles<MODE>::NLAG>(a, S, it % AUX, F2 ? 2 * pair + rank : pair, F2 && rank != 0);
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
        // ---- epilogue: TMEM -> per-warp (max, smallest lag, count) records
        for (int it = 0; it < npairs; ++it) {
            TC_T0();
            tc_wait_mdone<AUX>(S, it);
            if constexpr (!TcRoles<MODE>::MERGE_WARP) tc_wait_xdone<AUX>(S, it);  // lag warps' records in
            if (threadIdx.x == kEpiWarp0 * 32) TC_ACC(3);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            {
                TC_T0();
                if constexpr (F2) tc_epilogue_f2(a, S, it % AUX);
                else tc_epilogue<PITCH, F4>(a, S, it % AUX);
                if constexpr (!TcRoles<MODE>::MERGE_WARP) {
                    // int8 modes: the first epilogue warp merges once the four
                    // records are in (named barrier); every epilogue thread then
                    // frees the slot
                    asm volatile("bar.sync 4, 128;" ::: "memory");
                    if (warp == kEpiWarp0) {
                        const int64_t pair = base + (int64_t)it * stride;
                        tc_merge<PITCH, TcRoles<MODE>::NLAG>(a, S, it % AUX, pair, false, false);
                    }
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&S.tfree[it % AUX])) : "memory");
                }
                if (threadIdx.x == kEpiWarp0 * 32) TC_ACC(6);
            }
        }
    }
    // every MMA was waited on by the epilogue before TMEM is released
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // 2-SM: no CTA leaves (or frees TMEM) while its peer may still arrive on
    // its barriers or the leader's MMAs may still target its TMEM
    if constexpr (F2) cluster_sync_all();
#ifdef QX_TC_TIMING
    {
        unsigned long long k_g1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(k_g1));
        if ((blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && threadIdx.x == 0)
            printf("tc block %d: %lld pairs, %lld cycles, %.1f us -> %.0f MHz\n", blockIdx.x, (long long)npairs,
                   clock64() - k_t0, (k_g1 - k_g0) / 1e3, (double)(clock64() - k_t0) / ((k_g1 - k_g0) / 1e3));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && npairs)
        printf("tc timing block0 npairs=%lld debug=%d (cycles/pair): build-wait %llu build %llu | mma: wait-handoff %llu "
               "wait-tfree %llu issue %llu | epi: wait %llu run %llu\n",
               (long long)npairs, a.debug, S.tm[0] / npairs, S.tm[1] / npairs, S.tm[2] / npairs, S.tm[4] / npairs,
               S.tm[5] / npairs, S.tm[3] / npairs, S.tm[6] / npairs);
    if (blockIdx.x == 0 && threadIdx.x == 0 && npairs)
        printf("  t4 (cycles/pair): stager wait-free %llu stage %llu | mma wait-full %llu\n", S.tm[16] / npairs,
               S.tm[17] / npairs, S.tm[18] / npairs);
    if (blockIdx.x == 0 && threadIdx.x == 0 && npairs)
        printf("  build phases (cycles/pair): zero %llu quant %llu bar %llu copies %llu aux %llu | epi: tmem+scan %llu "
               "shfl %llu bars+merge %llu\n", S.tm[8] / npairs, S.tm[9] / npairs, S.tm[10] / npairs,
               S.tm[11] / npairs, S.tm[12] / npairs, S.tm[13] / npairs, S.tm[14] / npairs, S.tm[15] / npairs);
#endif
    if (warp == 0) {
        if constexpr (F2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(S.tmem_base), "n"(kTmemCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(S.tmem_base), "n"(kTmemCols));
    }
}

// fp4 shared-template mode: float32 rows, x a stride-0 row of <= 4096
// samples (template search), 16-B aligned rows, codes |c| <= 4 on both sides,
// every sum exact in f32 (nx * Kx * Ky < 2^24), one 8192-lag tile starting
// at a word boundary, y rows <= 12288 samples; QX_TC_F4=0 disables it
static bool tc_fp4_codes(const NttCall& c, int64_t nx)
{
    if (!c.knobs->tc_f4) return false;
    return c.op[0].dtype == DT_F32 && c.op[1].dtype == DT_F32 && c.op[0].ld == 0 && nx <= kTcFastN &&
           nx % 4 == 0 && (uintptr_t)c.op[0].data % 16 == 0 && (uintptr_t)c.op[1].data % 16 == 0 &&
           c.op[1].ld % 4 == 0 && c.op[0].q.mode == c.op[1].q.mode && c.op[0].q.k <= kF4MaxCode &&
           c.op[1].q.k <= kF4MaxCode && (double)nx * c.op[0].q.k * c.op[1].q.k < 16777216.0;
}

static bool tc_f4_mode(const NttCall& c, int64_t nx, int64_t ny)
{
    const int64_t W = c.am.t_hi - c.am.t_lo + 1, L0 = c.am.t_lo - (nx - 1);
    return tc_fp4_codes(c, nx) && ny <= kTcFastNY4 && W <= kF4Lags && L0 % 8 == 0 && L0 <= 0;
}

// (the 2-SM fp4 mode is retired: no call selects it)
static bool tc_f2_mode(const NttCall&, int64_t, int64_t) { return false; }

// eligibility: window of at most kTcMaxTiles*2048 lags (fp4 mode: 8192),
// nx + 15 <= kTcMaxK, |values| < 2^31 (nx * Kx * Ky), same input dtype and
// quantiser mode (float)
bool tc_window_eligible(const NttCall& c, int64_t nx, int64_t ny)
{
    const int64_t W = c.am.t_hi - c.am.t_lo + 1;
    if (W > (int64_t)kTcMaxTiles * kTcLags + kTcMaxExtra && !tc_f4_mode(c, nx, ny) && !tc_f2_mode(c, nx, ny))
        return false;
    if (nx + 15 > kTcMaxK) return false;
    if (c.op[0].dtype != c.op[1].dtype || c.op[0].dtype == DT_I64) return false;
    if (c.op[0].q.mode != c.op[1].q.mode) return false;
    if (c.op[0].q.k > 127 || c.op[1].q.k > 127) return false;
    if ((double)nx * c.op[0].q.k * c.op[1].q.k >= 2147483647.0) return false;
    return true;
}

template <typename T, int QM, int MODE = 0>
static cudaError_t launch_tc(const TcArgs& a, cudaStream_t s, int sms)
{
    const size_t smem = sizeof(TcSmem);
    if (cudaError_t e = set_max_smem((const void*)k_tc_window<T, QM, MODE>, smem); e != cudaSuccess) return e;
    if constexpr (MODE == 3) {
        // clusters of 2 CTAs (one pair-block per cluster at a time), as many
        // as can be resident at once: not every SM has a free partner in its
        // GPC, and a second wave of clusters would double the tail
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(tc_threads(MODE));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        static int clusters = 0;
        if (!clusters) {
            cfg.gridDim = dim3((unsigned)(sms & ~1));
            cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, k_tc_window<T, QM, MODE>, &cfg);
            if (e != cudaSuccess || clusters < 1) clusters = sms / 2;
        }
        const int64_t want = a.batch;
        cfg.gridDim = dim3((unsigned)(2 * (want < clusters ? want : clusters)));
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_tc_window<T, QM, MODE>, a);
        if (e != cudaSuccess) return e;
    } else {
        const int grid = (int)(a.batch < sms ? a.batch : sms);
        k_tc_window<T, QM, MODE><<<grid, tc_threads(MODE), smem, s>>>(a);
    }
    return cudaGetLastError();
}

namespace i8 {
cudaError_t tc_i8_window_run(const NttCall& c, int64_t nx, cudaStream_t s);
}

cudaError_t tc_window_run(const NttCall& c, int64_t nx, cudaStream_t s)
{
    // the int8 modes run the int8 kernel (qx_tc_i8.cu: its role layout is the
    // one an int8 pair's hand-off needs); this kernel keeps the fp4 modes
    if (!tc_f2_mode(c, nx, c.op[1].n) && !tc_f4_mode(c, nx, c.op[1].n)) return i8::tc_i8_window_run(c, nx, s);
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
    // shared x: a stride-0 x row (every pair correlates the same template;
    // also a single pair passed that way, e.g. a template search's last block)
    const bool sx = c.op[0].dtype == DT_F32 && c.op[0].ld == 0 && nx <= kTcFastN && nx % 4 == 0 &&
                    aligned;
    const bool f2 = tc_f2_mode(c, nx, ny);
    const bool f4 = !f2 && tc_f4_mode(c, nx, ny);
    a.shared_x = f2 || f4 || (sx && ny <= kTcFastNY && W <= 4096 + kTcMaxExtra);
    a.fast = a.shared_x || (c.op[0].dtype == DT_F32 && nx <= kTcFastN && ny <= kTcFastN && nx % 4 == 0 &&
                            ny % 4 == 0 && aligned && (c.batch == 1 || c.op[0].ld % 4 == 0));
    a.pitch = f4 ? kF4Pitch : a.shared_x ? 32 : 16;
    // shape: pitch 16: one M=64 tile (1024 lags) when it covers the window up
    // to the extra lags, else M=128 tiles (2048 lags each); pitch 32/64: M=128
    a.M = (a.pitch == 16 && W <= 1024 + kTcMaxExtra) ? 64 : 128;
    const int tl = a.pitch * a.M;
    a.ntiles = (int)((W - kTcMaxExtra + tl - 1) / tl);
    if (a.ntiles < 1) a.ntiles = 1;
    a.extra = (int)(W > (int64_t)a.ntiles * tl ? W - (int64_t)a.ntiles * tl : 0);
    a.idesc = tc_idesc(a.M, a.pitch);
    // B copy r holds x at k = m + r: K covers nx + pitch - 1 (pitch 32 needs
    // more than the pitch-16 default for templates with nx % 32 outside 1..17)
    if (a.pitch == 32) a.K = (int)((nx + 31 + 31) / 32 * 32);
    if (f4) {
        a.K = (int)((nx + kF4Pitch - 1 + 63) / 64 * 64);
        a.ntiles = 1;
        a.extra = 0;
        a.idesc = tc_idesc_f4(128, kF4Pitch);
    }
    a.ylen = a.ntiles * tl + kTcMaxExtra + a.K;
    if (f2) {
        a.pitch = kF2Pitch;
        a.M = 256;
        a.K = (int)((nx + kF2Pitch - 1 + 63) / 64 * 64);
        a.ntiles = 1;
        a.extra = 0;
        a.idesc = tc_idesc_f4(256, kF2Pitch);
        a.ylen = kF2CtaLags + a.K;  // each CTA's window
    }
#ifdef QX_TC_TIMING
    if (const char* ev = getenv("QX_TC_DEBUG")) a.debug = atoi(ev);
#endif
    const int sms = device_sms();
    // fp4 modes only (the int8 ones returned above)
    if (c.prof) c.prof->pre(KK_DIRECT_F4, s);
    cudaError_t e;
    const int qm = c.op[0].q.mode;
    // mode 2 only: the 2-SM (3) and A-in-TMEM (4) variants measured slower
    // at config 5 (r02: 0.635 and 0.72 ms vs 0.477 ms) and are not built
    (void)f2;
    if (qm == QM_K1) e = launch_tc<float, QM_K1, 2>(a, s, sms);
    else if (qm == QM_UNIFORM) e = launch_tc<float, QM_UNIFORM, 2>(a, s, sms);
    else e = launch_tc<float, QM_BSEARCH, 2>(a, s, sms);
    if (c.prof) c.prof->post(KK_DIRECT_F4, s);
    return e;
}

// ---- template search: device merge of per-block summaries
// Record i (qx_result layout) covers lags [i*block, ...) of the stream; the
// merged summary is {max value, smallest global lag at it, summed ties, any
// NaN, x all-zero in any block, y all-zero in every block, any failing
// block (status other than 0 / degenerate quantisation), the largest such
// status}: the reference's argmax_set summary of the unblocked correlogram
// (estimator.py:50-57) plus the inputs of its exceptions.
struct BlkSum {
    long long v, l, t;
    int nan, degx, degy_all, bad, badst;
};

__device__ __forceinline__ void blk_add(BlkSum& a, const BlkSum& b)
{
    if (b.t) {
        if (!a.t || b.v > a.v) { a.v = b.v; a.l = b.l; a.t = b.t; }
        else if (b.v == a.v) { a.l = min(a.l, b.l); a.t += b.t; }
    }
    a.nan |= b.nan;
    a.degx |= b.degx;
    a.degy_all &= b.degy_all;
    a.bad |= b.bad;
    a.badst = max(a.badst, b.badst);
}

__device__ BlkSum blk_shfl(const BlkSum& a, int o)
{
    BlkSum b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.l = __shfl_xor_sync(0xffffffffu, a.l, o);
    b.t = __shfl_xor_sync(0xffffffffu, a.t, o);
    b.nan = __shfl_xor_sync(0xffffffffu, a.nan, o);
    b.degx = __shfl_xor_sync(0xffffffffu, a.degx, o);
    b.degy_all = __shfl_xor_sync(0xffffffffu, a.degy_all, o);
    b.bad = __shfl_xor_sync(0xffffffffu, a.bad, o);
    b.badst = __shfl_xor_sync(0xffffffffu, a.badst, o);
    return b;
}

constexpr int kMergeThreads = 256;

// block-wide merge; the result is valid in thread 0
__device__ BlkSum blk_reduce(BlkSum a)
{
    __shared__ BlkSum sh[kMergeThreads / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) blk_add(a, blk_shfl(a, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
        BlkSum b = threadIdx.x < kMergeThreads / 32 ? sh[threadIdx.x] : BlkSum{0, LLONG_MAX, 0, 0, 0, 1, 0, 0};
#pragma unroll
        for (int o = 16; o; o >>= 1) blk_add(b, blk_shfl(b, o));
        a = b;
    }
    return a;
}

__global__ void __launch_bounds__(kMergeThreads) k_merge_blocks(const MergeSegs segs, long long lag_shift,
                                                                BlkSum* partials, int* counter, long long* out)
{
    BlkSum a{0, LLONG_MAX, 0, 0, 0, 1, 0, 0};
    const int64_t n = segs.seg[0].n + segs.seg[1].n + segs.seg[2].n;
    for (int64_t k = blockIdx.x * (int64_t)kMergeThreads + threadIdx.x; k < n; k += (int64_t)gridDim.x * kMergeThreads) {
        int sg = 0;
        int64_t i = k;
        while (i >= segs.seg[sg].n) i -= segs.seg[sg++].n;
        const MergeSeg& S = segs.seg[sg];
        const long long* r = S.recs + i * 8;
        const long long w7 = r[7];
        const int status = (int)(w7 >> 32), flags = (int)(w7 & 0xffffffff);
        BlkSum b;
        b.v = r[0];
        b.l = r[1] + S.base + (i / S.rpb) * S.block;
        b.t = status == 0 ? r[2] : 0;
        b.nan = (flags & 4) != 0;
        b.degx = (flags & 1) != 0;
        b.degy_all = r[6] == 0;
        b.bad = status != 0 && status != 2;
        b.badst = b.bad ? status : 0;
        blk_add(a, b);
    }
    a = blk_reduce(a);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = a;
        __threadfence();
        last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    BlkSum m{0, LLONG_MAX, 0, 0, 0, 1, 0, 0};
    for (int i = threadIdx.x; i < (int)gridDim.x; i += kMergeThreads) {
        const BlkSum* p = partials + i;  // other CTAs' records: L2 loads
        BlkSum b;
        b.v = __ldcg(&p->v);
        b.l = __ldcg(&p->l);
        b.t = __ldcg(&p->t);
        b.nan = __ldcg(&p->nan);
        b.degx = __ldcg(&p->degx);
        b.degy_all = __ldcg(&p->degy_all);
        b.bad = __ldcg(&p->bad);
        b.badst = __ldcg(&p->badst);
        blk_add(m, b);
    }
    m = blk_reduce(m);
    if (threadIdx.x == 0) {
        out[0] = m.t ? m.v : 0;
        out[1] = m.t ? m.l + lag_shift : 0;
        out[2] = m.t;
        out[3] = m.nan;
        out[4] = m.degx;
        out[5] = m.degy_all;
        out[6] = m.bad;
        out[7] = m.badst;
        *counter = 0;  // ready for the next launch
    }
}

cudaError_t merge_blocks_launch(const MergeSegs& segs, long long lag_shift, void* partials, int* counter,
                                long long* out, int sms, cudaStream_t s)
{
    const int64_t n = segs.seg[0].n + segs.seg[1].n + segs.seg[2].n;
    int64_t g = (n + kMergeThreads - 1) / kMergeThreads;
    const int grid = (int)(g < 1 ? 1 : (g > sms ? sms : g));
    k_merge_blocks<<<grid, kMergeThreads, 0, s>>>(segs, lag_shift, (BlkSum*)partials, counter, out);
    return cudaGetLastError();
}

}  // namespace qx
