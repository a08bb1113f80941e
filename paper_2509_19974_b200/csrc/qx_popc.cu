// qx_popc.cu -- word-parallel correlation of 1-level codes (k = 1: sign(),
// uniform(1, .), custom with k = 1; codes in {-1, 0, 1}) on the CUDA cores:
// the latency path for single short pairs (BASELINE config 1).
//
// Codes are two bit planes per signal, s (code < 0) and z (code != 0); for
// 32 aligned samples
//   sum_m u[m] v[m] = popc(zu & zv) - 2 popc(zu & zv & (su ^ sv)),
// and when neither signal has a zero code in range the first term is the
// overlap count of the lag, so one POPC per 32 products remains.  This is
// the reference's brute-force correlation (intxcorr.py:96-100) with the
// argmax summary of argmax_set (estimator.py:50-57) fused.
//
// k_popc_planes quantises both signals once into global bit planes (one
// warp ballot per 32 samples) with the statistics; k_popc, grid (G, batch),
// gives CTA g of a pair a contiguous run of 32-lag blocks: it stages x's
// planes and the y window its lags touch (realigned by funnel shifts) in
// shared memory, then every group of 4 warps
// correlates one 32-lag block at a time: lane k holds x words k, k+128, ...
// in registers and keeps 32 lag accumulators (the y word pair is loaded once
// per x word, the 32 shifts are immediate funnel shifts), REDUX sums each
// lag over the warp, and the group's first warp adds the four warps' sums.
// Per-lane running (max, smallest lag, count) records are merged by the
// NTT path's argmax_finish (block reduce -> per-CTA partial -> last CTA
// writes the qx_result with the statistics).
#include <climits>
#include <cstdio>

#include <cooperative_groups.h>

#include "qx_argmax.cuh"
#include "qx_internal.h"

namespace qx {

constexpr int kPopcThreads = 512;
constexpr int kPopcWarps = kPopcThreads / 32;
constexpr int kPopcGroup = 4;                        // warps per 32-lag block
constexpr int kPopcGroups = kPopcWarps / kPopcGroup;  // blocks in flight per CTA

// one operand as the popc kernels need it (rows + the two thresholds of a
// 1-level quantiser): a few dozen parameter bytes instead of OperandDesc's
// 2-KB threshold table, so the launch carries a small parameter block
struct PopcOp {
    const void* data;
    int64_t ld, n;
    double t0, t1;
};

struct PopcArgs {
    PopcOp op[2];
    unsigned long long* stats;  // [batch][2][4]
    ArgmaxOut am;
    int64_t dlo;   // first lag (relative: x[m] y[m + d]) of the window
    int64_t dhi;   // last lag
    int nblk;      // 32-lag blocks of the window
    int bpc;       // blocks per CTA
    int nxw;       // x words
    int nyw;       // y words (whole signal)
    uint32_t* planes;  // [batch][xs | xz | ys | yz]: 2 * (nxw + nyw) words per pair
    unsigned* spart;   // fused kernel: [batch][G][4] per-CTA nonzero counts (x, y) and flags
};

__device__ __forceinline__ uint32_t* plane_x(const PopcArgs& a, int64_t pair)
{
    return a.planes + pair * 2 * (int64_t)(a.nxw + a.nyw);
}

// global planes of both signals of a pair: warp w of the grid row quantises
// word w (x words first, then y), statistics per CTA into the pair's record
template <typename T>
__global__ void __launch_bounds__(kPopcThreads) k_popc_planes(const __grid_constant__ PopcArgs a)
{
    __shared__ unsigned s_nz[2], s_fl;
    const int64_t pair = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int w = blockIdx.x * kPopcWarps + (threadIdx.x >> 5);
    if (threadIdx.x < 2) s_nz[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_fl = 0;
    __syncthreads();
    const bool isx = w < a.nxw;
    if (w < a.nxw + a.nyw) {
        const PopcOp& o = a.op[isx ? 0 : 1];
        const T* row = reinterpret_cast<const T*>(o.data) + pair * o.ld;
        const int64_t i = 32ll * (isx ? w : w - a.nxw) + lane;
        const T v = i < o.n ? row[i] : (T)0;
        const int c = level_k1(v, (T)o.t0, (T)o.t1);
        const uint32_t sb = __ballot_sync(0xffffffffu, c < 0), zb = __ballot_sync(0xffffffffu, c != 0);
        const bool nan = __any_sync(0xffffffffu, v != v);
        if (lane == 0) {
            uint32_t* px = plane_x(a, pair);
            if (isx) {
                px[w] = sb;
                px[a.nxw + w] = zb;
            } else {
                uint32_t* py = px + 2 * a.nxw;
                py[w - a.nxw] = sb;
                py[a.nyw + (w - a.nxw)] = zb;
            }
            atomicAdd(&s_nz[isx ? 0 : 1], __popc(zb));
            if (nan) atomicOr(&s_fl, SF_NONFINITE);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* st = a.stats + pair * 8;
        // sum of squares = nonzero count for 1-level codes
        if (s_nz[0]) {
            atomicAdd(st + 0, (unsigned long long)s_nz[0]);
            atomicAdd(st + 1, (unsigned long long)s_nz[0]);
        }
        if (s_nz[1]) {
            atomicAdd(st + 4, (unsigned long long)s_nz[1]);
            atomicAdd(st + 5, (unsigned long long)s_nz[1]);
        }
        if (s_fl) atomicOr(st + 6, (unsigned long long)s_fl);
    }
}

// bits of word w (samples lo .. lo + 31) that lie inside [0, n)
__device__ __forceinline__ uint32_t popc_valid(int64_t lo, int64_t n)
{
    const int64_t a = lo < 0 ? -lo : 0, b = n - lo < 32 ? n - lo : 32;
    if (b <= a) return 0u;
    const uint32_t hi = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
    return hi & ~((1u << a) - 1u);
}

template <bool ALLNZ>
__device__ void popc_blocks(const PopcArgs& a, const uint32_t* xs, const uint32_t* xz, const uint32_t* ys,
                            const uint32_t* yz, int b0, int b1, int64_t yb, Best& best, int* part)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = warp / kPopcGroup, wg = warp % kPopcGroup;
    const int nxw = a.nxw;
    const int64_t nx = a.op[0].n, ny = a.op[1].n;
    for (int b = b0 + grp; b < b1; b += kPopcGroups) {
        int acc[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) acc[l] = 0;
        const int q0 = b - b0;  // y word of x word 0, lag l of the block at bit l
        for (int i = wg * 32 + lane; i < nxw; i += 32 * kPopcGroup) {
            const uint32_t sx = xs[i], zx = xz[i];
            const uint32_t y0 = ys[q0 + i], y1 = ys[q0 + i + 1], z0 = yz[q0 + i], z1 = yz[q0 + i + 1];
#pragma unroll
            for (int l = 0; l < 32; ++l) {
                const uint32_t yy = __funnelshift_r(y0, y1, l), zz = __funnelshift_r(z0, z1, l);
                const uint32_t az = zz & zx;
                const uint32_t d = (sx ^ yy) & az;
                if constexpr (ALLNZ) acc[l] += __popc(d);
                else acc[l] += __popc(az) - 2 * __popc(d);
            }
        }
        // lane l <- the warp's sum for lag l; the group's first warp adds the four
        int mine = 0;
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            const int v = __reduce_add_sync(0xffffffffu, acc[l]);
            if (lane == l) mine = v;
        }
        part[(grp * kPopcGroup + wg) * 32 + lane] = mine;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(32 * kPopcGroup) : "memory");
        if (wg == 0) {
            int sum = 0;
#pragma unroll
            for (int w = 0; w < kPopcGroup; ++w) sum += part[(grp * kPopcGroup + w) * 32 + lane];
            const int64_t d = a.dlo + 32ll * b + lane;
            if (d <= a.dhi) {
                long long v = sum;
                if constexpr (ALLNZ) {
                    // overlap of the lag: m in [0, nx) with m + d in [0, ny)
                    const int64_t lo = d < 0 ? -d : 0, hi = nx < ny - d ? nx : ny - d;
                    v = (hi > lo ? hi - lo : 0) - 2ll * sum;
                }
                best_add(best, v, d + nx - 1);
            }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(32 * kPopcGroup) : "memory");  // part reusable
    }
}

__device__ __forceinline__ void popc_correlate(const PopcArgs& a)
{
    extern __shared__ uint32_t pw[];
    __shared__ unsigned s_zero;
    __shared__ int part[kPopcWarps * 32];
    const int64_t pair = blockIdx.y;
    const int g = blockIdx.x, G = gridDim.x;
    const int64_t nx = a.op[0].n, ny = a.op[1].n;
    const int b0 = min(a.nblk, g * a.bpc), b1 = min(a.nblk, b0 + a.bpc);
    // y window: lags d of blocks [b0, b1) pair x[m] with y[m + d]
    const int64_t yb = a.dlo + 32ll * b0;
    const int nxw = a.nxw, nyw = (b1 - b0) + nxw + 1;
    uint32_t* xs = pw;
    uint32_t* xz = xs + nxw;
    uint32_t* ys = xz + nxw;
    uint32_t* yz = ys + nyw;
    if (threadIdx.x == 0) s_zero = 0;
    __syncthreads();
#ifdef QX_POPC_TIMING
    const long long tp0 = clock64();
#endif
    // stage the planes: x as is, y realigned to sample yb (zero outside y)
    const uint32_t* gx = plane_x(a, pair);
    const uint32_t* gy = gx + 2 * a.nxw;
    unsigned zero = 0;
    for (int w = threadIdx.x; w < nxw; w += kPopcThreads) {
        const uint32_t sv = gx[w], zv = gx[nxw + w];
        xs[w] = sv;
        xz[w] = zv;
        zero |= zv != popc_valid(32ll * w, nx);  // a zero code in range: the 2-POPC form
    }
    const int64_t q = yb >= 0 ? yb / 32 : -((31 - yb) / 32);  // floor(yb / 32)
    const int sh = (int)(yb - 32 * q);
    for (int w = threadIdx.x; w < nyw; w += kPopcThreads) {
        const int64_t w0 = q + w;
        const uint32_t s0 = (w0 >= 0 && w0 < a.nyw) ? gy[w0] : 0u, s1 = (w0 + 1 >= 0 && w0 + 1 < a.nyw) ? gy[w0 + 1] : 0u;
        const uint32_t z0 = (w0 >= 0 && w0 < a.nyw) ? gy[a.nyw + w0] : 0u;
        const uint32_t z1 = (w0 + 1 >= 0 && w0 + 1 < a.nyw) ? gy[a.nyw + w0 + 1] : 0u;
        const uint32_t sv = __funnelshift_r(s0, s1, sh), zv = __funnelshift_r(z0, z1, sh);
        ys[w] = sv;
        yz[w] = zv;
        zero |= zv != popc_valid(yb + 32ll * w, ny);
    }
    zero = __reduce_or_sync(0xffffffffu, zero);
    if ((threadIdx.x & 31) == 0 && zero) atomicOr(&s_zero, 1u);
    __syncthreads();
#ifdef QX_POPC_TIMING
    const long long tp1 = clock64();
#endif
    Best best = best_init();
    if (s_zero) popc_blocks<false>(a, xs, xz, ys, yz, b0, b1, yb, best, part);
    else popc_blocks<true>(a, xs, xz, ys, yz, b0, b1, yb, best, part);
#ifdef QX_POPC_TIMING
    __syncthreads();
    const long long tp2 = clock64();
#endif
    argmax_finish<kPopcWarps>(best, a.am, a.stats, pair, G, g);
#ifdef QX_POPC_TIMING
    if (threadIdx.x == 0 && (g == 0 || g == G - 1))
        printf("popc cta %d/%d: stage %lld, blocks %lld, finish %lld cycles (bpc %d, nyw %d, allnz %d)\n", g, G,
               tp1 - tp0, tp2 - tp1, clock64() - tp2, a.bpc, nyw, !s_zero);
#endif
}
__global__ void __launch_bounds__(kPopcThreads) k_popc(const __grid_constant__ PopcArgs a) { popc_correlate(a); }

// one cooperative launch: the planes of every pair (CTA g of pair p takes
// words g*16 + warp + k*16G), per-CTA counts into spart, a grid-wide sync,
// CTA 0 of each pair turns the counts into the pair's statistics record (no
// memset, no atomics), then the correlation as in k_popc
template <typename T>
__global__ void __launch_bounds__(kPopcThreads) k_popc_fused(const __grid_constant__ PopcArgs a)
{
    __shared__ unsigned s_cnt[3];
    const int64_t pair = blockIdx.y;
    const int g = blockIdx.x, G = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#ifdef QX_POPC_TIMING
    unsigned long long f0, f1, f2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(f0));
#endif
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    uint32_t* px = plane_x(a, pair);
    unsigned nzx = 0, nzy = 0;
    bool nan = false;
    for (int w = g * kPopcWarps + warp; w < a.nxw + a.nyw; w += G * kPopcWarps) {
        const bool isx = w < a.nxw;
        const PopcOp& o = a.op[isx ? 0 : 1];
        const T* row = reinterpret_cast<const T*>(o.data) + pair * o.ld;
        const int64_t i = 32ll * (isx ? w : w - a.nxw) + lane;
        const T v = i < o.n ? row[i] : (T)0;
        const int c = level_k1(v, (T)o.t0, (T)o.t1);
        const uint32_t sb = __ballot_sync(0xffffffffu, c < 0), zb = __ballot_sync(0xffffffffu, c != 0);
        nan |= v != v;
        if (lane == 0) {
            if (isx) {
                px[w] = sb;
                px[a.nxw + w] = zb;
                nzx += __popc(zb);
            } else {
                uint32_t* py = px + 2 * a.nxw;
                py[w - a.nxw] = sb;
                py[a.nyw + (w - a.nxw)] = zb;
                nzy += __popc(zb);
            }
        }
    }
    nan = __any_sync(0xffffffffu, nan);
    if (lane == 0) {
        if (nzx) atomicAdd(&s_cnt[0], nzx);
        if (nzy) atomicAdd(&s_cnt[1], nzy);
        if (nan) atomicOr(&s_cnt[2], SF_NONFINITE);
    }
    __syncthreads();
    if (threadIdx.x < 3) a.spart[(pair * G + g) * 4 + threadIdx.x] = s_cnt[threadIdx.x];
#ifdef QX_POPC_TIMING
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(f1));
#endif
    cooperative_groups::this_grid().sync();
#ifdef QX_POPC_TIMING
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(f2));
    if (threadIdx.x == 0 && (g == 0 || g == G - 1))
        printf("fused cta %d: planes %.2f us, grid sync %.2f us\n", g, (f1 - f0) / 1e3, (f2 - f1) / 1e3);
#endif
    if (g == 0 && warp == 0) {
        unsigned cx = 0, cy = 0, fl = 0;
        for (int i = lane; i < G; i += 32) {
            const unsigned* sp = a.spart + (pair * G + i) * 4;
            cx += sp[0];
            cy += sp[1];
            fl |= sp[2];
        }
        cx = __reduce_add_sync(0xffffffffu, cx);
        cy = __reduce_add_sync(0xffffffffu, cy);
        fl = __reduce_or_sync(0xffffffffu, fl);
        unsigned long long* st = a.stats + pair * 8;
        // sum of squares = nonzero count for 1-level codes
        if (lane < 8) st[lane] = lane == 0 || lane == 1 ? cx : lane == 4 || lane == 5 ? cy : lane == 6 ? fl : 0ull;
    }
    popc_correlate(a);
}


// launch plan: ~2 CTAs per SM over the whole batch, at least kPopcGroups
// 32-lag blocks per CTA when there are enough; returns the shared memory
static size_t popc_plan(const NttCall& c, int64_t nx, PopcArgs& a, int64_t& G, bool fused = false)
{
    a.dlo = c.am.t_lo - (nx - 1);
    a.dhi = c.am.t_hi - (nx - 1);
    const int64_t nlag = a.dhi - a.dlo + 1;
    const int64_t nblk = (nlag + 31) / 32;
    a.nblk = (int)nblk;
    a.nxw = (int)((nx + 31) / 32);
    a.nyw = (int)((c.op[1].n + 31) / 32);
    const int sms = device_sms();
    // fused (cooperative) launch: every CTA resident at once, one per SM
    G = fused ? (int64_t)sms / c.batch : ((int64_t)sms + c.batch - 1) / c.batch;
    const int64_t gmax = (nblk + kPopcGroups - 1) / kPopcGroups;
    if (G > gmax) G = gmax;
    if (G > kMaxPartialsLarge) G = kMaxPartialsLarge;
    if (G < 1) G = 1;
    const int64_t bpc = (nblk + G - 1) / G;
    a.bpc = (int)(bpc < INT_MAX ? bpc : INT_MAX);
    G = (nblk + bpc - 1) / bpc;
    return (size_t)(2 * a.nxw + 2 * (bpc + a.nxw + 1)) * 4;
}

// eligibility: argmax mode, 1-level quantisers on float rows, x <= 2^16
// samples, planes within 200 KB of shared memory; on AUTO also little enough
// work that one GPU-wide launch beats the NTT's three (batch * nx * window
// <= 2^31 code products)
bool popc_eligible(const NttCall& c, int64_t nx, int64_t ny, bool auto_path)
{
    (void)ny;
    if (auto_path && !c.knobs->popc) return false;
    if (c.op[0].q.mode != QM_K1 || c.op[1].q.mode != QM_K1) return false;
    if (c.op[0].dtype == DT_I64 || c.op[0].dtype != c.op[1].dtype) return false;
    if (nx > 65536) return false;
    const double W = (double)(c.am.t_hi - c.am.t_lo + 1);
    if (auto_path && (double)c.batch * (double)nx * W > 2147483648.0) return false;
    PopcArgs a;
    int64_t G;
    return popc_plan(c, nx, a, G) <= 200 * 1024;
}

cudaError_t popc_run(const NttCall& c, int64_t nx, cudaStream_t s)
{
    PopcArgs a;
    for (int i = 0; i < 2; ++i)
        a.op[i] = PopcOp{c.op[i].data, c.op[i].ld, c.op[i].n, c.op[i].q.thr[0], c.op[i].q.thr[1]};
    a.stats = c.stats;
    a.am = c.am;
    a.planes = c.popc_planes;
    a.spart = c.popc_spart;
    const int sms = device_sms();
    const bool fused = c.batch <= sms && c.knobs->popc_fused;
    int64_t G;
    const size_t smem = popc_plan(c, nx, a, G, fused);
    if (G > c.am.pstride) return cudaErrorInvalidValue;
    const int ti = c.op[0].dtype == DT_F32 ? 0 : 1;
    auto raise = [&](const void* fn, int) -> cudaError_t {
        return smem > 48 * 1024 ? set_max_smem(fn, smem) : cudaSuccess;
    };
    cudaError_t e;
    if (fused) {
        const void* fn = ti == 0 ? (const void*)k_popc_fused<float> : (const void*)k_popc_fused<double>;
        if ((e = raise(fn, ti)) != cudaSuccess) return e;
        if (c.prof) c.prof->pre(KK_POPC, s);
        void* args[] = {(void*)&a};
        e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)G, (unsigned)c.batch), dim3(kPopcThreads), args, smem, s);
        if (c.prof) c.prof->post(KK_POPC, s);
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    // two launches: planes (statistics by atomics into zeroed records), correlation
    if ((e = raise((const void*)k_popc, 2)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(c.stats, 0, (size_t)c.batch * 64, s)) != cudaSuccess) return e;
    if (c.prof) c.prof->pre(KK_POPC, s);
    const dim3 pgrid((unsigned)((a.nxw + a.nyw + kPopcWarps - 1) / kPopcWarps), (unsigned)c.batch);
    if (c.op[0].dtype == DT_F32) k_popc_planes<float><<<pgrid, kPopcThreads, 0, s>>>(a);
    else k_popc_planes<double><<<pgrid, kPopcThreads, 0, s>>>(a);
    if (c.prof) c.prof->post(KK_POPC, s);
    if (c.prof) c.prof->pre(KK_POPC, s);
    k_popc<<<dim3((unsigned)G, (unsigned)c.batch), kPopcThreads, smem, s>>>(a);
    if (c.prof) c.prof->post(KK_POPC, s);
    return cudaGetLastError();
}

}  // namespace qx
