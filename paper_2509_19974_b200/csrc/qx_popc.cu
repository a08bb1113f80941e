// qx_popc.cu -- word-parallel correlation of 1-level codes (k = 1: sign(),
// uniform(1, .), custom with k = 1; codes in {-1, 0, 1}) on the CUDA cores:
// the latency path for single short pairs (BASELINE config 1).
//
// Codes are two bit planes per signal, s (code < 0) and z (code != 0); for
// 32 aligned samples
//   sum_m u[m] v[m] = popc(zu & zv) - 2 popc(zu & zv & (su ^ sv)),
// and when neither signal has a zero code the first term is the overlap
// count of the lag, so one POPC per 32 products remains
// (value(d) = overlap(d) - 2 * mismatches(d)).  This is the reference's
// brute-force correlation (intxcorr.py:96-100) with the argmax summary of
// argmax_set (estimator.py:50-57) fused.
//
// One cooperative launch (every CTA of a pair resident, one per SM), no
// second kernel and no host round trip:
//   1. planes: the pair's G CTAs split the plane words (x words, then y
//      words; one ballot per 32 samples, a warp's loads in flight together)
//      and write them to global memory with per-CTA nonzero counts and NaN /
//      zero-code flags; meanwhile each CTA reads its block range from the
//      host-computed schedule and builds its unit prefix;
//   2. a per-pair grid barrier (acq_rel counter);
//   3. each CTA stages x's planes and the y window of its 32-lag blocks
//      (realigned by funnel shifts so lag block b, x word i reads y' words
//      i+b, i+b+1) in shared memory.  A block covers only the x words its
//      lags overlap (overlap-exact: half the rectangle of a full window);
//      the schedule gives every CTA a contiguous block range of near-equal
//      units (one per x word plus a fixed block overhead, partitioned on
//      the host, cached per shape).  Lane = lag: a warp walks a run of x
//      words of one block with broadcast shared loads, each lane
//      funnel-shifting the y words by its own lag, so the 32 lag sums need
//      no cross-lane reduction; runs of a block from several warps meet in
//      shared accumulators;
//   4. the CTA keeps (max, smallest lag, count) by REDUX and the pair's last
//      CTA (acq_rel ticket) merges the records with the statistics and
//      resets the pair's counters.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <vector>

#include "qx_argmax.cuh"
#include "qx_internal.h"

namespace qx {

constexpr int kPcThreads = 1024;  // one CTA per SM
constexpr int kPcWarps = kPcThreads / 32;
constexpr int kPcWordsPerWarp = 4;   // plane words per warp per round (loads in flight)
constexpr int kPcAccBlocks = 128;    // 32-lag block accumulators per pass of a CTA
constexpr int kPcBlockUnits = 28;    // per-block overhead in x-word units (setup, edge words, flush; measured)
constexpr int kPcMaxSmem = 200 * 1024;
constexpr unsigned kPcZeroCode = 0x100u;  // spart flag: a code 0 inside a signal

// one operand as the popc kernel needs it: rows + the two thresholds of a
// 1-level quantiser (a few dozen parameter bytes, not a 2-KB table)
struct PopcOp {
    const void* data;
    int64_t ld;
    double t0, t1;
};

struct PopcArgs {
    PopcOp op[2];
    ArgmaxOut am;               // am.counters: [2 * batch] (ticket, barrier) per pair
    unsigned long long* stats;  // [batch][8] statistics records (written by the pair's last CTA)
    uint32_t* planes;           // [batch][2 (sxw + syw)]: xs | xz | ys | yz, sample i at bit i % 32
    unsigned* spart;            // [batch][G][4] per-CTA nonzero counts (x, y) and flags
    const int* sched;           // [G + 1] first block of each CTA (host-computed, per shape)
    int batch;
    int dlo, dhi;               // lag window: x[m] * y[m + d], d in [dlo, dhi]
    int nx, ny;                 // samples (nx <= 2^16, ny <= 2^24: 32-bit index math)
    int nblk;                   // 32-lag blocks of the window
    int sxw, syw;               // words of the signals
};

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// x words [w0, w1) touched by the lags of block b: sample m pairs y[m + d]
// inside both signals for some d in [d0, d1]
__host__ __device__ __forceinline__ void block_words(int dlo, int dhi, int nx, int ny, int b, int& w0, int& w1)
{
    const int d0 = dlo + 32 * b;
    const int d1 = d0 + 31 < dhi ? d0 + 31 : dhi;
    const int mlo = -d1 > 0 ? -d1 : 0;
    const int mhi = nx < ny - d0 ? nx : ny - d0;
    w0 = mlo >> 5;
    w1 = mhi > mlo ? (mhi + 31) >> 5 : w0;
}

__host__ __device__ __forceinline__ int block_units(int dlo, int dhi, int nx, int ny, int b)
{
    int w0, w1;
    block_words(dlo, dhi, nx, ny, b, w0, w1);
    return w1 - w0 + kPcBlockUnits;
}

// (max value, smallest index, count) of a warp's lanes; v = INT_MIN, c = 0
// for lanes without a lag
__device__ __forceinline__ void warp_best(int& v, int& t, int& c)
{
    const int m = __reduce_max_sync(0xffffffffu, v);
    t = (int)__reduce_min_sync(0xffffffffu, v == m ? (unsigned)t : 0xffffffffu);
    c = (int)__reduce_add_sync(0xffffffffu, v == m ? (unsigned)c : 0u);
    v = m;
}

template <typename T, bool TIMING>
__global__ void __launch_bounds__(kPcThreads, 1) k_popc(const __grid_constant__ PopcArgs a)
{
    extern __shared__ uint32_t sm[];
    __shared__ unsigned s_cnt[3];
    __shared__ int s_best[kPcWarps][3];
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t pair = blockIdx.y;
    const int g = blockIdx.x, G = gridDim.x;
    const int nxw = a.sxw, nx = a.nx, ny = a.ny;
    unsigned long long tm[6] = {0, 0, 0, 0, 0, 0};
    if (TIMING) tm[0] = gtimer();
    uint32_t* P = a.planes + pair * 2 * (int64_t)(a.sxw + a.syw);
    int* bar = a.am.counters + a.batch + pair;
    if (tid < 3) s_cnt[tid] = 0;

    // 1. planes: warp j of the pair's grid row quantises plane words j, j + W, ...
    const int cb0 = a.sched[g], cb1 = a.sched[g + 1], nb = cb1 - cb0;
    {
        const T* X = reinterpret_cast<const T*>(a.op[0].data) + pair * a.op[0].ld;
        const T* Y = reinterpret_cast<const T*>(a.op[1].data) + pair * a.op[1].ld;
        const T x0 = (T)a.op[0].t0, x1 = (T)a.op[0].t1, y0 = (T)a.op[1].t0, y1 = (T)a.op[1].t1;
        const int nw = a.sxw + a.syw, W = G * kPcWarps;
        unsigned nzx = 0, nzy = 0;
        bool nan = false, zero = false;
        __syncthreads();  // s_cnt
        for (int j0 = g * kPcWarps + warp; j0 < nw; j0 += W * kPcWordsPerWarp) {
            T v[kPcWordsPerWarp];
            bool in[kPcWordsPerWarp];
#pragma unroll
            for (int u = 0; u < kPcWordsPerWarp; ++u) {
                const int j = j0 + u * W;
                const bool isx = j < a.sxw;
                const int i = 32 * (isx ? j : j - a.sxw) + lane;
                in[u] = j < nw && i < (isx ? nx : ny);
                v[u] = (T)0;
                if (in[u]) v[u] = isx ? X[i] : Y[i];
            }
#pragma unroll
            for (int u = 0; u < kPcWordsPerWarp; ++u) {
                const int j = j0 + u * W;
                if (j >= nw) break;  // warp-uniform
                const bool isx = j < a.sxw;
                const int c = isx ? level_k1(v[u], x0, x1) : level_k1(v[u], y0, y1);
                const uint32_t sb = __ballot_sync(0xffffffffu, in[u] && c < 0);
                const uint32_t zb = __ballot_sync(0xffffffffu, in[u] && c != 0);
                nan |= v[u] != v[u];
                zero |= in[u] && c == 0;
                if (lane == 0) {
                    // xs | xz | ys | yz
                    const int o = isx ? j : a.sxw + j;
                    P[o] = sb;
                    P[o + (isx ? a.sxw : a.syw)] = zb;
                }
                if (isx) nzx += __popc(zb);
                else nzy += __popc(zb);
            }
        }
        const unsigned fl = (__any_sync(0xffffffffu, nan) ? SF_NONFINITE : 0u) |
                            (__any_sync(0xffffffffu, zero) ? kPcZeroCode : 0u);
        if (lane == 0) {
            if (nzx) atomicAdd(&s_cnt[0], nzx);
            if (nzy) atomicAdd(&s_cnt[1], nzy);
            if (fl) atomicOr(&s_cnt[2], fl);
        }
    }
    // the CTA's unit prefix (warp 0) while the plane stores drain
    int* units = reinterpret_cast<int*>(sm);  // [nb + 1]
    if (warp == 0) {
        int base = 0;
        for (int c0 = 0; c0 < nb; c0 += 32) {
            const int b = cb0 + c0 + lane;
            const int u = b < cb1 ? block_units(a.dlo, a.dhi, nx, ny, b) : 0;
            int incl = u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (b < cb1) units[c0 + lane] = base + incl - u;
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) units[nb] = base;
    }
    __syncthreads();
    if (tid < 3) a.spart[(pair * G + g) * 4 + tid] = s_cnt[tid];
    if (TIMING) tm[1] = gtimer();

    // 2. per-pair grid barrier: every CTA's planes and records are visible
    if (G > 1) {
        if (tid == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(bar) : "memory");
            int seen;
            do {
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
            } while (seen < G);
        }
        __syncthreads();
    }
    if (TIMING) tm[2] = gtimer();

    // 3. stage x's planes and the CTA's y' window; a zero code anywhere
    // selects the two-POPC form
    const int nyq = nxw + nb + 1;  // y' word jl holds y[dlo + 32 (cb0 + jl) + k] at bit k
    uint32_t* xs = reinterpret_cast<uint32_t*>(units) + ((nb + 1 + 3) & ~3);
    uint32_t* xz = xs + nxw;
    uint32_t* ys = xz + nxw;
    uint32_t* yz = ys + nyq;
    int* acc = reinterpret_cast<int*>(yz + nyq);  // [kPcAccBlocks][32]
    int zero = 0;
    {
        const uint32_t* gys = P + 2 * a.sxw;
        const uint32_t* gyz = gys + a.syw;
        for (int i = tid; i < G; i += kPcThreads) zero |= __ldcg(&a.spart[(pair * G + i) * 4 + 2]) & kPcZeroCode;
        for (int w = tid; w < nxw; w += kPcThreads) {
            xs[w] = __ldcg(&P[w]);
            xz[w] = __ldcg(&P[nxw + w]);
        }
        const int s0 = a.dlo + 32 * cb0;
        const int q0 = s0 >> 5, sh = s0 & 31;  // floor division
        for (int w = tid; w < nyq; w += kPcThreads) {
            const int q = q0 + w;
            const bool in0 = q >= 0 && q < a.syw, in1 = q + 1 >= 0 && q + 1 < a.syw;
            const uint32_t s_0 = in0 ? __ldcg(&gys[q]) : 0u, s_1 = in1 ? __ldcg(&gys[q + 1]) : 0u;
            const uint32_t z_0 = in0 ? __ldcg(&gyz[q]) : 0u, z_1 = in1 ? __ldcg(&gyz[q + 1]) : 0u;
            ys[w] = __funnelshift_r(s_0, s_1, sh);
            yz[w] = __funnelshift_r(z_0, z_1, sh);
        }
    }
    const bool allnz = !__syncthreads_or(zero);
    if (TIMING) tm[3] = gtimer();

    int bv = INT_MIN, bt = INT_MAX, bc = 0;  // this thread's (max, smallest index, count)
    for (int pb0 = 0; pb0 < nb; pb0 += kPcAccBlocks) {  // CTA-local block indices
        const int pb1 = min(nb, pb0 + kPcAccBlocks);
        for (int i = tid; i < kPcAccBlocks * 32; i += kPcThreads) acc[i] = 0;
        __syncthreads();
        // this pass's units split evenly over the warps (lane = lag: a warp
        // correlates a run of x words of one block for its 32 lags at once)
        const int u0 = units[pb0], nu = units[pb1] - u0;
        const int my0 = u0 + (int)((long long)nu * warp / kPcWarps);
        const int my1 = u0 + (int)((long long)nu * (warp + 1) / kPcWarps);
        if (my0 < my1) {
            int lo = pb0, hi = pb1;  // block of unit my0: last lb with units[lb] <= my0
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (units[mid] <= my0) lo = mid;
                else hi = mid;
            }
            for (int lb = lo; lb < pb1 && units[lb] < my1; ++lb) {
                int w0, w1;
                block_words(a.dlo, a.dhi, nx, ny, cb0 + lb, w0, w1);
                // units of block lb: kPcBlockUnits of overhead, then one per x word
                const int ws = w0 + max(0, max(my0, units[lb]) - units[lb] - kPcBlockUnits);
                const int we = w0 + max(0, min(my1, units[lb + 1]) - units[lb] - kPcBlockUnits);
                if (ws >= we) continue;
                // interior x words [i0, i1): the word and the 63 y samples its
                // 32 lags read lie inside the signals
                const int yb0 = a.dlo + 32 * (cb0 + lb);  // y sample of x word 0, lag 0
                const int i0 = yb0 >= 0 ? 0 : (31 - yb0) >> 5;
                const int i1 = min(nx >> 5, ny - 63 - yb0 >= 0 ? ((ny - 63 - yb0) >> 5) + 1 : 0);
                const int f0 = allnz ? max(ws, min(we, i0)) : we;
                const int f1 = allnz ? max(f0, min(we, i1)) : we;
                const uint32_t* yq = ys + lb;  // y' words of x word i: yq[i], yq[i + 1]
                const uint32_t* zq = yz + lb;
                int sum = 0;
                auto masked = [&](int i) {
                    const uint32_t yy = __funnelshift_r(yq[i], yq[i + 1], lane);
                    const uint32_t az = xz[i] & __funnelshift_r(zq[i], zq[i + 1], lane);
                    const uint32_t d = (xs[i] ^ yy) & az;
                    sum += allnz ? __popc(d) : __popc(az) - 2 * __popc(d);
                };
                for (int i = ws; i < f0; ++i) masked(i);
                {
                    int i = f0;
                    uint32_t ya = i < f1 ? yq[i] : 0u;
                    for (; i + 4 <= f1; i += 4) {
                        const uint32_t y1 = yq[i + 1], y2 = yq[i + 2], y3 = yq[i + 3], y4 = yq[i + 4];
                        const uint32_t s0 = xs[i], s1 = xs[i + 1], s2 = xs[i + 2], s3 = xs[i + 3];
                        sum += __popc(s0 ^ __funnelshift_r(ya, y1, lane)) + __popc(s1 ^ __funnelshift_r(y1, y2, lane));
                        sum += __popc(s2 ^ __funnelshift_r(y2, y3, lane)) + __popc(s3 ^ __funnelshift_r(y3, y4, lane));
                        ya = y4;
                    }
                    for (; i < f1; ++i) {
                        const uint32_t y1 = yq[i + 1];
                        sum += __popc(xs[i] ^ __funnelshift_r(ya, y1, lane));
                        ya = y1;
                    }
                }
                for (int i = f1; i < we; ++i) masked(i);
                atomicAdd(&acc[(lb - pb0) * 32 + lane], sum);
            }
        }
        __syncthreads();  // every partial sum of this pass has landed
        for (int i = tid; i < (pb1 - pb0) * 32; i += kPcThreads) {
            const int d = a.dlo + 32 * (cb0 + pb0) + i;
            if (d > a.dhi) continue;
            int val = acc[i];
            if (allnz) val = max(0, min(nx, ny - d) - max(0, -d)) - 2 * val;  // overlap - 2 mismatches
            const int t = d + nx - 1;
            if (val > bv) {
                bv = val;
                bt = t;
                bc = 1;
            } else if (val == bv) {
                bt = min(bt, t);
                ++bc;
            }
        }
        __syncthreads();  // acc reads done before the next pass zeroes it
    }
    if (TIMING) tm[4] = gtimer();

    // 4. per-CTA record, ticket; the pair's last CTA merges and writes the result
    warp_best(bv, bt, bc);
    if (lane == 0) {
        s_best[warp][0] = bv;
        s_best[warp][1] = bt;
        s_best[warp][2] = bc;
    }
    __syncthreads();
    if (warp == 0) {
        bv = lane < kPcWarps ? s_best[lane][0] : INT_MIN;
        bt = lane < kPcWarps ? s_best[lane][1] : INT_MAX;
        bc = lane < kPcWarps ? s_best[lane][2] : 0;
        warp_best(bv, bt, bc);
        if (lane == 0) {
            long long* pp = a.am.partials + (pair * a.am.pstride + g) * 3;
            pp[0] = bv;
            pp[1] = bt;
            pp[2] = bc;
            int ticket;
            asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(ticket) : "l"(a.am.counters + pair) : "memory");
            s_last = ticket == G - 1;
        }
    }
    __syncthreads();
    if (TIMING && tid == 0) {
        tm[5] = gtimer();
        if (g == 0 || g == G / 2 || g == G - 1 || s_last)
            printf("popc cta %d/%d blocks [%d,%d) units %d: planes %.2f barrier %.2f stage %.2f corr %.2f "
                   "ticket %.2f us%s\n",
                   g, G, cb0, cb1, units[nb], (tm[1] - tm[0]) / 1e3, (tm[2] - tm[1]) / 1e3, (tm[3] - tm[2]) / 1e3,
                   (tm[4] - tm[3]) / 1e3, (tm[5] - tm[4]) / 1e3, s_last ? " (last)" : "");
    }
    if (!s_last) return;
    // last CTA: every CTA's record (one per thread) and counts
    const volatile long long* pp = a.am.partials + pair * a.am.pstride * 3;
    bv = INT_MIN;
    bt = INT_MAX;
    bc = 0;
    unsigned cx = 0, cy = 0, fl = 0;
    for (int i = tid; i < G; i += kPcThreads) {
        const int v = (int)pp[3 * i], t = (int)pp[3 * i + 1], c = (int)pp[3 * i + 2];
        if (v > bv) {
            bv = v;
            bt = t;
            bc = c;
        } else if (v == bv) {
            bt = min(bt, t);
            bc += c;
        }
        const unsigned* sp = a.spart + (pair * G + i) * 4;
        cx += __ldcg(sp);
        cy += __ldcg(sp + 1);
        fl |= __ldcg(sp + 2);
    }
    warp_best(bv, bt, bc);
    cx = __reduce_add_sync(0xffffffffu, cx);
    cy = __reduce_add_sync(0xffffffffu, cy);
    fl = __reduce_or_sync(0xffffffffu, fl);
    __syncthreads();  // s_best / s_cnt reads of the first merge are done
    if (tid < 3) s_cnt[tid] = 0;
    if (lane == 0) {
        s_best[warp][0] = bv;
        s_best[warp][1] = bt;
        s_best[warp][2] = bc;
    }
    __syncthreads();
    if (lane == 0 && (cx | cy | fl)) {
        atomicAdd(&s_cnt[0], cx);
        atomicAdd(&s_cnt[1], cy);
        atomicOr(&s_cnt[2], fl);
    }
    __syncthreads();
    if (warp == 0) {
        bv = lane < kPcWarps ? s_best[lane][0] : INT_MIN;
        bt = lane < kPcWarps ? s_best[lane][1] : INT_MAX;
        bc = lane < kPcWarps ? s_best[lane][2] : 0;
        warp_best(bv, bt, bc);
        if (lane == 0) {
            // sum of squares = nonzero count for 1-level codes
            unsigned long long* st = a.stats + pair * 8;
            st[0] = s_cnt[0];
            st[1] = s_cnt[0];
            st[2] = s_cnt[2] & ~kPcZeroCode;
            st[3] = 0;
            st[4] = s_cnt[1];
            st[5] = s_cnt[1];
            st[6] = 0;
            st[7] = 0;
            write_result(reinterpret_cast<long long*>(a.am.results) + pair * 8, Best{bv, bt, bc}, a.am.first_lag, st);
            a.am.counters[pair] = 0;  // ticket
            *bar = 0;                 // every CTA of the pair is past the barrier
        }
    }
}

// ------------------------------------------------------------------ host

static void popc_window(const NttCall& c, int64_t nx, PopcArgs& a)
{
    const int64_t dlo = c.am.t_lo - (nx - 1), dhi = c.am.t_hi - (nx - 1);
    a.dlo = (int)dlo;
    a.dhi = (int)dhi;
    a.nx = (int)nx;
    a.ny = (int)c.op[1].n;
    a.nblk = (int)((dhi - dlo + 1 + 31) / 32);
    a.sxw = (int)((nx + 31) / 32);
    a.syw = (int)((c.op[1].n + 31) / 32);
    a.batch = (int)c.batch;
}

// dynamic shared memory of a CTA holding blocks of at most `nbmax` blocks:
// unit prefix, x's planes, the y' window and the accumulators
static size_t popc_smem(const PopcArgs& a, int64_t nbmax)
{
    return (size_t)(((nbmax + 1 + 3) & ~3ll) + 2ll * a.sxw + 2 * (a.sxw + nbmax + 1) + kPcAccBlocks * 32) * 4;
}

// resident CTAs per SM for a dynamic shared memory size, cached per device
static int popc_per_sm(size_t smem)
{
    static int cache[64][32] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    const int bucket = (int)((smem + 4095) / 4096) < 32 ? (int)((smem + 4095) / 4096) : 31;
    if (!cache[dev][bucket]) {
        int n = 0;
        if (set_max_smem((const void*)k_popc<float, false>, kPcMaxSmem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, (const void*)k_popc<float, false>, kPcThreads,
                                                          (size_t)bucket * 4096) != cudaSuccess || n < 1) {
            cudaGetLastError();
            n = 1;
        }
        cache[dev][bucket] = n;
    }
    return cache[dev][bucket];
}

// CTAs per pair: every pair's CTAs resident at once (cooperative launch),
// the SMs shared by the batch, at most one per ~1024 units of work
static int popc_ctas(const NttCall& c, const PopcArgs& a)
{
    const int64_t units = (int64_t)a.nblk * (a.sxw + kPcBlockUnits);
    const int64_t resident = (int64_t)device_sms() * popc_per_sm(popc_smem(a, a.nblk));
    int64_t G = resident / c.batch;
    if (G > (units + 1023) / 1024) G = (units + 1023) / 1024;
    if (G > a.nblk) G = a.nblk;
    if (G > kMaxPartialsLarge) G = kMaxPartialsLarge;
    return G < 1 ? 1 : (int)G;
}

// contiguous block ranges of G CTAs minimising the largest unit sum (binary
// search on the bound, greedy fill); out[g] = first block of CTA g
void popc_schedule(const NttCall& c, int64_t nx, int* G_out, std::vector<int>& out)
{
    PopcArgs a;
    popc_window(c, nx, a);
    const int G = popc_ctas(c, a);
    std::vector<int> u((size_t)a.nblk);
    int64_t total = 0, umax = 0;
    for (int b = 0; b < a.nblk; ++b) {
        u[b] = block_units(a.dlo, a.dhi, a.nx, a.ny, b);
        total += u[b];
        umax = std::max<int64_t>(umax, u[b]);
    }
    auto fits = [&](int64_t cap, std::vector<int>* starts) {
        int k = 0;
        int64_t run = 0;
        if (starts) starts->assign(1, 0);
        for (int b = 0; b < a.nblk; ++b) {
            if (run + u[b] > cap && run > 0) {
                if (++k >= G) return false;
                if (starts) starts->push_back(b);
                run = 0;
            }
            run += u[b];
        }
        return true;
    };
    int64_t lo = std::max<int64_t>(umax, (total + G - 1) / G), hi = total;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (fits(mid, nullptr)) hi = mid;
        else lo = mid + 1;
    }
    fits(lo, &out);
    out.resize((size_t)G + 1, a.nblk);  // trailing CTAs (if any) get empty ranges
    *G_out = G;
}

// eligibility: argmax mode, 1-level quantisers on float rows, x <= 2^16 and
// y <= 2^24 samples, a CTA's shared memory within 200 KB; on AUTO also
// little enough work that one GPU-wide launch beats the NTT's three
// (batch * nx * window <= 2^31 code products)
bool popc_eligible(const NttCall& c, int64_t nx, int64_t ny, bool auto_path)
{
    if (auto_path && !c.knobs->popc) return false;
    if (c.op[0].q.mode != QM_K1 || c.op[1].q.mode != QM_K1) return false;
    if (c.op[0].dtype == DT_I64 || c.op[0].dtype != c.op[1].dtype) return false;
    if (nx > 65536 || ny > (1 << 24)) return false;
    const double W = (double)(c.am.t_hi - c.am.t_lo + 1);
    if (auto_path && (double)c.batch * (double)nx * W > 2147483648.0) return false;
    PopcArgs a;
    popc_window(c, nx, a);
    return popc_smem(a, a.nblk) <= (size_t)kPcMaxSmem;
}

// global plane words of a popc call (scratch)
size_t popc_planes_words(int64_t batch, int64_t nx, int64_t ny)
{
    return (size_t)batch * 2 * ((nx + 31) / 32 + (ny + 31) / 32);
}

cudaError_t popc_run(const NttCall& c, int64_t nx, cudaStream_t s)
{
    PopcArgs a;
    for (int i = 0; i < 2; ++i) a.op[i] = PopcOp{c.op[i].data, c.op[i].ld, c.op[i].q.thr[0], c.op[i].q.thr[1]};
    popc_window(c, nx, a);
    a.stats = c.stats;
    a.am = c.am;
    a.planes = c.popc_planes;
    a.spart = c.popc_spart;
    a.sched = c.popc_sched;
    const int G = c.popc_G;
    if (G > c.am.pstride || !a.sched) return cudaErrorInvalidValue;
    const size_t smem = popc_smem(a, a.nblk);
    const bool f32 = c.op[0].dtype == DT_F32, tm = c.knobs->popc_timing != 0;
    const void* fn = f32 ? (tm ? (const void*)k_popc<float, true> : (const void*)k_popc<float, false>)
                         : (tm ? (const void*)k_popc<double, true> : (const void*)k_popc<double, false>);
    if (cudaError_t e = set_max_smem(fn, kPcMaxSmem); e != cudaSuccess) return e;
    if (c.prof) c.prof->pre(KK_POPC, s);
    void* args[] = {(void*)&a};
    // cooperative: the per-pair barrier needs every CTA of the pair resident
    cudaError_t e = G > 1 ? cudaLaunchCooperativeKernel(fn, dim3((unsigned)G, (unsigned)c.batch), dim3(kPcThreads), args, smem, s)
                          : cudaLaunchKernel(fn, dim3(1, (unsigned)c.batch), dim3(kPcThreads), args, smem, s);
    if (c.prof) c.prof->post(KK_POPC, s);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace qx
