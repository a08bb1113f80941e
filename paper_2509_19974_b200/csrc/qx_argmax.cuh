// qx_argmax.cuh -- the fused argmax epilogue shared by the NTT and popc
// paths: (value, smallest correlogram index, count) records, the block /
// per-pair merge through per-CTA partials and a last-CTA ticket, and the
// qx_result record writer.  argmax_set semantics: estimator.py:50-57.
#pragma once
#include <climits>

#include "qx_internal.h"

namespace qx {


struct Best {
    long long v, t, c;
};

__device__ __forceinline__ void best_merge(Best& a, const Best& b)
{
    if (b.v > a.v) a = b;
    else if (b.v == a.v) { a.t = min(a.t, b.t); a.c += b.c; }
}

__device__ __forceinline__ void best_add(Best& a, long long v, long long t)
{
    if (v > a.v) { a.v = v; a.t = t; a.c = 1; }
    else if (v == a.v) { a.t = min(a.t, t); a.c += 1; }
}

__device__ __forceinline__ Best best_init() { return Best{LLONG_MIN, LLONG_MAX, 0}; }

// one qx_result record (include/qxcorr_b200.h) from the peak summary and the
// pass-1 statistics of a pair
__device__ inline void write_result(long long* res, const Best& r, long long first_lag, const unsigned long long* st)
{
    const long long nzx = (long long)st[1], nzy = (long long)st[5];
    const unsigned f = (unsigned)(st[2] | st[6]);
    int flags = 0;
    if (nzx == 0) flags |= 1;
    if (nzy == 0) flags |= 2;
    if (f & SF_NONFINITE) flags |= 4;
    if (f & SF_CODE_RANGE) flags |= 8;
    int status = 0;
    if (flags & 4) status = 9;       // QX_ERR_NONFINITE
    else if (flags & 8) status = 1;  // QX_ERR_INVALID (codes exceed bound)
    else if (flags & 3) status = 2;  // QX_DEGENERATE_QUANTIZATION
    res[0] = r.v;
    res[1] = first_lag + r.t;
    res[2] = r.c;
    res[3] = (long long)st[0];
    res[4] = (long long)st[4];
    res[5] = nzx;
    res[6] = nzy;
    res[7] = ((long long)status << 32) | (unsigned)flags;
}

// block-wide reduce (NW warps), per-block partial, last block writes the qx_result
template <int NW>
__device__ void argmax_finish(Best b, const ArgmaxOut& am, const unsigned long long* stats, int64_t pair,
                              int nblk, int blk)
{
    __shared__ Best sb[NW];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        Best o2{__shfl_xor_sync(0xffffffffu, b.v, o), __shfl_xor_sync(0xffffffffu, b.t, o),
                __shfl_xor_sync(0xffffffffu, b.c, o)};
        best_merge(b, o2);
    }
    if (lane == 0) sb[warp] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        Best r = sb[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best_merge(r, sb[w]);
        long long* pp = am.partials + (pair * am.pstride + blk) * 3;
        pp[0] = r.v; pp[1] = r.t; pp[2] = r.c;
        __threadfence();
        const int ticket = atomicAdd(am.counters + pair, 1);
        s_last = (ticket == nblk - 1);
    }
    __syncthreads();
    if (!s_last) return;
    // last block: every thread merges a strided share of the partials
    __threadfence();
    Best r = best_init();
    const volatile long long* pp = am.partials + pair * am.pstride * 3;
    for (int i = threadIdx.x; i < nblk; i += blockDim.x) best_merge(r, Best{pp[3 * i], pp[3 * i + 1], pp[3 * i + 2]});
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        Best o2{__shfl_xor_sync(0xffffffffu, r.v, o), __shfl_xor_sync(0xffffffffu, r.t, o),
                __shfl_xor_sync(0xffffffffu, r.c, o)};
        best_merge(r, o2);
    }
    __syncthreads();  // sb reads of the first merge are done
    if (lane == 0) sb[warp] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best_merge(r, sb[w]);
        write_result(reinterpret_cast<long long*>(am.results) + pair * 8, r, am.first_lag, stats + pair * 8);
        am.counters[pair] = 0;
    }
}

}  // namespace qx
