// qx_quant.cu -- quantiser support: exact threshold tables (host) and the
// standalone quantise kernel behind quantize.apply (quantize.py:105-107).
//
// The reference evaluates Quantizer.__call__ (quantize.py:53-65) in float64
// after upcasting every sample (signals.py:46).  Every reference quantiser is
// monotone non-decreasing in its input, so for a given input type the map is
// fully described by 2k thresholds T[i] = min{ v : q(v) >= i - k + 1 }, found
// here by bisection over the totally ordered bit patterns of that type while
// evaluating the reference formula in float64.  The kernels then compute
// level(v) = -k + #{i : v >= T[i]}, which is exact for every finite or
// infinite input (NaN is reported, the reference's result for it is
// undefined).  This file is compiled without fast-math or FMA contraction.
#include <cmath>
#include <cstring>

#include "qx_internal.h"

namespace qx {

// reference map, float64 (quantize.py:53-65)
static long long ref_level(double v, int kind, long long k, double step, const double* thr)
{
    if (kind == 0) return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0);  // np.sign
    if (kind == 1) {
        volatile double a = std::fabs(v) / step;  // volatile: no contraction
        double s = v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0);
        double o = s * std::floor(a + 0.5);
        if (o > (double)k) o = (double)k;
        if (o < -(double)k) o = -(double)k;
        return (long long)o;
    }
    long long lo = 0, hi = 2 * k;  // searchsorted(t, v, side="right")
    while (lo < hi) {
        long long mid = (lo + hi) >> 1;
        if (thr[mid] <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo - k;
}

static inline uint32_t f32_key(float f)
{
    uint32_t b;
    std::memcpy(&b, &f, 4);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
static inline float f32_from_key(uint32_t k)
{
    uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}
static inline uint64_t f64_key(double f)
{
    uint64_t b;
    std::memcpy(&b, &f, 8);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
static inline double f64_from_key(uint64_t k)
{
    uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    double f;
    std::memcpy(&f, &b, 8);
    return f;
}

// out[i] (i < 2k) = smallest value of the input type with level >= i-k+1
int thresholds(int kind, long long k, double step, const double* thr, int dtype, double* out)
{
    for (long long i = 0; i < 2 * k; ++i) {
        const long long want = i - k + 1;
        if (dtype == DT_F32) {
            uint32_t lo = f32_key(-INFINITY), hi = f32_key(INFINITY);
            while (lo < hi) {
                uint32_t mid = lo + (hi - lo) / 2;
                if (ref_level((double)f32_from_key(mid), kind, k, step, thr) >= want) hi = mid;
                else lo = mid + 1;
            }
            out[i] = (double)f32_from_key(lo);
        } else {
            uint64_t lo = f64_key(-INFINITY), hi = f64_key(INFINITY);
            while (lo < hi) {
                uint64_t mid = lo + (hi - lo) / 2;
                if (ref_level(f64_from_key(mid), kind, k, step, thr) >= want) hi = mid;
                else lo = mid + 1;
            }
            out[i] = f64_from_key(lo);
        }
    }
    return 0;
}

// standalone quantise (apply): codes[b*n + i] = level(x[b*ld + i])
struct QuantArgs {
    const void* x;
    int64_t ld, n, batch;
    int64_t* codes;
    unsigned long long* sums;  // [batch][2]: sumsq, nnz
    unsigned* flags;
    QTable q;
};

template <typename T, int QM>
__global__ void __launch_bounds__(256) k_quantize(const __grid_constant__ QuantArgs a)
{
    __shared__ T sthr[kMaxThr];
    for (int i = threadIdx.x; i < a.q.tsize; i += blockDim.x) sthr[i] = (T)a.q.thr[i];
    __syncthreads();
    const int64_t b = blockIdx.y;
    const T* x = reinterpret_cast<const T*>(a.x) + b * a.ld;
    const T t0 = sthr[0], t1 = sthr[1], inv_step = (T)a.q.inv_step;
    unsigned long long ssq = 0, nnz = 0;
    unsigned fl = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
        const T v = x[i];
        if (v != v) fl |= SF_NONFINITE;
        int c;
        if constexpr (QM == QM_K1) c = level_k1(v, t0, t1);
        else if constexpr (QM == QM_UNIFORM) c = level_uniform(v, sthr, a.q.k, inv_step);
        else c = level_bsearch(v, sthr, a.q.tbits) - a.q.k;
        a.codes[b * a.n + i] = c;
        ssq += (unsigned long long)((long long)c * c);
        nnz += (c != 0);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
        fl |= __shfl_xor_sync(0xffffffffu, fl, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (a.sums) {
            atomicAdd(a.sums + 2 * b, ssq);
            atomicAdd(a.sums + 2 * b + 1, nnz);
        }
        if (fl) atomicOr(a.flags, fl);
    }
}


// Bit-packed codes (BASELINE north_star subsystem 1): every thread quantises
// 4 consecutive samples from one 16-byte (float4) or two 16-byte (double2)
// vector loads, 32 / (4 BITS) neighbouring lanes OR their fields into one
// little-endian 32-bit word (sample i at bit BITS * (i % (32 / BITS))), and
// the first lane of the group stores it.  BITS = 2, 4, 8 hold the code in
// two's complement; BITS = 1 writes two planes, sign (code < 0) then nonzero
// (code != 0), for 1-level quantisers.  Per-row sum of squares / nonzero
// counts are reduced per CTA (one 64-bit atomic per CTA and row).
struct PackArgs {
    const void* x;
    int64_t ld, n, batch;
    uint32_t* codes;
    int64_t wpr;               // words per row (both planes for BITS = 1)
    unsigned long long* sums;  // [batch][2]: sumsq, nnz
    unsigned* flags;           // QX_RF_NONFINITE if any row holds a NaN
    int vec;                   // rows 16-byte aligned: vector loads
    QTable q;
};

template <typename T>
__device__ __forceinline__ void load4(const T* row, int64_t i, int64_t n, bool vec, T (&v)[4])
{
    if (vec && i + 3 < n) {
        if constexpr (sizeof(T) == 4) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(row + i));
            v[0] = f.x, v[1] = f.y, v[2] = f.z, v[3] = f.w;
        } else {
            const double2 a = __ldg(reinterpret_cast<const double2*>(row + i));
            const double2 b = __ldg(reinterpret_cast<const double2*>(row + i + 2));
            v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = i + k < n ? row[i + k] : (T)0;  // level(0) = 0 (padding)
}

constexpr int kPackUnroll = 4;  // 4-sample quads per thread and trip (16-64 B in flight each)

template <typename T, int QM, int BITS>
__global__ void __launch_bounds__(256) k_quantize_packed(const __grid_constant__ PackArgs a)
{
    __shared__ T sthr[kMaxThr];
    __shared__ unsigned long long s_sum[2];
    __shared__ unsigned s_fl;
    for (int i = threadIdx.x; i < a.q.tsize; i += blockDim.x) sthr[i] = (T)a.q.thr[i];
    if (threadIdx.x < 2) s_sum[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_fl = 0;
    __syncthreads();
    const int64_t b = blockIdx.y;
    const T* row = reinterpret_cast<const T*>(a.x) + b * a.ld;
    uint32_t* out = a.codes + b * a.wpr;
    const T t0 = sthr[0], t1 = sthr[1], inv_step = (T)a.q.inv_step;
    constexpr int LPW = BITS == 1 ? 8 : 32 / (4 * BITS);  // lanes per output word
    const int lane = threadIdx.x & 31;
    const int64_t nq = (a.n + 3) / 4;  // 4-sample quads, padded to whole words below
    const int64_t nqw = (nq + LPW - 1) / LPW * LPW;
    const int64_t nw1 = (a.n + 31) / 32;  // plane words (BITS = 1)
    unsigned long long ssq = 0, nnz = 0;
    bool nan = false;
    // kPackUnroll quads per thread and trip, every load issued before the first use
    const int64_t span = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x; q0 < nqw; q0 += span * kPackUnroll) {
        T v[kPackUnroll][4];
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) load4(row, 4 * (q0 + u * span + threadIdx.x), a.n, a.vec, v[u]);
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) {
            const int64_t qi = q0 + u * span + threadIdx.x;  // lanes past the end quantise zeros
            if (q0 + u * span >= nqw) break;                // warp-uniform (span, q0 multiples of 32)
            uint32_t f = 0, zf = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const T x = v[u][k];
                int c;
                if constexpr (QM == QM_K1) c = level_k1(x, t0, t1);
                else if constexpr (QM == QM_UNIFORM) c = level_uniform(x, sthr, a.q.k, inv_step);
                else c = level_bsearch(x, sthr, a.q.tbits) - a.q.k;
                nan |= x != x;
                ssq += (unsigned)(c * c);
                nnz += c != 0;
                if constexpr (BITS == 1) {
                    f |= (uint32_t)(c < 0) << k;
                    zf |= (uint32_t)(c != 0) << k;
                } else {
                    f |= ((uint32_t)c & ((1u << BITS) - 1u)) << (BITS * k);
                }
            }
            const int sh = (lane % LPW) * 4 * BITS;
            f <<= sh;
            zf <<= sh;
#pragma unroll
            for (int o = 1; o < LPW; o <<= 1) {
                f |= __shfl_xor_sync(0xffffffffu, f, o);
                zf |= __shfl_xor_sync(0xffffffffu, zf, o);
            }
            const int64_t w = qi / LPW;  // output word
            if (lane % LPW == 0) {
                if constexpr (BITS == 1) {
                    if (w < nw1) {
                        out[w] = f;
                        out[nw1 + w] = zf;
                    }
                } else if (w < a.wpr) {
                    out[w] = f;
                }
            }
        }
    }
    // per-CTA sums (warp shuffles, then one shared atomic per warp)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
    }
    nan = __any_sync(0xffffffffu, nan);
    if (lane == 0) {
        atomicAdd(&s_sum[0], ssq);
        atomicAdd(&s_sum[1], nnz);
        if (nan) atomicOr(&s_fl, 4u);  // QX_RF_NONFINITE (qxcorr_b200.h)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.sums) {
            if (s_sum[0]) atomicAdd(a.sums + 2 * b, s_sum[0]);
            if (s_sum[1]) atomicAdd(a.sums + 2 * b + 1, s_sum[1]);
        }
        if (s_fl) atomicOr(a.flags, s_fl);
    }
}

template <typename T, int QM>
static void packed_dispatch_bits(int bits, dim3 grid, const PackArgs& a, cudaStream_t s)
{
    switch (bits) {
    case 1: k_quantize_packed<T, QM, 1><<<grid, 256, 0, s>>>(a); break;
    case 2: k_quantize_packed<T, QM, 2><<<grid, 256, 0, s>>>(a); break;
    case 4: k_quantize_packed<T, QM, 4><<<grid, 256, 0, s>>>(a); break;
    default: k_quantize_packed<T, QM, 8><<<grid, 256, 0, s>>>(a); break;
    }
}

// words per row of a packed row of n samples
int64_t packed_words(int64_t n, int bits)
{
    return bits == 1 ? 2 * ((n + 31) / 32) : (n * bits + 31) / 32;
}

cudaError_t quantize_packed_launch(const void* x, int64_t ld, int64_t n, int64_t batch, int dtype, const QTable& q,
                                   int bits, uint32_t* codes, unsigned long long* sums, unsigned* flags, int sms,
                                   cudaStream_t s)
{
    PackArgs a;
    a.x = x;
    a.ld = ld;
    a.n = n;
    a.batch = batch;
    a.codes = codes;
    a.wpr = packed_words(n, bits);
    a.sums = sums;
    a.flags = flags;
    const size_t es = dtype == DT_F32 ? 4 : 8;
    a.vec = ((uintptr_t)x % 16 == 0) && ((ld * es) % 16 == 0);
    a.q = q;
    // CTAs: ~8 per SM over the whole batch, at least one per row
    const int64_t quads = (n + 3) / 4;
    int64_t gx = (quads + 256 * kPackUnroll - 1) / (256 * kPackUnroll);
    const int64_t cap = (8 * (int64_t)sms + batch - 1) / batch;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    const dim3 grid((unsigned)gx, (unsigned)batch);
    if (dtype == DT_F32) {
        if (q.mode == QM_K1) packed_dispatch_bits<float, QM_K1>(bits, grid, a, s);
        else if (q.mode == QM_UNIFORM) packed_dispatch_bits<float, QM_UNIFORM>(bits, grid, a, s);
        else packed_dispatch_bits<float, QM_BSEARCH>(bits, grid, a, s);
    } else {
        if (q.mode == QM_K1) packed_dispatch_bits<double, QM_K1>(bits, grid, a, s);
        else if (q.mode == QM_UNIFORM) packed_dispatch_bits<double, QM_UNIFORM>(bits, grid, a, s);
        else packed_dispatch_bits<double, QM_BSEARCH>(bits, grid, a, s);
    }
    return cudaGetLastError();
}

// PCM16 (little-endian int16) -> float32 pcm / 32768, the sample decode of
// signalgen.load_wav_bytes (signalgen.py:150-172) on the device.  Exact:
// every value is a multiple of 2^-15 with at most 16 significant bits, so
// the float32 path quantises it exactly as the reference's float64 does.
// 8 samples (16 B in, 32 B out) per thread-iteration, grid-stride; the
// caller's buffers are cudaMalloc-aligned, the tail is scalar.
__global__ void __launch_bounds__(256) k_pcm16_to_f32(const int16_t* __restrict__ in, int64_t n,
                                                      float* __restrict__ out)
{
    const int64_t n8 = n >> 3;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint4* in8 = reinterpret_cast<const uint4*>(in);
    float4* out4 = reinterpret_cast<float4*>(out);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += stride) {
        const uint4 w = __ldg(&in8[i]);
        const uint32_t v[4] = {w.x, w.y, w.z, w.w};
        float f[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            f[2 * j] = (float)(int16_t)(v[j] & 0xffffu) * (1.0f / 32768.0f);
            f[2 * j + 1] = (float)(int16_t)(v[j] >> 16) * (1.0f / 32768.0f);
        }
        out4[2 * i] = make_float4(f[0], f[1], f[2], f[3]);
        out4[2 * i + 1] = make_float4(f[4], f[5], f[6], f[7]);
    }
    for (int64_t i = (n8 << 3) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (float)in[i] * (1.0f / 32768.0f);
}

cudaError_t pcm16_launch(const void* in, int64_t n, float* out, int sms, cudaStream_t s)
{
    int64_t blocks = ((n >> 3) + 255) / 256;
    if (blocks > 8 * (int64_t)sms) blocks = 8 * (int64_t)sms;
    if (blocks < 1) blocks = 1;
    k_pcm16_to_f32<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const int16_t*>(in), n, out);
    return cudaGetLastError();
}

cudaError_t quantize_launch(const void* x, int64_t ld, int64_t n, int64_t batch, int dtype, const QTable& q,
                            int64_t* codes, unsigned long long* sums, unsigned* flags, cudaStream_t s)
{
    QuantArgs a;
    a.x = x;
    a.ld = ld;
    a.n = n;
    a.batch = batch;
    a.codes = codes;
    a.sums = sums;
    a.flags = flags;
    a.q = q;
    int gx = (int)((n + 255) / 256);
    if (gx > 1184) gx = 1184;
    dim3 grid(gx, (unsigned)batch);
    if (dtype == DT_F32) {
        if (q.mode == QM_K1) k_quantize<float, QM_K1><<<grid, 256, 0, s>>>(a);
        else if (q.mode == QM_UNIFORM) k_quantize<float, QM_UNIFORM><<<grid, 256, 0, s>>>(a);
        else k_quantize<float, QM_BSEARCH><<<grid, 256, 0, s>>>(a);
    } else {
        if (q.mode == QM_K1) k_quantize<double, QM_K1><<<grid, 256, 0, s>>>(a);
        else if (q.mode == QM_UNIFORM) k_quantize<double, QM_UNIFORM><<<grid, 256, 0, s>>>(a);
        else k_quantize<double, QM_BSEARCH><<<grid, 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace qx
