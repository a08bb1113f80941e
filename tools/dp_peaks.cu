// dp_peaks.cu -- does the FP64 pipe pay for the Shoup quotient?
//
// The lazy Shoup butterfly spends one IMAD.HI.U32 (the quotient estimate
// floor(a*wq / 2^32)) and two IMAD on the heavy FMA sub-pipe.  B200 keeps a
// full-rate FP64 pipe that the integer kernels leave idle; the quotient
// rint(a*w/p) is one DFMA on it:
//     (2^52 + a) * (W / 2^52) + (2^52 - W)  =  2^52 + a*W/2^52   (exact product,
//     one rounding to the integer grid of [2^52, 2^53)),  W = rint(w 2^52 / p),
// whose low mantissa word is q = rint(a w / p + e), |e| <= 2^-21; then
// r = a*w - q*p + p lies in (0.49p, 1.51p).
// Measures, on register-resident data: IMAD, IMAD.HI (with addend, nothing
// else in the loop), IMAD.WIDE, DFMA, DFMA and IMAD interleaved, the Shoup
// butterfly, the two DFMA butterflies and mixed loops in which every 3rd /
// 4th / 8th / 16th butterfly takes its quotient from the FP64 pipe; checks
// the DFMA product against the exact residue for every 32-bit input and eight
// twiddles.  Output: one JSON object.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2509_19974_b200/csrc/qx_common.cuh"

using namespace qx;

constexpr int ITERS = 4096;
constexpr int CH = 16;
constexpr uint32_t kP = 1012924417u;

struct TwD {
    double winv;  // W / 2^52
    double k;     // 2^52 - W
    uint32_t w;
};

__device__ __forceinline__ uint32_t mul_dfma1(uint32_t a, const TwD& t, uint32_t p, uint32_t np)
{
    const double y = fma(__hiloint2double(0x43300000, (int)a), t.winv, t.k);
    const uint32_t q = (uint32_t)__double2loint(y);
    return q * np + (a * t.w + p);
}

__device__ __forceinline__ uint32_t mul_dfma2(uint32_t a, const TwD& t, uint32_t p, uint32_t np)
{
    const double d = __hiloint2double(0x43300000, (int)a) - 4503599627370496.0;
    const double y = fma(d, t.winv, 4503599627370496.0);
    const uint32_t q = (uint32_t)__double2loint(y);
    return q * np + (a * t.w + p);
}

template <int MODE>
__global__ void k_bfly(uint32_t* out, uint32_t seed, uint2 w, TwD t)
{
    ModP m{kP, 2u * kP, 0, 0};
    const uint32_t np = 0u - kP;
    uint32_t a[CH], b[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        a[i] = (seed * (threadIdx.x + 7 * i)) % m.p;
        b[i] = (seed * (threadIdx.x + 3 * i + 1)) % m.p;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (MODE == 0 || (MODE >= 3 && (i % MODE) != 0)) bfly_dif(a[i], b[i], w, m);
            else {
                const uint32_t s = a[i] + b[i] + m.zero;
                const uint32_t d = a[i] - b[i] + m.p2;
                a[i] = red2p(s, m.p2);
                b[i] = MODE != 2 ? mul_dfma1(d, t, m.p, np) : mul_dfma2(d, t, m.p, np);
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s ^= a[i] ^ b[i];
    if (s == 0x12345678u) out[threadIdx.x] = s;
}

template <int MODE>
__global__ void k_stream(uint32_t* out, uint32_t seed, double c)
{
    uint32_t a[CH];
    unsigned long long l[CH];
    double d[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        a[i] = seed + threadIdx.x * i + 1;
        l[i] = a[i];
        d[i] = (double)a[i];
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (MODE == 0) a[i] = a[i] * 0x9E3779B1u + seed;
            if (MODE == 1) a[i] = __umulhi(a[i], 0x9E3779B1u) + seed;
            if (MODE == 2) l[i] = (unsigned long long)(uint32_t)l[i] * 0x9E3779B1u + l[i];
            if (MODE == 3) d[i] = fma(d[i], c, c);
            if (MODE == 4) {
                d[i] = fma(d[i], c, c);
                a[i] = a[i] * 0x9E3779B1u + seed;
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s ^= a[i] ^ (uint32_t)l[i] ^ (uint32_t)__double2loint(d[i]);
    if (s == 0x12345678u) out[threadIdx.x] = s;
}

// exactness: every a in a strided sweep of [0, 2^32) and the edges, a few twiddles
__global__ void k_check(unsigned long long* bad, uint32_t w, TwD t)
{
    const uint32_t np = 0u - kP;
    const unsigned long long n = 1ull << 32;
    for (unsigned long long a = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; a < n;
         a += (unsigned long long)gridDim.x * blockDim.x) {
        const uint32_t r1 = mul_dfma1((uint32_t)a, t, kP, np), r2 = mul_dfma2((uint32_t)a, t, kP, np);
        const uint32_t want = (uint32_t)((a * w) % kP);
        if (r1 >= 2u * kP || r1 % kP != want || r2 >= 2u * kP || r2 % kP != want) atomicAdd(bad, 1ull);
    }
}

template <typename F>
static double time_kernel(F launch, int reps)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps / 1e3;
}

static TwD make_tw(uint32_t w)
{
    const unsigned __int128 num = ((unsigned __int128)w << 52) + kP / 2;
    const uint64_t W = (uint64_t)(num / kP);
    TwD t;
    t.winv = (double)W / 4503599627370496.0;
    t.k = 4503599627370496.0 - (double)W;
    t.w = w;
    return t;
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, 4096);
    unsigned long long* bad;
    cudaMalloc(&bad, 8);
    cudaMemset(bad, 0, 8);
    const uint32_t ws[] = {1u, 2u, 123456789u, kP - 1, kP / 2, kP / 2 + 1, 998244353u % kP, 3u};
    for (uint32_t w : ws) k_check<<<sms * 8, 256>>>(bad, w, make_tw(w));
    unsigned long long hbad = 0;
    cudaMemcpy(&hbad, bad, 8, cudaMemcpyDeviceToHost);

    const int blocks = sms * 8, threads = 256;
    const double per = (double)blocks * threads * ITERS * CH;
    const uint2 w = make_uint2(123456789u, (uint32_t)(((uint64_t)123456789u << 32) / kP));
    const TwD t = make_tw(123456789u);
    const double b0 = time_kernel([&] { k_bfly<0><<<blocks, threads>>>(out, 3, w, t); }, 5);
    const double b1 = time_kernel([&] { k_bfly<1><<<blocks, threads>>>(out, 3, w, t); }, 5);
    const double b2 = time_kernel([&] { k_bfly<2><<<blocks, threads>>>(out, 3, w, t); }, 5);
    // mixed loops: every MODE-th butterfly takes its quotient from the FP64 pipe
    const double b3 = time_kernel([&] { k_bfly<3><<<blocks, threads>>>(out, 3, w, t); }, 5);
    const double b4 = time_kernel([&] { k_bfly<4><<<blocks, threads>>>(out, 3, w, t); }, 5);
    const double b8 = time_kernel([&] { k_bfly<8><<<blocks, threads>>>(out, 3, w, t); }, 5);
    const double bh = time_kernel([&] { k_bfly<16><<<blocks, threads>>>(out, 3, w, t); }, 5);
    double s[5];
    s[0] = time_kernel([&] { k_stream<0><<<blocks, threads>>>(out, 3, 0.999); }, 5);
    s[1] = time_kernel([&] { k_stream<1><<<blocks, threads>>>(out, 3, 0.999); }, 5);
    s[2] = time_kernel([&] { k_stream<2><<<blocks, threads>>>(out, 3, 0.999); }, 5);
    s[3] = time_kernel([&] { k_stream<3><<<blocks, threads>>>(out, 3, 0.999); }, 5);
    s[4] = time_kernel([&] { k_stream<4><<<blocks, threads>>>(out, 3, 0.999); }, 5);
    printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_check_bad\": %llu, \"bfly_shoup_per_s\": %.6e, "
           "\"bfly_dfma1_per_s\": %.6e, \"bfly_dfma2_per_s\": %.6e, \"bfly_mixed_1of3_per_s\": %.6e, "
           "\"bfly_mixed_1of4_per_s\": %.6e, \"bfly_mixed_1of8_per_s\": %.6e, \"bfly_mixed_1of16_per_s\": %.6e, "
           "\"imad_per_s\": %.6e, \"imad_hi_per_s\": %.6e, "
           "\"imad_wide_per_s\": %.6e, \"dfma_per_s\": %.6e, \"dfma_plus_imad_pairs_per_s\": %.6e, \"err\": \"%s\"}\n",
           sms, clk, hbad, per / b0, per / b1, per / b2, per / b3, per / b4, per / b8, per / bh, per / s[0], per / s[1], per / s[2], per / s[3], per / s[4],
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
