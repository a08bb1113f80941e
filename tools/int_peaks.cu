// int_peaks.cu -- measured integer-pipe peaks on this GPU, the denominators
// of bench.py's "int_roofline" (MEASURED_PEAKS.json has only HBM and bf16).
//
//   butterfly : the NTT path's lazy DIF butterfly (Shoup multiply, p < 2^30)
//               on register-resident data, no memory traffic
//   imad      : dependent-free 32-bit IMAD stream
//   imad_hi   : IMAD.HI.U32 stream (with addend; r01 had a shift + xor beside it, which
//               made the loop ALU-bound at 25/clk/SM: the pipe itself does 31/clk/SM)
//   popc      : POPC + LOP3 (the 1-bit correlation inner op)
// Output: one JSON object on stdout.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o tools/int_peaks tools/int_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2509_19974_b200/csrc/qx_common.cuh"

using namespace qx;

constexpr int ITERS = 4096;
constexpr int CH = 16;  // independent chains per thread

__global__ void k_bfly(uint32_t* out, uint32_t seed, uint2 w)
{
    ModP m{1012924417u, 2u * 1012924417u, 0};
    uint32_t a[CH], b[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        a[i] = (seed * (threadIdx.x + 7 * i)) % m.p;
        b[i] = (seed * (threadIdx.x + 3 * i + 1)) % m.p;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) bfly_dif(a[i], b[i], w, m);
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s ^= a[i] ^ b[i];
    if (s == 0x12345678u) out[threadIdx.x] = s;
}

__global__ void k_imad(uint32_t* out, uint32_t seed)
{
    uint32_t a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = seed + threadIdx.x * i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = a[i] * 0x9E3779B1u + seed;
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s ^= a[i];
    if (s == 0x12345678u) out[threadIdx.x] = s;
}

__global__ void k_imadhi(uint32_t* out, uint32_t seed)
{
    uint32_t a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = seed + threadIdx.x * i + 1;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = __umulhi(a[i], 0x9E3779B1u) + seed;  // one IMAD.HI.U32, nothing else
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s ^= a[i];
    if (s == 0x12345678u) out[threadIdx.x] = s;
}

__global__ void k_popc(uint32_t* out, uint32_t seed)
{
    uint32_t a[CH], c[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        a[i] = seed * (threadIdx.x + i);
        c[i] = 0;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) c[i] += __popc(a[i] ^ (seed + it));
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s ^= c[i];
    if (s == 0x12345678u) out[threadIdx.x] = s;
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

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 4096);
    const int blocks = sms * 8, threads = 256;
    const double per_launch = (double)blocks * threads * ITERS * CH;
    uint2 w = make_uint2(123456789u, (uint32_t)(((uint64_t)123456789u << 32) / 1012924417u));
    double tb = time_kernel([&] { k_bfly<<<blocks, threads>>>(out, 3, w); }, 5);
    double ti = time_kernel([&] { k_imad<<<blocks, threads>>>(out, 3); }, 5);
    double th = time_kernel([&] { k_imadhi<<<blocks, threads>>>(out, 3); }, 5);
    double tp = time_kernel([&] { k_popc<<<blocks, threads>>>(out, 3); }, 5);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"sms\": %d, \"clock_khz\": %d, \"butterflies_per_s\": %.6e, \"imad_per_s\": %.6e, "
           "\"imad_hi_per_s\": %.6e, \"popc_per_s\": %.6e, \"err\": \"%s\"}\n",
           sms, clk, per_launch / tb, per_launch / ti, per_launch / th, per_launch / tp,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
