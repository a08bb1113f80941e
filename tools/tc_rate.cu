// tc_rate.cu -- measured tcgen05.mma kind::i8 throughput per SM for the
// operand shapes the window path can use (one CTA per SM, one issuing
// thread, operands resident in shared memory).  Prints cycles per MMA and
// int8 MACs per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_rate tools/tc_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

template <int M, int N, int NACC, bool TS, bool WARP = false>
__global__ void k_rate(long long* out, int iters, uint32_t albo, uint32_t asbo)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (WARP && threadIdx.x < 32) {
        const uint32_t a = su32(sm), b = su32(sm + 64 * 1024);
        const long long t0 = clock64();
        const uint64_t bd = desc(b, 256, 128);
        for (int i = 0; i < iters; i += 4) {
            const uint64_t ad = desc(a, albo, asbo) + (uint64_t)((i & 63) * 2);
            asm volatile(
                "{\n\t.reg .pred e, p;\n\t"
                "elect.sync _|e, 0xffffffff;\n\t"
                "setp.ne.b32 p, %3, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %4, p;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %5, %2, %4, 1;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %6, %2, %4, 1;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %7, %2, %4, 1;\n\t"
                "}" ::"r"(tbase), "l"(ad), "l"(bd), "r"((uint32_t)(i > 0)), "n"(idesc),
                "l"(ad + 2), "l"(ad + 4), "l"(ad + 6));
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    }
    if (!WARP && threadIdx.x == 0) {
        const uint32_t a = su32(sm), b = su32(sm + 64 * 1024);
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += 64) {
            uint64_t ad = desc(a, albo, asbo), bd = desc(b, 256, 128);
#pragma unroll 4
            for (int kk = 0; kk < 64; ++kk) {
                const uint32_t d = tbase + (uint32_t)((kk % NACC) * N);
                if (TS) {
                    const uint32_t ta = tbase + 256u + (uint32_t)((kk & 15) * 8);
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                        "r"(ta), "l"(bd), "n"(idesc), "r"((uint32_t)(i + kk >= NACC)));
                } else {
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                        "l"(ad), "l"(bd), "n"(idesc), "r"((uint32_t)(i + kk >= NACC)));
                }
                ad += 2;
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int M, int N, int NACC, bool TS = false, bool WARP = false>
static void run(const char* name, uint32_t albo, uint32_t asbo)
{
    long long* d;
    cudaMalloc(&d, 148 * 8);
    const int iters = 8192;
    cudaFuncSetAttribute(k_rate<M, N, NACC, TS, WARP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    k_rate<M, N, NACC, TS, WARP><<<148, 128, 96 * 1024>>>(d, iters, albo, asbo);
    cudaDeviceSynchronize();
    k_rate<M, N, NACC, TS, WARP><<<148, 128, 96 * 1024>>>(d, iters, albo, asbo);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("{\"nacc\": %d, \"a_in_tmem\": %d, \"warp_issue\": %d, \"shape\": \"%s\", \"cycles_per_mma\": %.2f, \"macs_per_clk_sm\": %.1f, \"err\": \"%s\"}\n", NACC, (int)TS, (int)WARP, name,
           avg / iters, (double)M * N * 32 / (avg / iters), cudaGetErrorString(e));
    cudaFree(d);
}

int main()
{
    run<128, 16, 1, false, true>("M128 N16 A-overlap", 16, 128);
    run<128, 32, 1, false, true>("M128 N32 A-overlap", 16, 128);
    run<128, 64, 1, false, true>("M128 N64 A-overlap", 16, 128);
    run<128, 128, 1, false, true>("M128 N128 A-overlap", 16, 128);
    run<64, 8, 1, false, true>("M64 N8 A-overlap", 16, 128);
    run<64, 16, 1, false, true>("M64 N16 A-overlap", 16, 128);
    run<64, 24, 1, false, true>("M64 N24 A-overlap", 16, 128);
    run<64, 32, 1, false, true>("M64 N32 A-overlap", 16, 128);
    run<64, 64, 1, false, true>("M64 N64 A-overlap", 16, 128);
    run<64, 128, 1, false, true>("M64 N128 A-overlap", 16, 128);
    run<128, 16, 1>("M128 N16 A-overlap (1-thread issue)", 16, 128);
    run<64, 24, 1>("M64 N24 A-overlap (1-thread issue)", 16, 128);
    return 0;
}
