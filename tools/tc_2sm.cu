// tc_2sm.cu -- operand split of tcgen05.mma.cta_group::2.kind::i8 (2-SM
// MMA, M = 256, N = 64) as the shared-template window path would use it:
// CTA r of the pair holds A rows 128r..128r+127 (a pitch-64 SW64 Hankel of
// its own y_r) and B rows 32r..32r+31; expected D rows of CTA r (in its own
// TMEM) = y_r[64 m' + (n mod 32)] with B_r[n'][k] = (k == n').
// Also times the MMA (cycles per 2-SM instruction) for N = 64 and 128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_2sm tools/tc_2sm.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ uint32_t swz64(uint32_t o) { return o ^ (((o >> 7) & 3u) << 4); }

__device__ __forceinline__ uint32_t cta_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) k_2sm(int* bad, int* checked, long long* cycles, int reps)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* A = sm;          // 24 KB: y_r bytes, SW64-swizzled
    unsigned char* B = sm + 24576;  // N/2 rows, no-swizzle K-major core matrices
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const uint32_t rank = cta_rank();
    constexpr int NH = N / 2;
    for (int L = threadIdx.x; L < 24576; L += blockDim.x)
        A[swz64((uint32_t)L)] = (unsigned char)((L * 5 + 11 * (int)rank + 1) & 0x3f);
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) B[i] = 0;
    __syncthreads();
    if (threadIdx.x < NH && threadIdx.x < 32) {
        const int n = threadIdx.x, k = n;  // local row n' = k
        B[(n / 8) * 128 + (k / 16) * (NH * 16) + (n % 8) * 16 + (k % 16)] = 1;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((256u >> 4) << 24);
    if (rank == 0 && threadIdx.x < 32) {
        const uint64_t ad = desc(su32(A), 16, 8 * 64, 4);  // SW64, rows 64 B apart
        const uint64_t bd = desc(su32(B), NH * 16, 128, 0);
        const long long t0 = clock64();
        for (int i = 0; i < reps; ++i) {
            asm volatile(
                "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tbase),
                "l"(ad), "l"(bd), "r"(idesc), "r"(0u));  // overwrite: D = the last MMA's product
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}"
            ::"r"(su32(&bar)), "h"((unsigned short)3));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
        if (threadIdx.x == 0) *cycles = clock64() - t0;
    } else if (rank == 1 && threadIdx.x == 0) {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int s0 = 0;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = w * 32 + lane;
    for (int n0 = 0; n0 < N; n0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tbase + ((uint32_t)(w * 32) << 16) + (uint32_t)n0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int i = 0; i < 8; ++i) {
            const int n = n0 + i;
            if ((n % NH) >= 32) continue;  // B rows beyond K = 32 are zero
            const int L = s0 + 64 * m + (n % NH);
            const int want = (L * 5 + 11 * (int)rank + 1) & 0x3f;
            atomicAdd(checked, 1);
            if ((int)v[i] != want) atomicAdd(bad, 1);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

template <int N>
static void run(int reps)
{
    int *d, h[2];
    long long* c, hc;
    cudaMalloc(&d, 8);
    cudaMalloc(&c, 8);
    cudaMemset(d, 0, 8);
    cudaFuncSetAttribute(k_2sm<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    k_2sm<N><<<2, 128, 32768>>>(d, d + 1, c, reps);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("{\"N\": %d, \"reps\": %d, \"bad\": %d, \"checked\": %d, \"cycles_per_mma\": %.2f, \"err\": \"%s\"}\n", N,
           reps, h[0], h[1], (double)hc / reps, cudaGetErrorString(e));
    cudaFree(d);
    cudaFree(c);
}

int main()
{
    run<64>(1);
    run<64>(8);
    run<64>(4096);
    run<128>(1);
    run<128>(4096);
    return 0;
}
