// tc_swz.cu -- does a swizzled K-major tcgen05 A operand act as a linear
// buffer under any 32-B-advanced start address?  Stores y[L] at the
// physical address swz(L) of a 1024-B-aligned buffer (SW32: bit 4 ^= bit 7,
// SW64: bits 4-5 ^= 7-8, SW128: bits 4-6 ^= 7-9), describes A with row
// pitch = swizzle width (SBO = 8 rows), multiplies by an identity B
// (N columns) and checks D[m][n] == y[start + pitch*m + n] for several starts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_swz tools/tc_swz.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// sm_100 shared-memory descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version 1 at 46,
// base offset [49,52), layout [61,64): 0 none, 2 SW128, 4 SW64, 6 SW32
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ uint32_t swz(uint32_t o, int bits)  // bits = 1 (SW32), 2 (SW64), 3 (SW128)
{
    const uint32_t mask = (1u << bits) - 1u;
    return o ^ (((o >> 7) & mask) << 4);
}

constexpr int M = 128;

template <int N, int BITS, int LAYOUT>
__global__ void k_swz(int* bad, int* checked, int start)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* A = sm;              // 16 KB: y bytes, swizzled
    unsigned char* B = sm + 16384;      // identity, no-swizzle K-major core matrices
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    constexpr int PITCH = 16 << BITS;   // 32 / 64 / 128
    for (int L = threadIdx.x; L < 16384; L += blockDim.x) A[swz((uint32_t)L, BITS)] = (unsigned char)((L * 7 + 3) & 0x3f);
    // B[n][k] = (k == n) for k < 32 (one K=32 MMA): core matrix (n/8, k/16) at
    // (n/8)*SBO + (k/16)*LBO, row n%8 at 16*(n%8); LBO = 16*N... use LBO = N*16, SBO = 128
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) B[i] = 0;
    __syncthreads();
    if (threadIdx.x < N) {
        const int n = threadIdx.x;
        if (n < 32) {
            const int k = n;
            B[(n / 8) * 128 + (k / 16) * (N * 16) + (n % 8) * 16 + (k % 16)] = 1;
        }
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (threadIdx.x == 0) {
        const uint64_t ad = desc(su32(A) + start, 16, 8 * PITCH, LAYOUT);
        const uint64_t bd = desc(su32(B), N * 16, 128, 0);
        asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;" ::"r"(tbase), "l"(ad), "l"(bd), "r"(idesc));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // 4 warps read lanes 32w..32w+31 = rows m, columns n < min(N, 32)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w < 4) {
        const int m = w * 32 + lane;
        for (int n0 = 0; n0 < N && n0 < 32; n0 += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tbase + ((uint32_t)(w * 32) << 16) + (uint32_t)n0));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int i = 0; i < 8; ++i) {
                const int n = n0 + i;
                const int L = start + PITCH * m + n;
                const int want = (L * 7 + 3) & 0x3f;
                atomicAdd(checked, 1);
                if ((int)v[i] != want) atomicAdd(bad, 1);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

template <int N, int BITS, int LAYOUT>
static void run(const char* name)
{
    int *d, h[2];
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k_swz<N, BITS, LAYOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int start : {0, 32, 64, 96, 128, 160, 224, 256, 288, 992, 1024, 1056, 2080}) {
        cudaMemset(d, 0, 8);
        k_swz<N, BITS, LAYOUT><<<1, 128, 32768>>>(d, d + 1, start);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"layout\": \"%s\", \"start\": %d, \"bad\": %d, \"checked\": %d, \"err\": \"%s\"}\n", name, start, h[0],
               h[1], cudaGetErrorString(e));
        if (e != cudaSuccess) break;
    }
    cudaFree(d);
}

int main()
{
    run<32, 1, 6>("SW32 pitch 32");
    run<64, 2, 4>("SW64 pitch 64");
    run<128, 3, 2>("SW128 pitch 128");
    return 0;
}
