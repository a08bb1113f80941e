// tc_fp4_2sm.cu -- the template-search window path on a CTA pair
// (tcgen05.mma.cta_group::2.kind::mxf4.block_scale, M = 256, N = 128, K = 64):
// CTA r of the cluster holds A rows 128r..128r+127, a pitch-128 (64-B SW64)
// Hankel of its own stream window, and template copies n = 64r..64r+63 of
// B; D rows of CTA r (in its own TMEM) are lags 128*(128r + a) + n.  Checks
// every one of the 32768 lags against a CPU correlation (codes -1..1 and
// -4..4) and times the chain with fresh operands (descriptors advancing
// along K, as in the kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_fp4_2sm tools/tc_fp4_2sm.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ uint32_t e2m1(int c)
{
    const int a = c < 0 ? -c : c;
    const uint32_t m = a == 0 ? 0u : a == 1 ? 2u : a == 2 ? 4u : a == 3 ? 5u : 6u;
    return m | (c < 0 ? 8u : 0u);
}

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

constexpr int NX = 4096;
constexpr int PITCH = 128;                       // samples per Hankel row (64 B, SW64)
constexpr int M = 256, N = 128, NH = 64;         // per CTA: 128 rows, 64 B rows
constexpr int KS = 64;
constexpr int NK = (NX + N - 1 + KS - 1) / KS;  // 66
constexpr int KTOT = NK * KS;
constexpr int LBO = NH * 16 + 16;               // 1040
constexpr int NCH = KTOT / 32;
constexpr int LAGS = M * N;                     // 32768
constexpr int YW = 128 * PITCH + KTOT;          // stream samples per CTA
constexpr int ABYTES = ((YW / 2 + 1023) / 1024) * 1024;
constexpr int NY = LAGS + KTOT;
constexpr int SMEM = ABYTES + NCH * LBO + 1024;

__global__ void __cluster_dims__(2, 1, 1) k_fp4_2sm(const int8_t* x, const int8_t* y, int* out, long long* cyc, int reps)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* A = sm;
    unsigned char* B = sm + ABYTES;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const uint32_t rank = cta_rank();
    const int8_t* yr = y + 128 * PITCH * rank;
    for (int i = threadIdx.x; i < ABYTES; i += blockDim.x) {
        const int j = 2 * i;
        const uint32_t lo = j < YW ? e2m1(yr[j]) : 0u, hi = j + 1 < YW ? e2m1(yr[j + 1]) : 0u;
        A[i ^ (((i >> 7) & 3) << 4)] = (unsigned char)(lo | (hi << 4));
    }
    for (int i = threadIdx.x; i < NCH * NH * 16; i += blockDim.x) {
        const int byte = i & 15, jr = (i >> 4) % NH, kc = (i >> 4) / NH;
        const int n = NH * (int)rank + jr;
        const int m0 = 32 * kc - n + 2 * byte;
        const uint32_t lo = (m0 >= 0 && m0 < NX) ? e2m1(x[m0]) : 0u;
        const uint32_t hi = (m0 + 1 >= 0 && m0 + 1 < NX) ? e2m1(x[m0 + 1]) : 0u;
        B[kc * LBO + (jr / 8) * 128 + (jr % 8) * 16 + byte] = (unsigned char)(lo | (hi << 4));
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t SF = 256;
    if (w < 4) {
        const uint32_t v = 0x7f7f7f7fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                tbase + ((uint32_t)(w * 32) << 16) + SF),
            "r"(v));
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                tbase + ((uint32_t)(w * 32) << 16) + SF + 16),
            "r"(v));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
    constexpr uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
    if (rank == 0 && w == 4) {
        const long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep)
            for (int s = 0; s < NK; ++s) {
                const uint64_t ad = desc(su32(A) + 32 * s, 16, 8 * 64, 4);
                const uint64_t bd = desc(su32(B) + 2 * LBO * s, LBO, 128, 0);
                const uint32_t acc = (rep > 0 || s > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n}" ::"r"(
                        tbase),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(tbase + SF));
            }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}"
            ::"r"(su32(&bar)), "h"((unsigned short)3));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
        if (lane == 0) *cyc = clock64() - t0;
    } else if (rank == 1 && threadIdx.x == 0) {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (w < 4) {
        const int a = w * 32 + lane;  // local row
        for (int c0 = 0; c0 < N; c0 += 16) {
            float v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                  "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
                : "r"(tbase + ((uint32_t)(w * 32) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int i = 0; i < 16; ++i) {
                const float f = v[i] / (float)reps;
                out[(128 * rank + a) * N + c0 + i] = (float)(int)f == f ? (int)f : INT32_MIN;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main()
{
    std::vector<int8_t> hx(NX), hy(NY);
    int8_t *dx, *dy;
    int* dout;
    long long* dcyc;
    cudaMalloc(&dx, NX);
    cudaMalloc(&dy, NY + 64);
    cudaMalloc(&dout, LAGS * 4);
    cudaMalloc(&dcyc, 8);
    cudaFuncSetAttribute(k_fp4_2sm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    std::vector<int> out(LAGS);
    srand(11);
    int fails = 0;
    for (int kind = 0; kind < 2; ++kind) {
        for (int i = 0; i < NX; ++i) hx[i] = kind == 0 ? (rand() % 3) - 1 : (rand() % 9) - 4;
        for (int i = 0; i < NY; ++i) hy[i] = kind == 0 ? (rand() % 3) - 1 : (rand() % 9) - 4;
        cudaMemcpy(dx, hx.data(), NX, cudaMemcpyHostToDevice);
        cudaMemcpy(dy, hy.data(), NY, cudaMemcpyHostToDevice);
        k_fp4_2sm<<<2, 160, SMEM>>>(dx, dy, dout, dcyc, 1);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("{\"kind\": %d, \"err\": \"%s\"}\n", kind, cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(out.data(), dout, LAGS * 4, cudaMemcpyDeviceToHost);
        int bad = 0, first = -1;
        for (int row = 0; row < M; ++row)
            for (int n = 0; n < N; ++n) {
                const int j = PITCH * row + n;
                long long c = 0;
                for (int m = 0; m < NX; ++m) c += hx[m] * hy[m + j];
                if (out[row * N + n] != c) {
                    if (first < 0) first = j;
                    ++bad;
                }
            }
        printf("{\"codes\": \"%s\", \"lags\": %d, \"bad\": %d, \"first_bad\": %d}\n", kind == 0 ? "-1..1" : "-4..4", LAGS,
               bad, first);
        fails += bad;
    }
    for (int reps : {1, 16}) {
        k_fp4_2sm<<<2, 160, SMEM>>>(dx, dy, dout, dcyc, reps);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
        printf("{\"timing\": \"2-SM M256 N128 K64 mxf4, fresh operands\", \"reps\": %d, \"cycles_per_mma\": %.2f, "
               "\"lags_x_samples_per_clk_per_sm\": %.0f}\n",
               reps, (double)c / (reps * NK), 256.0 * 128 * 64 / ((double)c / (reps * NK)) / 2);
    }
    return fails ? 2 : 0;
}
