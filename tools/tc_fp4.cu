// tc_fp4.cu -- can the template-search window path run on packed-fp4
// tensor cores (tcgen05.mma kind::mxf4.block_scale, e2m1 x e2m1 -> f32,
// every ue8m0 scale = 2^0) and stay bit-exact?
//
// Codes of the k <= 4 quantisers (-4..4) are exact e2m1 values, products are
// integers and every partial sum of a 4096-sample template is an integer
// below 2^24, so an exact f32 accumulation gives the integer correlation.
// This checks that on the window-path geometry:
//   A = Hankel rows of the stream codes, 64 samples (32 B) apart, read
//       through a SWIZZLE_32B K-major descriptor from a linear nibble buffer;
//   B = 64 shifted copies of the template (no swizzle, K-chunk stride 1040 B);
//   D[a][r] = c[64a + r] for 8192 lags, K = 64 samples per MMA,
// against a CPU correlation (random codes in {-1,0,1} and in -4..4, plus the
// all-ones worst case), and times the MMA chain (cycles per instruction).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_fp4 tools/tc_fp4.cu
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

__device__ __forceinline__ uint32_t e2m1(int c)  // exact for |c| <= 4
{
    const int a = c < 0 ? -c : c;
    const uint32_t m = a == 0 ? 0u : a == 1 ? 2u : a == 2 ? 4u : a == 3 ? 5u : 6u;
    return m | (c < 0 ? 8u : 0u);
}

constexpr int NX = 4096;            // template samples
constexpr int PITCH = 64;           // Hankel row pitch (samples) = number of shifts N
constexpr int M = 128, N = 64;
constexpr int KS = 64;              // samples per MMA
constexpr int NK = (NX + PITCH - 1 + KS - 1) / KS;  // 65
constexpr int KTOT = NK * KS;       // 4160
constexpr int LBO = 1040;           // B K-chunk (32 samples, 16 B) stride
constexpr int NCH = KTOT / 32;      // 130 chunks
constexpr int LAGS = M * N;         // 8192
constexpr int NY = LAGS + KTOT;     // stream codes needed
constexpr int ABYTES = 8192;        // >= NY / 2, 1024-aligned
constexpr int SMEM = ABYTES + NCH * LBO + 1024;

__global__ void k_fp4(const int8_t* x, const int8_t* y, int* out, long long* cyc, int reps, int nibble_hi_first)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* A = sm;
    unsigned char* B = sm + ABYTES;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int sh0 = nibble_hi_first ? 4 : 0, sh1 = 4 - sh0;
    // A: byte i holds stream samples 2i, 2i+1, stored at swz32(i)
    for (int i = threadIdx.x; i < ABYTES; i += blockDim.x) {
        const int j = 2 * i;
        const uint32_t lo = j < NY ? e2m1(y[j]) : 0u, hi = j + 1 < NY ? e2m1(y[j + 1]) : 0u;
        A[i ^ (((i >> 7) & 1) << 4)] = (unsigned char)((lo << sh0) | (hi << sh1));
    }
    // B: chunk (kc, r) = x[32kc - r, +32) at kc*LBO + (r/8)*128 + (r%8)*16
    for (int i = threadIdx.x; i < NCH * N * 16; i += blockDim.x) {
        const int byte = i & 15, r = (i >> 4) % N, kc = (i >> 4) / N;
        const int m0 = 32 * kc - r + 2 * byte;
        const uint32_t lo = (m0 >= 0 && m0 < NX) ? e2m1(x[m0]) : 0u;
        const uint32_t hi = (m0 + 1 >= 0 && m0 + 1 < NX) ? e2m1(x[m0 + 1]) : 0u;
        B[kc * LBO + (r / 8) * 128 + (r % 8) * 16 + byte] = (unsigned char)((lo << sh0) | (hi << sh1));
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // scale factors: columns 256..287 of every lane = 0x7f bytes (2^0)
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
    asm volatile("tcgen05.fence::after_thread_sync;");
    // kind::mxf4: A = B = E2M1 (1), scale UE8M0 (bit 23), N >> 3 at 17, M >> 4 at 24, K64
    constexpr uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
    if (w == 4) {
        long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep) {
            for (int s = 0; s < NK; ++s) {
                const uint64_t ad = desc(su32(A) + 32 * s, 16, 256, 6);
                const uint64_t bd = desc(su32(B) + 2 * LBO * s, LBO, 128, 0);
                const uint32_t acc = (rep > 0 || s > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred e, p;\n\t"
                    "elect.sync _|e, 0xffffffff;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(
                        tbase),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(tbase + SF), "r"(tbase + SF + 8));
            }
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
        if (lane == 0) *cyc = clock64() - t0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (w < 4) {
        const int a = w * 32 + lane;
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
                out[a * N + c0 + i] = (float)(int)f == f ? (int)f : INT32_MIN;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

// peak-rate probe: the same chain at M128 x N (K64), operands from a zeroed
// buffer (content irrelevant for timing), B K-chunk stride 16*N bytes
template <int NN>
__global__ void k_fp4_rate(long long* cyc, int reps)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = 0x22;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    const int w = threadIdx.x >> 5;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t SF = 480;
    if (w < 4) {
        const uint32_t v = 0x7f7f7f7fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                tbase + ((uint32_t)(w * 32) << 16) + SF),
            "r"(v));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    constexpr uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
    if (w == 4) {
        const uint64_t ad = desc(su32(sm), 16, 256, 6);
        const uint64_t bd = desc(su32(sm + 8192), 16 * NN, 128, 0);
        long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep)
            asm volatile(
                "{\n\t.reg .pred e;\n\t"
                "elect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%4], 1;\n}" ::"r"(
                    tbase),
                "l"(ad), "l"(bd), "r"(idesc), "r"(tbase + SF));
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
        if ((threadIdx.x & 31) == 0) *cyc = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int NN>
static void rate(long long* dcyc)
{
    cudaFuncSetAttribute(k_fp4_rate<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    k_fp4_rate<NN><<<1, 160, 65536>>>(dcyc, 1024);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
    const double cpm = (double)c / 1024;
    printf("{\"timing\": \"M128 N%d K64 mxf4 (rate probe)\", \"cycles_per_mma\": %.2f, \"macs_per_clk_sm\": %.0f}\n", NN, cpm,
           128.0 * NN * 64 / cpm);
}

int main()
{
    std::vector<int8_t> hx(NX), hy(NY);
    int8_t *dx, *dy;
    int* dout;
    long long* dcyc;
    cudaMalloc(&dx, NX);
    cudaMalloc(&dy, NY);
    cudaMalloc(&dout, LAGS * 4);
    cudaMalloc(&dcyc, 8);
    cudaFuncSetAttribute(k_fp4, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    std::vector<int> out(LAGS);
    srand(7);
    int fails = 0;
    for (int order = 0; order < 2; ++order)
        for (int kind = 0; kind < 3; ++kind) {
            for (int i = 0; i < NX; ++i) hx[i] = kind == 2 ? 1 : kind == 0 ? (rand() % 3) - 1 : (rand() % 9) - 4;
            for (int i = 0; i < NY; ++i) hy[i] = kind == 2 ? 1 : kind == 0 ? (rand() % 3) - 1 : (rand() % 9) - 4;
            cudaMemcpy(dx, hx.data(), NX, cudaMemcpyHostToDevice);
            cudaMemcpy(dy, hy.data(), NY, cudaMemcpyHostToDevice);
            k_fp4<<<1, 160, SMEM>>>(dx, dy, dout, dcyc, 1, order);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("{\"order\": %d, \"kind\": %d, \"err\": \"%s\"}\n", order, kind, cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(out.data(), dout, LAGS * 4, cudaMemcpyDeviceToHost);
            int bad = 0, first = -1;
            for (int a = 0; a < M; ++a)
                for (int r = 0; r < N; ++r) {
                    const int j = 64 * a + r;  // lag: sum_m x[m] y[m + j]
                    long long c = 0;
                    for (int m = 0; m < NX; ++m) c += hx[m] * hy[m + j];
                    if (out[a * N + r] != c) {
                        if (first < 0) first = j;
                        ++bad;
                    }
                }
            printf("{\"order\": \"%s\", \"codes\": \"%s\", \"lags\": %d, \"bad\": %d, \"first_bad\": %d}\n",
                   order ? "hi-first" : "lo-first", kind == 0 ? "-1..1" : kind == 1 ? "-4..4" : "all ones", LAGS, bad,
                   first);
            if (order == 0) fails += bad;
        }
    // timing: reps chains of NK MMAs back to back
    for (int reps : {1, 8, 64}) {
        k_fp4<<<1, 160, SMEM>>>(dx, dy, dout, dcyc, reps, 0);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
        printf("{\"timing\": \"M128 N64 K64 mxf4\", \"reps\": %d, \"mmas\": %d, \"cycles_per_mma\": %.2f}\n", reps,
               reps * NK, (double)c / (reps * NK));
    }
    rate<32>(dcyc);
    rate<64>(dcyc);
    rate<128>(dcyc);
    rate<256>(dcyc);
    return fails ? 2 : 0;
}
