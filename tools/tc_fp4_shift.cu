// tc_fp4_shift.cu -- a TMEM-resident sliding Hankel A operand for the fp4
// window MMA: per K-step the MMA thread issues the MMA on an 8-column A block,
// tcgen05.shift.down (row block up one lane inside each 32-lane quarter: row a
// at step s+1 = row a+1 at step s) and four tcgen05.cp.4x256b that refill
// lanes 28-31 of each quarter from the SW32 stream buffer (4 x 32 B), all
// pipelined tensor ops of one thread.  Checks exactness against a CPU
// correlation and times the chain (cycles per K-step).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_fp4_shift tools/tc_fp4_shift.cu
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

constexpr int NX = 4096;
constexpr int M = 128, N = 64, KS = 64;
constexpr int NK = (NX + N - 1 + KS - 1) / KS;  // 65
constexpr int KTOT = NK * KS;
constexpr int LBO = 1040;
constexpr int NCH = KTOT / 32;
constexpr int LAGS = M * N;
constexpr int NY = LAGS + KTOT;
constexpr int ABYTES = 8192;
constexpr int ACOL = 128, SF = 256;
constexpr int SMEM = ABYTES + NCH * LBO + 1024;

__global__ void k_shift(const int8_t* x, const int8_t* y, int* out, long long* cyc, int reps)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* A = sm;  // stream nibbles, SW32 (rows 32 B apart)
    unsigned char* B = sm + ABYTES;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < ABYTES; i += blockDim.x) {
        const int j = 2 * i;
        const uint32_t lo = j < NY ? e2m1(y[j]) : 0u, hi = j + 1 < NY ? e2m1(y[j + 1]) : 0u;
        A[i ^ (((i >> 7) & 1) << 4)] = (unsigned char)(lo | (hi << 4));
    }
    for (int i = threadIdx.x; i < NCH * N * 16; i += blockDim.x) {
        const int byte = i & 15, r = (i >> 4) % N, kc = (i >> 4) / N;
        const int m0 = 32 * kc - r + 2 * byte;
        const uint32_t lo = (m0 >= 0 && m0 < NX) ? e2m1(x[m0]) : 0u;
        const uint32_t hi = (m0 + 1 >= 0 && m0 + 1 < NX) ? e2m1(x[m0 + 1]) : 0u;
        B[kc * LBO + (r / 8) * 128 + (r % 8) * 16 + byte] = (unsigned char)(lo | (hi << 4));
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
    if (w < 4) {
        const uint32_t lb = tbase + ((uint32_t)(w * 32) << 16);
        const uint32_t v = 0x7f7f7f7fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(lb + SF),
            "r"(v));
        // A block = Hankel rows at step 0: row a = stream bytes [32a, +32) (unswizzled words)
        const int a = w * 32 + lane;
        uint32_t q[8];
        for (int i = 0; i < 8; ++i) {
            const int wi = 8 * a + i, byte = 4 * wi;
            q[i] = *reinterpret_cast<const uint32_t*>(A + (byte ^ (((byte >> 7) & 1) << 4)));
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lb + ACOL),
                     "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    constexpr uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
    if (w == 4) {
        const long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep)
            for (int s = 0; s < NK; ++s) {
                const uint64_t bd = desc(su32(B) + 2 * LBO * s, LBO, 128, 0);
                const uint32_t acc = (rep > 0 || s > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n}" ::"r"(
                        tbase),
                    "r"(tbase + ACOL), "l"(bd), "r"(idesc), "r"(acc), "r"(tbase + SF));
                if (s + 1 < NK) {
                    // rows 32q + 28 .. 32q + 31 at step s + 1 = stream rows 32q + 29 + s .. (+3): 128 B
                    uint64_t d[4];
                    for (int qq = 0; qq < 4; ++qq) d[qq] = desc(su32(A) + 32 * (32 * qq + 28 + s + 1), 16, 256, 6);
                    asm volatile(
                        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                        "@e tcgen05.shift.cta_group::1.down [%0];\n\t"
                        "@e tcgen05.cp.cta_group::1.4x256b [%1], %5;\n\t"
                        "@e tcgen05.cp.cta_group::1.4x256b [%2], %6;\n\t"
                        "@e tcgen05.cp.cta_group::1.4x256b [%3], %7;\n\t"
                        "@e tcgen05.cp.cta_group::1.4x256b [%4], %8;\n}" ::"r"(tbase + ACOL),
                        "r"(tbase + ACOL + (28u << 16)), "r"(tbase + ACOL + (60u << 16)), "r"(tbase + ACOL + (92u << 16)),
                        "r"(tbase + ACOL + (124u << 16)), "l"(d[0]), "l"(d[1]), "l"(d[2]), "l"(d[3]));
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
            for (int i = 0; i < 16; ++i) out[a * N + c0 + i] = (float)(int)v[i] == v[i] ? (int)v[i] : INT32_MIN;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
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
    cudaFuncSetAttribute(k_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    std::vector<int> out(LAGS);
    srand(9);
    for (int i = 0; i < NX; ++i) hx[i] = (rand() % 3) - 1;
    for (int i = 0; i < NY; ++i) hy[i] = (rand() % 3) - 1;
    cudaMemcpy(dx, hx.data(), NX, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, hy.data(), NY, cudaMemcpyHostToDevice);
    k_shift<<<1, 160, SMEM>>>(dx, dy, dout, dcyc, 1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("{\"err\": \"%s\"}\n", cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(out.data(), dout, LAGS * 4, cudaMemcpyDeviceToHost);
    int bad = 0, first = -1, rowbad[128] = {0};
    for (int a = 0; a < M; ++a)
        for (int r = 0; r < N; ++r) {
            const int j = 64 * a + r;
            long long c = 0;
            for (int m = 0; m < NX; ++m) c += hx[m] * hy[m + j];
            if (out[a * N + r] != c) {
                if (first < 0) first = j;
                ++bad;
                ++rowbad[a];
            }
        }
    printf("{\"A\": \"tmem, shift + cp per K-step\", \"lags\": %d, \"bad\": %d, \"first_bad\": %d}\n", LAGS, bad, first);
    printf("bad rows:");
    for (int a = 0; a < 128; ++a)
        if (rowbad[a]) printf(" %d", a);
    printf("\n");
    long long c;
    cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"timing\": \"one chain of %d K-steps (mma + shift + 4 cp)\", \"cycles_per_step\": %.2f}\n", NK,
           (double)c / NK);
    return bad ? 2 : 0;
}
