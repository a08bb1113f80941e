// tmem_st_rate.cu -- tcgen05.st / tcgen05.ld throughput probe: one warp per
// TMEM lane quarter (4 warps) or one warp, 32x32b.x32 (4 KB per warp-op),
// back to back; bytes per cycle per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_st_rate tools/tmem_st_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_rate(long long* out, int iters, int nwarps, int mode)
{
    __shared__ uint32_t tbase;
    const int w = threadIdx.x >> 5;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 33 + i;
    long long t0 = clock64();
    if (w < nwarps) {
        const uint32_t lb = tbase + ((uint32_t)((w & 3) * 32) << 16);
        for (int it = 0; it < iters; ++it) {
            const uint32_t a = lb + (uint32_t)((it & 7) * 32);
            if (mode == 0)
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
                    "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                    "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                    "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                    "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
            else {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
                    "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(a));
                asm volatile("tcgen05.wait::ld.sync.aligned;");
            }
        }
        if (mode == 0) asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x == 0) out[0] = clock64() - t0;
    if (mode == 1 && threadIdx.x < 32) out[1] = v[0] + v[31];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main()
{
    long long* d;
    cudaMalloc(&d, 16);
    for (int mode = 0; mode < 2; ++mode)
        for (int nw : {1, 4, 8}) {
            const int iters = 2048;
            k_rate<<<1, 256>>>(d, iters, nw, mode);
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
            const double bytes = (double)iters * nw * 4096;
            printf("{\"op\": \"%s 32x32b.x32\", \"warps\": %d, \"cycles\": %lld, \"bytes_per_clk_sm\": %.1f}\n",
                   mode ? "tcgen05.ld (+wait each)" : "tcgen05.st", nw, c, bytes / c);
        }
    return 0;
}
