// tc_shift.cu -- semantics probe for tcgen05.shift (UTCSHIFT): fill 128 lanes
// x 32 columns of TMEM with lane*1000 + column, shift once at column 0, read
// back, and print which (lane, column) cells moved where.  A sliding Hankel
// A operand (row a at K-step s+1 = row a+1 at step s) is one row shift per
// K-step if this moves a 256-bit (8-column) row block down one lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_shift tools/tc_shift.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_shift(uint32_t* out)
{
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t lb = tbase + ((uint32_t)(w * 32) << 16);
    const int row = w * 32 + lane;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = row * 1000 + c;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(lb),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (w == 0) {
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.shift.cta_group::1.down [%0];\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];\n}" ::"r"(tbase),
            "r"(su32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(su32(&bar)));
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(lb));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < 32; ++c) out[row * 32 + c] = v[c];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase));
}

int main()
{
    uint32_t* d;
    cudaMalloc(&d, 128 * 32 * 4);
    k_shift<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    static uint32_t h[128 * 32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(e));
    int moved = 0, cols_moved[32] = {0};
    for (int r = 0; r < 128; ++r)
        for (int c = 0; c < 32; ++c)
            if (h[r * 32 + c] != (uint32_t)(r * 1000 + c)) {
                ++moved;
                ++cols_moved[c];
            }
    printf("{\"cells_changed\": %d}\n", moved);
    printf("columns changed:");
    for (int c = 0; c < 32; ++c) printf(" %d", cols_moved[c]);
    printf("\nsample: ");
    for (int r : {0, 1, 2, 31, 32, 126, 127})
        printf("[lane %d: col0=%u col7=%u col8=%u] ", r, h[r * 32], h[r * 32 + 7], h[r * 32 + 8]);
    printf("\n");
    return 0;
}
