// mma_rate_lab.cu — tcgen05 kind::i8 issue rate for the column-prefix MMA shapes (not part of
// the product): M = 128, K = 32, N in {64, 128, 256}, A K-major (no swizzle), B MN-major SW32.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
template <int N, int BMAJ>
__global__ void k(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = (uint8_t)i;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | ((uint32_t)BMAJ << 16) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t ad = desc(sa(sm), 128, 256, 0);
        const uint64_t bd = BMAJ ? desc(sa(sm) + 16384, 1024, 256, 6) : desc(sa(sm) + 16384, 128, 256, 0);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tb + (uint32_t)((it & 1) * 256)),
                "l"(ad), "l"(bd), "r"(idesc), "r"(it & 3)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
template <int N, int BMAJ>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(k<N, BMAJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    const int iters = 4096;
    k<N, BMAJ><<<148, 128, 65536 + 1024>>>(iters, d);
    k<N, BMAJ><<<148, 128, 65536 + 1024>>>(iters, d);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const double c = (double)h[0] / iters;
    printf("%-28s N=%3d: %.1f cycles per MMA, %.0f MAC/cycle  (%s)\n", name, N, c, 128.0 * N * 32 / c,
           cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<64, 1>("B MN-major SW32");
    run<128, 1>("B MN-major SW32");
    run<256, 1>("B MN-major SW32");
    run<64, 0>("B K-major none");
    run<256, 0>("B K-major none");
    return 0;
}
