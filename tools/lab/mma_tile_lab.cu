// mma_tile_lab.cu — the matcher's MMA issue pattern in isolation (not part of the product):
// per "tile" 16 kind::i8 MMAs (M = N = 128, K = 32, SW128 K-major operands, K stepping through
// 4 atoms) into one of two accumulators, then 0 / 1 / 2 tcgen05.commit; cycles per tile.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <int COMMITS, int ATMEM, int RT = 0>
__global__ void k(int tiles, unsigned long long* cyc, int atoms = 4) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tb;
    for (int i = threadIdx.x; i < 131072; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[1])));
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
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t a0 = desc_sw128(sa(sm)), b0 = desc_sw128(sa(sm) + 65536);
        uint32_t abase = sa(sm), bbase = sa(sm) + 65536;
        asm volatile("" : "+r"(abase), "+r"(bbase));
        long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            const uint32_t d = tb + (uint32_t)((t & 1) * 128);
            for (int a = 0; a < (RT ? atoms : 4); ++a)
#pragma unroll
                for (int k32 = 0; k32 < 4; ++k32) {
                    const int ks = 4 * a + k32;
                    const uint64_t off = (uint64_t)((a * 16384 + k32 * 32) >> 4);
                    if (RT)
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                                     "l"(desc_sw128(abase + a * 16384 + k32 * 32)),
                                     "l"(desc_sw128(bbase + a * 16384 + k32 * 32)), "r"(idesc), "r"(ks)
                                     : "memory");
                    else if (ATMEM)
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                                     "r"(tb + 256u + (uint32_t)(ks * 8)), "l"(b0 + off), "r"(idesc), "r"(ks)
                                     : "memory");
                    else
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                                     "l"(a0 + off), "l"(b0 + off), "r"(idesc), "r"(ks)
                                     : "memory");
                }
            if (COMMITS >= 1)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar[0])) : "memory");
            if (COMMITS >= 2)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar[1])) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar[1])) : "memory");
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
template <int C, int AT, int RT = 0>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(k<C, AT, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024);
    const int tiles = 256;
    k<C, AT, RT><<<148, 128, 131072 + 1024>>>(tiles, d, 4);
    k<C, AT, RT><<<148, 128, 131072 + 1024>>>(tiles, d, 4);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("%-34s %.0f cycles per tile (ideal 1024)  %s\n", name, (double)h[0] / tiles, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<0, 0>("A smem, no commits");
    run<2, 0>("A smem, 2 commits per tile");
    run<0, 1>("A TMEM, no commits");
    run<2, 1>("A TMEM, 2 commits per tile");
    run<1, 0>("A smem, 1 commit per tile");
    run<1, 1>("A TMEM, 1 commit per tile");
    run<2, 0, 1>("A smem runtime descs, 2 commits");
    run<0, 0, 1>("A smem runtime descs, no commits");
    return 0;
}
