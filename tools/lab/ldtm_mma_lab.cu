// ldtm_mma_lab.cu — does reading TMEM (tcgen05.ld) slow down while the tensor core accumulates
// into another TMEM region? (not part of the product)  One CTA per SM: warp 8 lane 0 issues
// back-to-back kind::i8 MMAs (M = 128, N = 256, K = 32) into columns 0-255 when MMA = 1; warps
// 0-7 read columns 256-511 with tcgen05.ld (x32, or x16.pack::16b when P = 1) + wait::ld.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <int MMA, int P>
__global__ void __launch_bounds__(288, 1) k(int iters, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tb;
    __shared__ int done;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (threadIdx.x == 0) done = 0;
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 8) {
        if (MMA && lane == 0) {
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
            const uint64_t a0 = desc_sw128(sa(sm)), b0 = desc_sw128(sa(sm) + 16384);
            long n = 0;
            while (*(volatile int*)&done < 8) {
#pragma unroll
                for (int k32 = 0; k32 < 4; ++k32)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tb),
                                 "l"(a0 + (uint64_t)(k32 * 2)), "l"(b0 + (uint64_t)(k32 * 2)), "r"(idesc), "r"(k32)
                                 : "memory");
                ++n;
            }
            cyc[148 * 8 + blockIdx.x] = n;
        }
    } else {
        const uint32_t taddr = tb + 256u + (uint32_t)((warp & 3) * 32 << 16) + (uint32_t)((warp >> 2) * 128);
        uint32_t acc = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t v[32];
                if (P) {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                        : "r"(taddr + q * 32));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 16; ++c) acc += v[c];
                } else {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(taddr + q * 32));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int c = 0; c < 32; ++c) acc += v[c];
                }
            }
        }
        const long long t1 = clock64();
        if (lane == 0) {
            cyc[blockIdx.x * 8 + warp] = t1 - t0;
            atomicAdd(&done, 1);
        }
        if (acc == 0x12345678u) cyc[0] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
template <int MMA, int P>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 9 * 8);
    cudaMemset(d, 0, 148 * 9 * 8);
    cudaFuncSetAttribute(k<MMA, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    const int iters = 2000;
    k<MMA, P><<<148, 288, 65536 + 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148 * 9];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int w = 0; w < 8; ++w) s += (double)h[w];
    const double per_ld = s / 8 / (iters * 4.0);
    printf("%-28s %s: %.1f cycles per chunk (32 cols x 32 lanes) per warp; 8 warps -> %.0f B/cycle; MMA groups %llu\n", name,
           cudaGetErrorString(e), per_ld, 8 * 4096.0 / per_ld, h[148 * 8]);
}
int main() {
    run<0, 0>("ldtm x32, idle tensor core");
    run<1, 0>("ldtm x32, MMAs running");
    run<0, 1>("ldtm x16.pack16, idle");
    run<1, 1>("ldtm x16.pack16, MMAs running");
    return 0;
}
