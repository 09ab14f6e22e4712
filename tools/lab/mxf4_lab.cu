// mxf4_lab.cu — can the matcher's +-1 similarity run as tcgen05 kind::mxf4 (packed e2m1, block
// scales all 1.0)? (not part of the product)  One CTA: A, B = 128 rows x 256 e2m1 values
// (+1 = 0x2, -1 = 0xA) in one SWIZZLE_128B atom each, 4 MMAs (M = N = 128, K = 64), scale
// factors: 64 TMEM columns filled with 0x7F (ue8m0 1.0); D (f32) compared with the integer dot
// products.  Also times back-to-back MMAs against kind::i8 on the same shape.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__global__ void k(const uint8_t* A, const uint8_t* B, float* D, long long* cyc, int reps, int i8) {
    __shared__ __align__(1024) uint8_t sA[16384];
    __shared__ __align__(1024) uint8_t sB[16384];
    __shared__ uint32_t tb;
    __shared__ uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < 16384; i += blockDim.x) {  // row-major 128 x 128 bytes -> SW128
        const int r = i / 128, c = i % 128;
        const int dst = r * 128 + (((c >> 4) ^ (r & 7)) << 4) + (c & 15);
        sA[dst] = A[i];
        sB[dst] = B[i];
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tb;
    // scale factors: columns 256..383 of every lane = 0x7F7F7F7F
    {
        const uint32_t o = 0x7F7F7F7Fu;
        const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16);
        for (int c = 256; c < 384; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(base + c), "r"(o));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (t == 0) {
        const uint32_t idesc_f4 = (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
        const uint32_t idesc_i8 = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t a0 = desc_sw128(sa(sA)), b0 = desc_sw128(sa(sB));
        long long c0 = clock64();
        for (int r = 0; r < reps; ++r)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (!i8)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(tmem),
                                 "l"(a0 + (uint64_t)(kk * 2)), "l"(b0 + (uint64_t)(kk * 2)), "r"(idesc_f4), "r"(kk),
                                 "r"(tmem + 256u), "r"(tmem + 320u)
                                 : "memory");
                else
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                 "l"(a0 + (uint64_t)(kk * 2)), "l"(b0 + (uint64_t)(kk * 2)), "r"(idesc_i8), "r"(kk)
                                 : "memory");
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
        cyc[0] = clock64() - c0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
        for (int c = 0; c < 128; c += 32) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * 128 + c + j] = i8 ? (float)(int)v[j] : __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
    const int M = 128, Kf4 = 256;
    static int8_t a[128][256], b[128][256];
    srand(7);
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < Kf4; ++j) {
            a[i][j] = (rand() & 1) ? 1 : -1;
            b[i][j] = (rand() & 1) ? 1 : -1;
        }
    static uint8_t ha[16384], hb[16384], ha8[16384], hb8[16384];
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < 128; ++j) {  // fp4: element 2j in the low nibble
            auto e = [](int v) { return v > 0 ? 0x2 : 0xA; };
            ha[i * 128 + j] = (uint8_t)(e(a[i][2 * j]) | (e(a[i][2 * j + 1]) << 4));
            hb[i * 128 + j] = (uint8_t)(e(b[i][2 * j]) | (e(b[i][2 * j + 1]) << 4));
            ha8[i * 128 + j] = (uint8_t)a[i][j];  // int8: first 128 values
            hb8[i * 128 + j] = (uint8_t)b[i][j];
        }
    uint8_t *dA, *dB;
    float* dD;
    long long* dc;
    cudaMalloc(&dA, 16384);
    cudaMalloc(&dB, 16384);
    cudaMalloc(&dD, 128 * 128 * 4);
    cudaMalloc(&dc, 8);
    static float hD[128 * 128];
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemcpy(dA, mode ? ha8 : ha, 16384, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, mode ? hb8 : hb, 16384, cudaMemcpyHostToDevice);
        k<<<1, 256>>>(dA, dB, dD, dc, 1, mode);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
        int bad = 0;
        const int KK = mode ? 128 : 256;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) {
                int s = 0;
                for (int q = 0; q < KK; ++q) s += a[i][q] * b[j][q];
                if (hD[i * 128 + j] != (float)s) {
                    if (bad < 3) printf("  mismatch [%d][%d]: %f vs %d\n", i, j, hD[i * 128 + j], s);
                    ++bad;
                }
            }
        long long c;
        k<<<1, 256>>>(dA, dB, dD, dc, 1000, mode);
        cudaDeviceSynchronize();
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("%s: %s, %d mismatches of %d; %.1f cycles per MMA (K = %d per MMA)\n", mode ? "kind::i8" : "kind::mxf4",
               cudaGetErrorString(e), bad, M * M, c / 4000.0, mode ? 32 : 64);
    }
    return 0;
}
