// ubench.cu — micro-benchmarks of the on-chip resources the BAD test phase can read from
// (not part of the product).  One CTA per SM, 16 warps; each reports SM-wide cycles per
// warp-instruction for:
//   lds32     LDS.32, lane-distinct conflict-free addresses
//   lds128b   LDS.128 broadcast (all lanes same address)
//   lds32b    LDS.32 broadcast
//   ldcu      uniform constant loads (LDCU.64) from a small param table
//   ldtm1/2/4 tcgen05.ld.32x32b.x{1,2,4} (TMEM -> registers), wait::ld every 8 loads
//   ldtm8/16/32 tcgen05.ld.32x32b.x{8,16,32}, wait::ld every 4/2/1 loads (64 B..128 B per lane
//             in flight); ldtm16+lds: each x16 load interleaved with 8 LDS.32 (shared pipe?)
//   sts32     STS.32 conflict-free
//   shfl      SHFL.UP width 8
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

struct Tab {
    uint32_t v[2048];
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(512, 1) ub(uint32_t* out, int iters, const __grid_constant__ Tab tab, unsigned long long* cyc) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ uint32_t tmem_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16384; i += 512) sm[i] = i * 2654435761u;
    constexpr bool kTm = (MODE >= 4 && MODE <= 6) || MODE >= 9;
    if (kTm) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if (kTm) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t acc = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // LDS.32 lane-distinct
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += sm[((it * 37 + k * 131) & 511) * 32 + lane];
        } else if (MODE == 1) {  // LDS.128 broadcast
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint4 q = reinterpret_cast<const uint4*>(sm)[(it * 37 + k * 131) & 1023];
                acc += q.x ^ q.y ^ q.z ^ q.w;
            }
        } else if (MODE == 2) {  // LDS.32 broadcast
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += sm[(it * 37 + k * 131) & 4095];
        } else if (MODE == 3) {  // LDCU (uniform index)
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint2 q = reinterpret_cast<const uint2*>(tab.v)[(it * 37 + k * 131) & 255];
                acc += q.x ^ q.y;
            }
        } else if (MODE >= 4 && MODE <= 6) {  // LDTM
            const uint32_t ta = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
#pragma unroll
            for (int k = 0; k < 32; k += 8) {
                uint32_t r[8][4];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t col = ((it * 37 + (k + q) * 131) & 127) * 4;
                    if (MODE == 4)
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[q][0]) : "r"(ta + col));
                    else if (MODE == 5)
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                                     : "=r"(r[q][0]), "=r"(r[q][1])
                                     : "r"(ta + col));
                    else
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(r[q][0]), "=r"(r[q][1]), "=r"(r[q][2]), "=r"(r[q][3])
                                     : "r"(ta + col));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < 8; ++q) acc += r[q][0] + (MODE >= 5 ? r[q][1] : 0) + (MODE == 6 ? r[q][2] ^ r[q][3] : 0);
            }
        } else if (MODE >= 9) {  // LDTM x8 / x16 / x32 (+ LDS)
            const uint32_t ta = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
            constexpr int X = MODE == 9 ? 8 : MODE == 11 ? 32 : 16;
            constexpr int F = 64 / X;  // loads in flight
#pragma unroll
            for (int k = 0; k < 32; k += F) {
                uint32_t r[F][X];
#pragma unroll
                for (int q = 0; q < F; ++q) {
                    constexpr int XC = MODE == 13 ? 32 : X;  // columns per load
                    const uint32_t col = ((it * 37 + (k + q) * 131) & (512 / XC - 1)) * XC;
                    if (X == 8)
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                     : "=r"(r[q][0]), "=r"(r[q][1 % X]), "=r"(r[q][2 % X]), "=r"(r[q][3 % X]),
                                       "=r"(r[q][4 % X]), "=r"(r[q][5 % X]), "=r"(r[q][6 % X]), "=r"(r[q][7 % X])
                                     : "r"(ta + col));
                    else if (X == 16 && MODE == 13)  // 32 columns packed 2 x 16 bit per register
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                            : "=r"(r[q][0]), "=r"(r[q][1 % X]), "=r"(r[q][2 % X]), "=r"(r[q][3 % X]), "=r"(r[q][4 % X]),
                              "=r"(r[q][5 % X]), "=r"(r[q][6 % X]), "=r"(r[q][7 % X]), "=r"(r[q][8 % X]),
                              "=r"(r[q][9 % X]), "=r"(r[q][10 % X]), "=r"(r[q][11 % X]), "=r"(r[q][12 % X]),
                              "=r"(r[q][13 % X]), "=r"(r[q][14 % X]), "=r"(r[q][15 % X])
                            : "r"(ta + col));
                    else if (X == 16)
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                            : "=r"(r[q][0]), "=r"(r[q][1 % X]), "=r"(r[q][2 % X]), "=r"(r[q][3 % X]), "=r"(r[q][4 % X]),
                              "=r"(r[q][5 % X]), "=r"(r[q][6 % X]), "=r"(r[q][7 % X]), "=r"(r[q][8 % X]),
                              "=r"(r[q][9 % X]), "=r"(r[q][10 % X]), "=r"(r[q][11 % X]), "=r"(r[q][12 % X]),
                              "=r"(r[q][13 % X]), "=r"(r[q][14 % X]), "=r"(r[q][15 % X])
                            : "r"(ta + col));
                    else
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                            : "=r"(r[q][0]), "=r"(r[q][1 % X]), "=r"(r[q][2 % X]), "=r"(r[q][3 % X]), "=r"(r[q][4 % X]),
                              "=r"(r[q][5 % X]), "=r"(r[q][6 % X]), "=r"(r[q][7 % X]), "=r"(r[q][8 % X]),
                              "=r"(r[q][9 % X]), "=r"(r[q][10 % X]), "=r"(r[q][11 % X]), "=r"(r[q][12 % X]),
                              "=r"(r[q][13 % X]), "=r"(r[q][14 % X]), "=r"(r[q][15 % X]), "=r"(r[q][16 % X]),
                              "=r"(r[q][17 % X]), "=r"(r[q][18 % X]), "=r"(r[q][19 % X]), "=r"(r[q][20 % X]),
                              "=r"(r[q][21 % X]), "=r"(r[q][22 % X]), "=r"(r[q][23 % X]), "=r"(r[q][24 % X]),
                              "=r"(r[q][25 % X]), "=r"(r[q][26 % X]), "=r"(r[q][27 % X]), "=r"(r[q][28 % X]),
                              "=r"(r[q][29 % X]), "=r"(r[q][30 % X]), "=r"(r[q][31 % X])
                            : "r"(ta + col));
                    if (MODE == 12) {
#pragma unroll
                        for (int z = 0; z < 8; ++z) acc += sm[((it * 37 + (k + q) * 131 + z * 17) & 511) * 32 + lane];
                    }
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < F; ++q)
#pragma unroll
                    for (int z = 0; z < X; ++z) acc ^= r[q][z];
            }
        } else if (MODE == 7) {  // STS.32 conflict-free
#pragma unroll
            for (int k = 0; k < 32; ++k) sm[((it * 37 + k * 131) & 511) * 32 + lane] = acc + k;
        } else if (MODE == 8) {  // SHFL.UP width 8
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += __shfl_up_sync(0xffffffffu, acc + k, 1 + (k & 3), 8);
        }
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) atomicAdd(cyc, t1 - t0);
    out[blockIdx.x * 512 + threadIdx.x] = acc;
    if (kTm) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

template <int MODE>
void run(const char* name, uint32_t* out, unsigned long long* cyc, const Tab& tab) {
    const int iters = 256, smem = 65536;
    cudaFuncSetAttribute(ub<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    ub<MODE><<<148, 512, smem>>>(out, 8, tab, cyc);
    cudaDeviceSynchronize();
    cudaMemset(cyc, 0, 8);
    ub<MODE><<<148, 512, smem>>>(out, iters, tab, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // c = sum over warps of per-warp elapsed cycles; per SM the 16 warps run concurrently
    const double per_warp = (double)c / (148.0 * 16);
    const double instrs_per_sm = 16.0 * iters * 32;
    printf("%-8s %s  SM cycles per warp-instr: %.3f\n", name, e == cudaSuccess ? "ok " : cudaGetErrorString(e),
           per_warp / instrs_per_sm);
}

int main() {
    uint32_t* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 8);
    static Tab tab;
    for (int i = 0; i < 2048; ++i) tab.v[i] = i * 7u;
    run<0>("lds32", out, cyc, tab);
    run<1>("lds128b", out, cyc, tab);
    run<2>("lds32b", out, cyc, tab);
    run<3>("ldcu", out, cyc, tab);
    run<4>("ldtm1", out, cyc, tab);
    run<5>("ldtm2", out, cyc, tab);
    run<6>("ldtm4", out, cyc, tab);
    run<7>("sts32", out, cyc, tab);
    run<8>("shfl", out, cyc, tab);
    run<9>("ldtm8", out, cyc, tab);
    run<10>("ldtm16", out, cyc, tab);
    run<11>("ldtm32", out, cyc, tab);
    run<12>("ldtm16+8lds", out, cyc, tab);
    run<13>("ldtm16p", out, cyc, tab);
    return 0;
}
