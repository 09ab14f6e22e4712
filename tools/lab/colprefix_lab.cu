// colprefix_lab.cu — feasibility test (not part of the product): the column prefix of 32x32
// u8 patches as a tcgen05 kind::i8 MMA.  D[32q + y][(s, x)] = sum_{y' <= y} P_{2q+s}[y'][x]:
//   A_q = rows 32q..32q+31 of blockdiag(L) (L lower-triangular ones), K-major, no swizzle,
//         built as a window into one zero-padded buffer (28 row groups, L in groups 12..15);
//   B   = pixels of pair q (patches 2q, 2q+1) straight from a TMA SWIZZLE_32B load of the
//         natural [patch][y][x] layout: MN-major (N = x contiguous), SW32 atoms of 8 rows x
//         32 B, LBO = 1024 B (next patch), SBO = 256 B (next 8 rows);
//   4 MMAs (q = 0..3, M = 128, N = 64, K = 32) accumulate into one 64-column D.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o colprefix_lab colprefix_lab.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

__global__ void lab(const __grid_constant__ CUtensorMap map, int32_t* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stg = smem;            // 8 KB: 8 patches (TMA, SWIZZLE_32B)
    uint8_t* Z = smem + 8192;       // 28 x 256 B
    __shared__ uint64_t bar_full, bar_mma;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 28 * 256; i += blockDim.x) {
        const int g = i / 256, w = i % 256, kc = w / 128, r = (w % 128) / 16, kk = w % 16;
        const int m = (g - 12) * 8 + r, k = kc * 16 + kk;  // L row m, column k
        Z[i] = (g >= 12 && g < 16 && k <= m) ? 1 : 0;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar_full)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar_mma)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar_full)), "r"(8192) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sa(stg)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(0), "r"(sa(&bar_full))
            : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}\n" ::"r"(sa(&bar_full))
            : "memory");
        const uint32_t idesc = (2u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
        for (int q = 0; q < 4; ++q) {
            const uint64_t ad = desc(sa(Z) + (12 - 4 * q) * 256, 128, 256, 0);
            const uint64_t bd = desc(sa(stg) + 2 * q * 1024, 1024, 256, 6);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
                "l"(ad), "l"(bd), "r"(idesc), "r"(q)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar_mma))
                     : "memory");
    }
    __syncwarp();
    if (warp < 4) {
        asm volatile(
            "{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(sa(&bar_mma))
            : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int c = 0; c < 64; c += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tbase + ((uint32_t)(32 * warp) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int i = 0; i < 8; ++i) out[(warp * 32 + lane) * 64 + c + i] = (int32_t)v[i];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tbase));
}

int main() {
    const int n = 8;
    uint8_t* h = (uint8_t*)malloc(n * 1024);
    srand(1);
    for (int i = 0; i < n * 1024; ++i) h[i] = rand() & 255;
    uint8_t* d;
    int32_t* dout;
    cudaMalloc(&d, n * 1024);
    cudaMalloc(&dout, 128 * 64 * 4);
    cudaMemcpy(d, h, n * 1024, cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    CUtensorMap map;
    const cuuint64_t dims[2] = {32, (cuuint64_t)n * 32};
    const cuuint64_t strides[1] = {32};
    const cuuint32_t box[2] = {32, 256};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    cudaFuncSetAttribute(lab, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 1024);
    lab<<<1, 128, 16384 + 1024>>>(map, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    int32_t* o = (int32_t*)malloc(128 * 64 * 4);
    cudaMemcpy(o, dout, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int qq = 0; qq < 4; ++qq)
        for (int y = 0; y < 32; ++y)
            for (int s = 0; s < 2; ++s)
                for (int x = 0; x < 32; ++x) {
                    int ref = 0;
                    for (int yy = 0; yy <= y; ++yy) ref += h[(2 * qq + s) * 1024 + yy * 32 + x];
                    const int got = o[(qq * 32 + y) * 64 + s * 32 + x];
                    if (got != ref && bad++ < 10) printf("q %d y %d s %d x %d: got %d ref %d\n", qq, y, s, x, got, ref);
                }
    printf("mismatches %d of %d\n", bad, 4 * 32 * 64);
    return bad != 0;
}
