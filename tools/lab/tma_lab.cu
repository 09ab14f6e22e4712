// tma_lab.cu — staging-bandwidth test (not part of the product): stream 4M 32x32 u8 patches
// through an 8 x 8 KB smem ring per SM, (a) TMA 2-D box 32 B x 256 rows SWIZZLE_32B, (b) the same
// box without swizzle, (c) cp.async.bulk 8 KB contiguous.  No compute: GB/s of the staging alone.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(sa(b)),
                 "r"(ph) : "memory");
}
template <int MODE>
__global__ void stream(const __grid_constant__ CUtensorMap map, const uint8_t* src, int64_t n_groups, unsigned* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[8];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned acc = 0;
    int64_t issued = 0, done = 0;
    const int64_t my0 = blockIdx.x, step = gridDim.x;
    auto issue = [&](int64_t gi) {
        const int s = issued % 8;
        uint8_t* dst = sm + s * 8192;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(8192) : "memory");
        if (MODE < 2)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    sa(dst)),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"((int)(gi * 256)), "r"(sa(&bar[s]))
                : "memory");
        else
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                         "l"(src + gi * 8192), "r"(8192), "r"(sa(&bar[s]))
                         : "memory");
        ++issued;
    };
    int64_t gnext = my0;
    for (int i = 0; i < 8 && gnext < n_groups; ++i, gnext += step) issue(gnext);
    for (int64_t g = my0; g < n_groups; g += step) {
        const int s = done % 8;
        wait(&bar[s], (uint32_t)((done / 8) & 1));
        acc += sm[s * 8192 + (done & 1023)];
        ++done;
        if (gnext < n_groups) { issue(gnext); gnext += step; }
    }
    sink[blockIdx.x] = acc;
}

int main() {
    const int64_t n = 4000000, groups = n / 8;
    uint8_t* d;
    unsigned* sink;
    cudaMalloc(&d, n * 1024);
    cudaMemset(d, 1, n * 1024);
    cudaMalloc(&sink, 4096);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    CUtensorMap m32, m0;
    const cuuint64_t dims[2] = {32, (cuuint64_t)n * 32};
    const cuuint64_t strides[1] = {32};
    const cuuint32_t box[2] = {32, 256};
    const cuuint32_t estr[2] = {1, 1};
    enc(&m32, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&m0, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    cudaFuncSetAttribute(stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    cudaFuncSetAttribute(stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[3] = {"tma 32Bx256 sw32", "tma 32Bx256 noswz", "bulk 8KB"};
    for (int mode = 0; mode < 3; ++mode)
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) stream<0><<<148, 32, 65536 + 1024>>>(m32, d, groups, sink);
            if (mode == 1) stream<1><<<148, 32, 65536 + 1024>>>(m0, d, groups, sink);
            if (mode == 2) stream<2><<<148, 32, 65536 + 1024>>>(m0, d, groups, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("%-20s %.3f ms  %.0f GB/s  (%s)\n", names[mode], ms, n * 1024 / ms / 1e6,
                                 cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
