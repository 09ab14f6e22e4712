// project.cu — §8(a) row a9: p = W v + b, bit k = [p_k >= 0] (P:242 D(x) = sgn(B[f;1]),
// sgn(0) = +1, R15), packed LSB-first (R16).  BJ.ns (4): "the 128 to N projection as a
// tensor-core GEMM over the batch, because that projection is the only truly dense
// contraction here".
//
// sm_100a tcgen05 kernel, kind::tf32, TMA-fed and pipelined:
//  * persistent CTAs, one 256-column chunk of W per CTA (blockIdx.y); the chunk (nc x 128
//    fp32, the B operand, K-major) is loaded ONCE into shared memory in the SWIZZLE_128B
//    K-major canonical layout (4 K-blocks of 32 fp32, 16-byte chunk c of row r at c^(r%8));
//  * A (the SIFT rows of a 128-descriptor tile) streams through a 3-stage ring of K-halves
//    (128 rows x 64 fp32 = 32 KB each), each filled by two 2-D TMA loads
//    (cp.async.bulk.tensor, SWIZZLE_128B, OOB rows zero-filled) — the tensor engine writes
//    exactly the canonical layout the MMA descriptor expects;
//  * warp 5 (one lane) is the TMA producer, running up to 3 K-halves (96 KB) ahead — the
//    bytes in flight that hide HBM latency at this SM's share of the bandwidth (a producer
//    that waited for its own load before issuing the MMAs kept one 32 KB load in flight:
//    47 % of HBM); warp 4 (one lane) issues per K-half 8 tcgen05.mma (M = 128, N = nc, K = 8)
//    into a TMEM accumulator; tcgen05.commit frees the A stage and, after the tile, signals
//    the epilogue; the accumulator is double-buffered in TMEM (2 x 256 columns) so the
//    epilogue of tile t overlaps the loads and MMAs of tile t+1;
//  * warps 0-3 (epilogue): warp w owns TMEM lanes 32w..32w+31 (= descriptor rows);
//    tcgen05.ld.32x32b.x32 returns 32 consecutive columns = 32 bits of that row, so each
//    thread adds the bias and packs its own word — no ballot needed;
//  * TF32 operands (10-bit mantissa) keep |p - p_fp64| ~ 1e-5 typical, inside the 1e-3
//    ambiguity band of R13 (R26).
#include "internal.cuh"
#include "tc.cuh"

namespace bd {
namespace kern {

constexpr int kM = 128;          // descriptors per tile (UMMA M)
constexpr int kNC = 256;         // max columns per CTA / MMA (UMMA N)
constexpr int kEpiWarps = 4;
constexpr int kThreads = (kEpiWarps + 2) * 32;  // + MMA issuer warp + TMA producer warp
constexpr int kStages = 3;                       // A ring: 3 K-halves (96 KB) in flight
constexpr int kStageBytes = kM * 64 * 4;   // one K-half of A: 32 KB
constexpr int kAtomBytes = kM * 128;       // 128 rows x 128 B (32 fp32): 16 KB

// byte offset of fp32 element (row r, k) in a SWIZZLE_128B K-major operand of `rows` rows
__device__ __forceinline__ uint32_t sw128_offset(int r, int k, int rows) {
    const int kb = k >> 5, c = (k >> 2) & 7;
    return (uint32_t)(kb * rows * 128 + r * 128 + ((c ^ (r & 7)) << 4) + ((k & 3) << 2));
}

using namespace tc;  // smem_addr, desc_sw128, idesc_tf32, mbarriers, TMA, commit, tmem_ld32

__global__ void __launch_bounds__(kThreads, 1)
    project_tc_kernel(const __grid_constant__ CUtensorMap tmA, int64_t n, const float* __restrict__ w,  // [N][128]
                      const float* __restrict__ bias, int N, uint32_t* __restrict__ out,
                      const uint8_t* __restrict__ status) {
    extern __shared__ uint8_t smem_raw[];
    debug_poison_smem(smem_raw);
    __shared__ uint64_t full[kStages], empty[kStages], dfull[2], dfree[2];
    __shared__ uint32_t tmem_base_s;
    __shared__ float s_bias[kNC];
    // 1024-byte aligned operand region (SWIZZLE_128B atoms)
    const uint32_t raw = smem_addr(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int ch = blockIdx.y;
    const int nc = min(kNC, N - ch * kNC);          // columns of this CTA (multiple of 32)
    uint8_t* sW = base;                              // nc x 128 fp32
    uint8_t* sA = base + nc * 512;                   // kStages x 32 KB (nc*512 is 1024-aligned)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // ---- one-time setup: W chunk into smem, bias, mbarriers, TMEM ----
    const float4* wsrc = reinterpret_cast<const float4*>(w + (int64_t)ch * kNC * 128);
    for (int idx = tid; idx < nc * 32; idx += kThreads) {
        const int r = idx >> 5, c4 = idx & 31;
        *reinterpret_cast<float4*>(sW + sw128_offset(r, 4 * c4, nc)) = __ldg(wsrc + idx);
    }
    for (int i = tid; i < nc; i += kThreads) s_bias[i] = bias[ch * kNC + i];
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&dfull[s], 1);
            mbar_init(&dfree[s], kEpiWarps * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    }
    if (warp == kEpiWarps) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_addr(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // W (generic writes) -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    const int words_out = N >> 5, words = nc >> 5;
    const int64_t n_tiles = (n + kM - 1) / kM;

    if (warp == kEpiWarps + 1) {
        // ---------------- TMA producer (one lane): K-halves up to kStages ahead ----------------
        if (lane == 0) {
            int g = 0;  // global K-half counter: slot g % kStages, use (g / kStages)
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x)
                for (int kh = 0; kh < 2; ++kh, ++g) {
                    const int slot = g % kStages, use = g / kStages;
                    if (use >= 1) mbar_wait(&empty[slot], (use - 1) & 1);  // consumed by the MMAs
                    mbar_expect_tx(&full[slot], kStageBytes);
                    uint8_t* st = sA + slot * kStageBytes;
                    tma_load_2d(st, &tmA, 64 * kh, (int)(t * kM), &full[slot]);
                    tma_load_2d(st + kAtomBytes, &tmA, 64 * kh + 32, (int)(t * kM), &full[slot]);
                }
        }
        __syncwarp();
    } else if (warp == kEpiWarps) {
        // ---------------- MMA issuer (one lane) ----------------
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32(kM, nc);
            const uint32_t aBase = smem_addr(sA), wBase = smem_addr(sW);
            int it = 0, g = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
                const int buf = it & 1;
                if (it >= 2) mbar_wait(&dfree[buf], ((it - 2) >> 1) & 1);  // accumulator drained
                for (int kh = 0; kh < 2; ++kh, ++g) {
                    const int slot = g % kStages;
                    mbar_wait(&full[slot], (g / kStages) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const int kb = ks >> 2, k8 = ks & 3;  // atom within the stage, K=8 step
                        const uint64_t ad = desc_sw128(aBase + slot * kStageBytes + kb * kAtomBytes + k8 * 32);
                        const uint64_t bd = desc_sw128(wBase + (2 * kh + kb) * nc * 128 + k8 * 32);
                        const uint32_t acc = (kh > 0 || ks > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                                tmem + (uint32_t)(buf * kNC)),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
                            : "memory");
                    }
                    mma_commit(&empty[slot]);  // this stage may be refilled once these MMAs finish
                }
                mma_commit(&dfull[buf]);       // accumulator complete
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: thread = descriptor row = TMEM lane ----------------
        int it = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
            const int buf = it & 1;
            mbar_wait(&dfull[buf], (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t r0 = t * kM;
            const int rows = (int)min((int64_t)kM, n - r0);
            const int row = warp * 32 + lane;
            const uint32_t taddr = tmem + (uint32_t)(buf * kNC) + ((uint32_t)(warp * 32) << 16);
            uint32_t* o = out + (r0 + row) * words_out + ch * (kNC / 32);
            // invalid keypoints (status != 0) get all-zero rows (bd_describe_warped)
            const uint32_t keep = (status && row < rows && status[r0 + row]) ? 0u : ~0u;
            for (int wd = 0; wd < words; ++wd) {
                uint32_t v[32];
                tmem_ld32(taddr + wd * 32, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                uint32_t b = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) b |= (uint32_t)(__uint_as_float(v[j]) + s_bias[wd * 32 + j] >= 0.f) << j;
                if (row < rows) o[wd] = b & keep;
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&dfree[buf]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == kEpiWarps) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

}  // namespace kern

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

using namespace kern;
cudaError_t launch_project(const float* sift, int64_t n, const float* w, const float* bias, int N, uint32_t* out,
                           const uint8_t* status, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (n > 0x7fffffffLL) return cudaErrorInvalidValue;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    // A = SIFT rows: 2-D fp32 tensor {K = 128, rows = n}, row stride 512 B, box {32, 128}
    CUtensorMap map;
    const cuuint64_t dims[2] = {128, (cuuint64_t)n};
    const cuuint64_t strides[1] = {512};
    const cuuint32_t box[2] = {32, (cuuint32_t)kM};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(sift), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    const int smem = kNC * 512 + kStages * kStageBytes + 1024;  // W chunk + A ring + alignment slack = 230400
    cudaError_t e0 = ensure_smem_attr((const void*)project_tc_kernel, smem);
    if (e0 != cudaSuccess) return e0;
    const int chunks = (N + kNC - 1) / kNC;
    const int64_t tiles = (n + kM - 1) / kM;
    int gx = num_sms() / chunks;
    if (tiles < gx) gx = (int)tiles;
    ProfScope ps("project", s);
    project_tc_kernel<<<dim3(gx, chunks), kThreads, smem, s>>>(map, n, w, bias, N, out, status);
    return cudaGetLastError();
}

}  // namespace bd
