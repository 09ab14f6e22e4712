// project.cu — §8(a) row a9: p = W v + b, bit k = [p_k >= 0] (P:242 D(x) = sgn(B[f;1]),
// sgn(0) = +1 (R15)), packed LSB-first with __ballot_sync (lane = bit position).
//
// v1: FP32 CUDA-core GEMM [n x 128] . [128 x N] with the sign/pack epilogue fused.
// Persistent CTAs, each owning one 256-column chunk of W^T (128 KB smem, loaded once) and
// looping over 64-descriptor tiles (33 KB).  Warp w computes descriptors 8w..8w+7, lane
// computes columns lane + 32m (m = 0..7): 64 fp32 accumulators per thread.  FP32 keeps the
// projection error ~1e-6, far inside the |p| < 1e-3 ambiguity band (R13).
#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kTileD = 64;
constexpr int kApitch = 132;  // floats per descriptor row in smem (528 B: 16-B aligned, skewed)
constexpr int kChunk = 256;
constexpr int kSmem = (128 * kChunk + kTileD * kApitch) * 4;

__global__ void __launch_bounds__(256, 1) project_kernel(const float* __restrict__ sift, int64_t n,
                                                         const float* __restrict__ wt,  // [128][N]
                                                         const float* __restrict__ bias, int N,
                                                         uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) float sm[];
    float* Ws = sm;                   // [128][256]
    float* As = sm + 128 * kChunk;    // [64][132]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int chunk = blockIdx.y;     // columns [256 chunk, 256 chunk + 256)
    const int ncols = min(kChunk, N - chunk * kChunk);
    for (int idx = threadIdx.x; idx < 128 * kChunk; idx += blockDim.x) {
        const int i = idx / kChunk, c = idx % kChunk;
        Ws[idx] = (c < ncols) ? wt[(int64_t)i * N + chunk * kChunk + c] : 0.f;
    }
    float bv[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const int c = lane + 32 * m;
        bv[m] = (c < ncols) ? bias[chunk * kChunk + c] : 0.f;
    }
    const int words = N >> 5;
    const int64_t n_tiles = (n + kTileD - 1) / kTileD;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        __syncthreads();
        const int64_t d0 = t * kTileD;
        const int nd = (int)min((int64_t)kTileD, n - d0);
        const float4* src = reinterpret_cast<const float4*>(sift + d0 * 128);
        for (int f = threadIdx.x; f < kTileD * 32; f += blockDim.x) {
            const int d = f >> 5, i4 = f & 31;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (d < nd) v = __ldg(src + f);
            *reinterpret_cast<float4*>(As + d * kApitch + 4 * i4) = v;
        }
        __syncthreads();
        float acc[8][8];
#pragma unroll
        for (int d = 0; d < 8; ++d)
#pragma unroll
            for (int m = 0; m < 8; ++m) acc[d][m] = 0.f;
        const float* Aw = As + (8 * warp) * kApitch;
#pragma unroll 2
        for (int i = 0; i < 128; i += 4) {
            float4 a[8];
#pragma unroll
            for (int d = 0; d < 8; ++d) a[d] = *reinterpret_cast<const float4*>(Aw + d * kApitch + i);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float w[8];
#pragma unroll
                for (int m = 0; m < 8; ++m) w[m] = Ws[(i + k) * kChunk + lane + 32 * m];
#pragma unroll
                for (int d = 0; d < 8; ++d) {
                    const float ad = k == 0 ? a[d].x : k == 1 ? a[d].y : k == 2 ? a[d].z : a[d].w;
#pragma unroll
                    for (int m = 0; m < 8; ++m) acc[d][m] = fmaf(ad, w[m], acc[d][m]);
                }
            }
        }
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            uint32_t mine = 0;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const uint32_t b = __ballot_sync(0xffffffffu, acc[d][m] + bv[m] >= 0.f);
                if (lane == m) mine = b;
            }
            const int dd = 8 * warp + d;
            if (lane < 8 && lane < (ncols >> 5) && dd < nd) out[(d0 + dd) * words + chunk * 8 + lane] = mine;
        }
    }
}

}  // namespace kern

using namespace kern;
cudaError_t launch_project(const float* sift, int64_t n, const float* wt, const float* bias, int N, uint32_t* out,
                           cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t tiles = (n + kTileD - 1) / kTileD;
    const int chunks = (N + kChunk - 1) / kChunk;
    int gx = (int)(tiles < num_sms() ? tiles : num_sms());
    if (chunks > 1) gx = (gx + chunks - 1) / chunks;
    dim3 grid(gx, chunks);
    ProfScope ps("project", s);
    project_kernel<<<grid, 256, kSmem, s>>>(sift, n, wt, bias, N, out);
    return cudaGetLastError();
}

}  // namespace bd
