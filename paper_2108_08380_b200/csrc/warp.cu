// warp.cu — §8(a) row a5 (configs[4]): nearest-neighbour 32x32 patch warp.
// Patch pixel (u, v) <- image at the R6 sample point of offset (u-16, v-16), clamped
// into the image (border replicate).  One warp per keypoint, lane = column u; the
// 32 rows are unrolled so 32 independent gathers per lane are in flight; each row leaves
// as one 32-byte coalesced store.
#include <math.h>

#include "internal.cuh"

namespace bd {
namespace kern {

__global__ void __launch_bounds__(256) warp_nn_kernel(const uint8_t* __restrict__ images, int n_img, int H, int W,
                                                      int64_t pitch, const bd_keypoint* __restrict__ kps,
                                                      const int32_t* __restrict__ kp_image, int64_t n_kp,
                                                      uint8_t* __restrict__ patches, uint8_t* __restrict__ status) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= n_kp) return;
    const float4 kv = __ldg(reinterpret_cast<const float4*>(kps) + i);
    const int img = kp_image ? __ldg(kp_image + i) : 0;
    const bool valid = isfinite(kv.x) && isfinite(kv.y) && isfinite(kv.z) && isfinite(kv.w) &&
                       kv.w > 0.0f && kv.x >= 0.0f && kv.y >= 0.0f && kv.x <= (float)(W - 1) &&
                       kv.y <= (float)(H - 1) && img >= 0 && img < n_img;
    uint8_t* o = patches + i * 1024 + lane;
    if (!valid) {
#pragma unroll
        for (int v = 0; v < 32; ++v) o[32 * v] = 0;
        if (status && lane == 0) status[i] = 1;
        return;
    }
    float a = 0.f, b = 0.f;
    if (lane == 0) {
        double sn, cs;
        sincos((double)kv.z, &sn, &cs);
        a = (float)((double)kv.w * cs);
        b = (float)((double)kv.w * sn);
    }
    a = __shfl_sync(0xffffffffu, a, 0);
    b = __shfl_sync(0xffffffffu, b, 0);
    const uint8_t* I = images + (int64_t)img * pitch * H;
    const float fdx = (float)(lane - 16);
    const float adx = __fmul_rn(a, fdx), bdx = __fmul_rn(b, fdx);
    uint8_t px[32];
#pragma unroll
    for (int v = 0; v < 32; ++v) {
        const float fdy = (float)(v - 16);
        const float X = __fadd_rn(kv.x, __fsub_rn(adx, __fmul_rn(b, fdy)));
        const float Y = __fadd_rn(kv.y, __fadd_rn(bdx, __fmul_rn(a, fdy)));
        int x = (int)floor((double)X + 0.5), y = (int)floor((double)Y + 0.5);
        x = min(max(x, 0), W - 1);
        y = min(max(y, 0), H - 1);
        px[v] = __ldg(I + (int64_t)y * pitch + x);
    }
#pragma unroll
    for (int v = 0; v < 32; ++v) o[32 * v] = px[v];
    if (status && lane == 0) status[i] = 0;
}

__global__ void zero_invalid_kernel(const uint8_t* __restrict__ status, int64_t n, uint32_t* __restrict__ out,
                                    int words) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * words) return;
    if (status[idx / words]) out[idx] = 0u;
}

}  // namespace kern

using namespace kern;
cudaError_t launch_warp_nn(const uint8_t* images, int n_img, int H, int W, int64_t pitch, const bd_keypoint* kps,
                           const int32_t* kp_image, int64_t n_kp, uint8_t* patches, uint8_t* status,
                           cudaStream_t s) {
    const int warps = 8;
    const int64_t blocks = (n_kp + warps - 1) / warps;
    ProfScope ps("warp_nn", s);
    warp_nn_kernel<<<(unsigned)blocks, warps * 32, 0, s>>>(images, n_img, H, W, pitch, kps, kp_image, n_kp,
                                                           patches, status);
    return cudaGetLastError();
}

using namespace kern;
cudaError_t launch_zero_invalid(const uint8_t* status, int64_t n, uint32_t* out, int words, cudaStream_t s) {
    const int64_t total = n * words;
    if (total == 0) return cudaSuccess;
    ProfScope ps("zero_invalid", s);
    zero_invalid_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(status, n, out, words);
    return cudaGetLastError();
}

}  // namespace bd
