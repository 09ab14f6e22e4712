// warp.cu — §8(a) row a5 (configs[4]): nearest-neighbour 32x32 patch warp.
// Patch pixel (u, v) <- image at the R6 sample point of offset (u-16, v-16), clamped
// into the image (border replicate).
//
// One warp per keypoint.  The kernel is bound by L1 tag lookups of its scattered byte
// gathers (one per distinct 128-byte line per warp instruction), so the 32 lanes of each
// gather instruction cover a compact aw x bh block of the sample grid (aw * bh = 32) whose
// shape is chosen per keypoint from its rotation and scale to minimise the lines one
// instruction touches (a 32x1 row for near-horizontal frames, 8x4 near 45 degrees, ...):
// 2x fewer line lookups than row-per-instruction on configs[4].  The bytes
// are re-assembled in a per-warp 32x36 shared tile and leave as 32-byte coalesced rows.
#include <math.h>

#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kWarpsNN = 8;
constexpr int kTilePitch = 36;  // bytes per patch row in the smem tile (conflict-free columns)

// Gather the 32x32 samples of one keypoint with lane blocks of (32 >> C) x (1 << C) samples
// and scatter them into the warp's smem tile.  CLAMP = false when the whole footprint is
// inside the image (the per-sample clamps are then no-ops and skipped).
template <int C, bool CLAMP>
__device__ __forceinline__ void gather_nn(const uint8_t* __restrict__ I, uint32_t pitch, int H, int W, float x0,
                                          float y0, float a, float b, int lane, uint8_t* tile) {
    constexpr int AW = 32 >> C, NBU = 1 << C;
    const int lu = lane & (AW - 1), lv = lane >> (5 - C);
    const float flu = (float)(lu - 16), flv = (float)(lv - 16);
    uint8_t px[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        const int ub = (k % NBU) * AW, vb = (k / NBU) * NBU;  // block origin (compile time)
        const float fdx = flu + (float)ub, fdy = flv + (float)vb;  // exact small integers
        // R6: X = x + (a*dx - b*dy), Y = y + (b*dx + a*dy) in fp32, this order, no FMA;
        // floor(X + 0.5) is exact in fp32 (|X| < 2^23)
        const float X = __fadd_rn(x0, __fsub_rn(__fmul_rn(a, fdx), __fmul_rn(b, fdy)));
        const float Y = __fadd_rn(y0, __fadd_rn(__fmul_rn(b, fdx), __fmul_rn(a, fdy)));
        int x = __float2int_rd(__fadd_rn(X, 0.5f)), y = __float2int_rd(__fadd_rn(Y, 0.5f));
        if (CLAMP) {
            x = min(max(x, 0), W - 1);
            y = min(max(y, 0), H - 1);
        }
        px[k] = __ldg(I + (uint32_t)((uint32_t)y * pitch + (uint32_t)x));
    }
    uint8_t* t = tile + lv * kTilePitch + lu;
#pragma unroll
    for (int k = 0; k < 32; ++k) t[(k / NBU) * NBU * kTilePitch + (k % NBU) * AW] = px[k];
}

__global__ void __launch_bounds__(kWarpsNN * 32) warp_nn_kernel(const uint8_t* __restrict__ images, int n_img,
                                                                int H, int W, int64_t pitch,
                                                                const bd_keypoint* __restrict__ kps,
                                                                const int32_t* __restrict__ kp_image, int64_t n_kp,
                                                                uint8_t* __restrict__ patches,
                                                                uint8_t* __restrict__ status) {
    __shared__ __align__(16) uint8_t s_tile[kWarpsNN][32 * kTilePitch];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * kWarpsNN + warp;
    if (i >= n_kp) return;
    const float4 kv = __ldg(reinterpret_cast<const float4*>(kps) + i);
    const int img = kp_image ? __ldg(kp_image + i) : 0;
    const bool valid = isfinite(kv.x) && isfinite(kv.y) && isfinite(kv.z) && isfinite(kv.w) &&
                       kv.w > 0.0f && kv.x >= 0.0f && kv.y >= 0.0f && kv.x <= (float)(W - 1) &&
                       kv.y <= (float)(H - 1) && img >= 0 && img < n_img;
    uint4* orow = reinterpret_cast<uint4*>(patches + i * 1024 + lane * 32);
    if (!valid) {
        orow[0] = make_uint4(0, 0, 0, 0);
        orow[1] = make_uint4(0, 0, 0, 0);
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
    // block shape aw x bh = (32 >> c) x (1 << c): estimated lines per instruction =
    // rows spanned x (1 + columns spanned / 128)
    const float fa = fabsf(a), fb = fabsf(b);
    int c = 0;
    float best = 3.0e38f;
#pragma unroll
    for (int cc = 0; cc < 6; ++cc) {
        const float aw1 = (float)((32 >> cc) - 1), bh1 = (float)((1 << cc) - 1);
        const float rows = fb * aw1 + fa * bh1 + 1.0f, cols = fa * aw1 + fb * bh1;
        const float est = rows * (1.0f + cols * (1.0f / 128.0f));
        if (est < best) {
            best = est;
            c = cc;
        }
    }
    // footprint inside the image?  every offset has |dx|, |dy| <= 16, so |X - x| and
    // |Y - y| <= 16 (|a| + |b|) (+ rounding slack)
    const float ext = 16.0f * (fa + fb) + 2.0f;
    const bool inside = kv.x - ext >= 0.0f && kv.y - ext >= 0.0f && kv.x + ext <= (float)(W - 1) &&
                        kv.y + ext <= (float)(H - 1) && (int64_t)H * pitch < (1ll << 31);
    const uint8_t* I = images + (int64_t)img * pitch * H;
    uint8_t* tile = s_tile[warp];
    const uint32_t p32 = (uint32_t)pitch;
#define BD_GATHER(CC)                                                                   \
    case CC:                                                                            \
        if (inside)                                                                     \
            gather_nn<CC, false>(I, p32, H, W, kv.x, kv.y, a, b, lane, tile);           \
        else                                                                            \
            gather_nn<CC, true>(I, p32, H, W, kv.x, kv.y, a, b, lane, tile);            \
        break;
    if ((int64_t)H * pitch < (1ll << 31)) {
        switch (c) {
            BD_GATHER(0)
            BD_GATHER(1)
            BD_GATHER(2)
            BD_GATHER(3)
            BD_GATHER(4)
            default:
                BD_GATHER(5)
        }
    } else {  // > 2 GiB images: 64-bit row offsets, clamped path only
        const float flu = (float)(lane - 16);
#pragma unroll 4
        for (int v = 0; v < 32; ++v) {
            const float fdx = flu, fdy = (float)(v - 16);
            const float X = __fadd_rn(kv.x, __fsub_rn(__fmul_rn(a, fdx), __fmul_rn(b, fdy)));
            const float Y = __fadd_rn(kv.y, __fadd_rn(__fmul_rn(b, fdx), __fmul_rn(a, fdy)));
            int x = __float2int_rd(__fadd_rn(X, 0.5f)), y = __float2int_rd(__fadd_rn(Y, 0.5f));
            x = min(max(x, 0), W - 1);
            y = min(max(y, 0), H - 1);
            tile[v * kTilePitch + lane] = __ldg(I + (int64_t)y * pitch + x);
        }
    }
#undef BD_GATHER
    __syncwarp();
    const uint32_t* trow = reinterpret_cast<const uint32_t*>(tile + lane * kTilePitch);
    orow[0] = make_uint4(trow[0], trow[1], trow[2], trow[3]);
    orow[1] = make_uint4(trow[4], trow[5], trow[6], trow[7]);
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
    const int64_t blocks = (n_kp + kWarpsNN - 1) / kWarpsNN;
    ProfScope ps("warp_nn", s);
    warp_nn_kernel<<<(unsigned)blocks, kWarpsNN * 32, 0, s>>>(images, n_img, H, W, pitch, kps, kp_image, n_kp,
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
