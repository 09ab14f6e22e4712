// warp.cu — §8(a) row a5 (configs[4]): nearest-neighbour 32x32 patch warp.
// Patch pixel (u, v) <- image at the R6 sample point of offset (u-16, v-16), clamped
// into the image (border replicate).
//
// One warp per keypoint.  The kernel is bound by L1 lookups of its scattered byte gathers
// (one per distinct 128-byte line per warp instruction), so the 32 lanes of every gather
// instruction follow a DIGITAL LINE of the sample grid along which the image row stays
// (nearly) constant: for a frame with |sin| <= |cos| the lanes are the 32 columns u and
// instruction k samples v = (k + r(u)) mod 32 with r(u) = round(u * -b/a) (otherwise roles of
// u and v swap).  Every (u, v) is visited exactly once, and the samples of one instruction
// lie on 1-2 short image-row segments: on configs[4] ~206 line lookups per keypoint against
// ~890 for row-per-instruction and a lower bound of ~170 distinct lines.
// The bytes are re-assembled in a per-warp 32x36 shared tile and leave as 32-byte rows.
#include <math.h>

#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kWarpsNN = 8;
constexpr int kTilePitch = 36;  // bytes per patch row in the smem tile

// exact float of a small non-negative int (< 2^23) minus 16: no I2F
__device__ __forceinline__ float off16(int i) {
    return __int_as_float(0x4B000000 | i) - 8388624.0f;  // 2^23 + 16
}

template <bool LANE_U, bool CLAMP>
__device__ __forceinline__ void gather_lines(const uint8_t* __restrict__ I, int64_t pitch, int H, int W, float x0,
                                             float y0, float a, float b, int lane, int r, uint8_t* tile) {
    const float fl = off16(lane);
#pragma unroll 16
    for (int k = 0; k < 32; ++k) {
        const int o = (k + r) & 31;                // the other coordinate of this lane's sample
        const float fo = off16(o);
        const float fdx = LANE_U ? fl : fo, fdy = LANE_U ? fo : fl;
        // R6: X = x + (a*dx - b*dy), Y = y + (b*dx + a*dy) in fp32, this order, no FMA;
        // p = floor(X + 1/2) of the EXACT sum: the add rounds toward -inf, so it never rounds
        // up onto an integer (e.g. X = 0.5 - 2^-25 gives 0, not 1) and, integers being
        // representable (|X| < 2^23), never drops below one either
        const float X = __fadd_rn(x0, __fsub_rn(__fmul_rn(a, fdx), __fmul_rn(b, fdy)));
        const float Y = __fadd_rn(y0, __fadd_rn(__fmul_rn(b, fdx), __fmul_rn(a, fdy)));
        int x = __float2int_rd(__fadd_rd(X, 0.5f)), y = __float2int_rd(__fadd_rd(Y, 0.5f));
        uint8_t px;
        if (CLAMP) {
            x = min(max(x, 0), W - 1);
            y = min(max(y, 0), H - 1);
            px = __ldg(I + (int64_t)y * pitch + x);
        } else {  // footprint inside an image of < 2 GiB: 32-bit offsets
            BD_CHECK(x >= 0 && x < W && y >= 0 && y < H);
            px = __ldg(I + ((uint32_t)y * (uint32_t)pitch + (uint32_t)x));
        }
        const int u = LANE_U ? lane : o, v = LANE_U ? o : lane;
        tile[v * kTilePitch + u] = px;
    }
}

// NEXT-2 bilinear sample (reading R28): offsets (u-15.5, v-15.5) under the R6
// fp32 rule, x0 = floor(X), fx = X - x0 (exact), the 4 neighbours clamped into the image,
// v = (1-fy)((1-fx)I00 + fx I01) + fy((1-fx)I10 + fx I11) in fp32 in this order without FMA,
// p = floor(v + 1/2): the quantisation decision is taken in fp32 by this fixed rule.
// two horizontally adjacent bytes p[0], p[1] (p[0] in the low byte) from 4-byte aligned words:
// the word holding p[0], and the next word only when p[0] is its last byte (a quarter of the
// lanes) — one gather where two byte gathers would touch the same sector twice.  Needs a
// 4-byte aligned image base and pitch (checked by the caller).
__device__ __forceinline__ uint32_t load_pair(const uint8_t* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
    const uint32_t w0 = __ldg(w);
    const uint32_t w1 = (a & 3) == 3 ? __ldg(w + 1) : 0u;
    return __funnelshift_r(w0, w1, 8u * (uint32_t)(a & 3)) & 0xffffu;
}

template <bool LANE_U, bool FAST>
__device__ __forceinline__ void gather_bilinear(const uint8_t* __restrict__ I, int64_t pitch, int H, int W, float x0,
                                                float y0, float a, float b, int lane, int r, uint8_t* tile) {
    const float fl = __fsub_rn((float)lane, 15.5f);
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
        const int o = (k + r) & 31;
        const float fo = __fsub_rn((float)o, 15.5f);
        const float du = LANE_U ? fl : fo, dv = LANE_U ? fo : fl;
        const float X = __fadd_rn(x0, __fsub_rn(__fmul_rn(a, du), __fmul_rn(b, dv)));
        const float Y = __fadd_rn(y0, __fadd_rn(__fmul_rn(b, du), __fmul_rn(a, dv)));
        const float fx0 = floorf(X), fy0 = floorf(Y);
        const float fx = __fsub_rn(X, fx0), fy = __fsub_rn(Y, fy0);
        const int xi = (int)fx0, yi = (int)fy0;
        float I00, I01, I10, I11;
        if (FAST) {  // footprint (and its +1 neighbours) inside the image: no clamping
            BD_CHECK(xi >= 0 && xi + 1 < W && yi >= 0 && yi + 1 < H);
            const uint8_t* ra = I + (int64_t)yi * pitch + xi;
            const uint32_t pa = load_pair(ra), pb = load_pair(ra + pitch);
            I00 = (float)(pa & 0xffu), I01 = (float)(pa >> 8), I10 = (float)(pb & 0xffu), I11 = (float)(pb >> 8);
        } else {
            const int xa = min(max(xi, 0), W - 1), xb = min(max(xi + 1, 0), W - 1);
            const int ya = min(max(yi, 0), H - 1), yb = min(max(yi + 1, 0), H - 1);
            const uint8_t* ra = I + (int64_t)ya * pitch;
            const uint8_t* rb = I + (int64_t)yb * pitch;
            I00 = (float)__ldg(ra + xa), I01 = (float)__ldg(ra + xb);
            I10 = (float)__ldg(rb + xa), I11 = (float)__ldg(rb + xb);
        }
        const float gx = __fsub_rn(1.0f, fx), gy = __fsub_rn(1.0f, fy);
        const float top = __fadd_rn(__fmul_rn(gx, I00), __fmul_rn(fx, I01));
        const float bot = __fadd_rn(__fmul_rn(gx, I10), __fmul_rn(fx, I11));
        const float val = __fadd_rn(__fmul_rn(gy, top), __fmul_rn(fy, bot));
        int p = __float2int_rd(__fadd_rn(val, 0.5f));
        p = min(max(p, 0), 255);
        const int u = LANE_U ? lane : o, v = LANE_U ? o : lane;
        tile[v * kTilePitch + u] = (uint8_t)p;
    }
}

template <int MODE>
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
    // digital line: lanes along u when |b| <= |a| (Y = y + b du + a dv constant along
    // dv/du = -b/a), else along v (du/dv = -a/b); r = the lane's offset along the line
    const bool lane_u = fabsf(b) <= fabsf(a);
    const float slope = lane_u ? -b / a : -a / b;  // |slope| <= 1
    const int r = (int)floorf(slope * (float)lane + 0.5f) & 31;
    // footprint inside the image?  every offset has |dx|, |dy| <= 16
    const float ext = 16.0f * (fabsf(a) + fabsf(b)) + 2.0f;
    const bool inside = kv.x - ext >= 0.0f && kv.y - ext >= 0.0f && kv.x + ext <= (float)(W - 1) &&
                        kv.y + ext <= (float)(H - 1) && (int64_t)H * pitch < (1ll << 31);
    const uint8_t* I = images + (int64_t)img * pitch * H;
    uint8_t* tile = s_tile[warp];
    if (MODE == BD_WARP_BILINEAR) {
        // fast path: every sample and its +1 neighbours inside, 4-byte aligned rows
        const bool fast = kv.x - ext >= 0.0f && kv.y - ext >= 0.0f && kv.x + ext <= (float)(W - 2) &&
                          kv.y + ext <= (float)(H - 2) && (pitch & 3) == 0 &&
                          (reinterpret_cast<uintptr_t>(images) & 3) == 0;
        if (lane_u) {
            if (fast)
                gather_bilinear<true, true>(I, pitch, H, W, kv.x, kv.y, a, b, lane, r, tile);
            else
                gather_bilinear<true, false>(I, pitch, H, W, kv.x, kv.y, a, b, lane, r, tile);
        } else {
            if (fast)
                gather_bilinear<false, true>(I, pitch, H, W, kv.x, kv.y, a, b, lane, r, tile);
            else
                gather_bilinear<false, false>(I, pitch, H, W, kv.x, kv.y, a, b, lane, r, tile);
        }
    } else if (lane_u) {
        if (inside)
            gather_lines<true, false>(I, pitch, H, W, kv.x, kv.y, a, b, lane, r, tile);
        else
            gather_lines<true, true>(I, pitch, H, W, kv.x, kv.y, a, b, lane, r, tile);
    } else {
        if (inside)
            gather_lines<false, false>(I, pitch, H, W, kv.x, kv.y, a, b, lane, r, tile);
        else
            gather_lines<false, true>(I, pitch, H, W, kv.x, kv.y, a, b, lane, r, tile);
    }
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
cudaError_t launch_warp_nn(const uint8_t* images, int n_img, int H, int W, int64_t pitch, int mode,
                           const bd_keypoint* kps,
                           const int32_t* kp_image, int64_t n_kp, uint8_t* patches, uint8_t* status,
                           cudaStream_t s) {
    const int64_t blocks = (n_kp + kWarpsNN - 1) / kWarpsNN;
    ProfScope ps("warp_nn", s);
    if (mode == BD_WARP_BILINEAR)
        warp_nn_kernel<BD_WARP_BILINEAR><<<(unsigned)blocks, kWarpsNN * 32, 0, s>>>(images, n_img, H, W, pitch, kps,
                                                                                     kp_image, n_kp, patches, status);
    else
        warp_nn_kernel<BD_WARP_NN><<<(unsigned)blocks, kWarpsNN * 32, 0, s>>>(images, n_img, H, W, pitch, kps,
                                                                               kp_image, n_kp, patches, status);
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
