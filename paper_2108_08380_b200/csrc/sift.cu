// sift.cu — §8(a) rows a6-a8: SIFT 4x4x8 histogram of a normalised 32x32 patch
// ("the vector of real valued features provided by SIFT"; conventions R10).
//
// One warp per patch, lane = pixel column x.  The warp walks the 32 rows; each lane keeps
// the column pixels of rows y-1, y, y+1 in registers and gets x-1, x+1 by shuffle
// (replicate border).  BJ.ns (3): "fuses the gradient and orientation binning with a
// warp-level histogram reduction":
//  * per pixel: m, theta (fp32), Gaussian weight w = g(x) g(y) (sigma 16), the 8
//    orientation weights max(0, 1 - |co - o|) (circular), accumulated into two per-lane
//    8-bin registers for the two spatial cell rows j0, j0+1 the pixel touches;
//  * when the walk leaves cell row j0 (y = 12, 20, 28, end) its per-lane partial
//    histogram is reduced across lanes with the spatial x-weights 1 - |k - 7.5|/8 through a
//    33-word-padded scratch (conflict-free), landing in lane (i, o) = (L/8, L%8);
//  * the final 4 registers per lane are the 128 entries j*32 + L: L2-normalise, clip at
//    0.2, renormalise (zero stays zero) with two warp all-reductions.
#include <math.h>

#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kWarps = 8;
constexpr int kScratch = 8 * 33;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// reduce the per-lane row histogram H[8] (column x = lane) into cell row j: lane L gets
// sum_k w_k H_{x = 8i-4+k}[o] for (i, o) = (L/8, L%8), w_k = 1 - |k - 7.5| / 8.
__device__ __forceinline__ float flush_row(const float (&H)[8], float* scr, int lane) {
#pragma unroll
    for (int o = 0; o < 8; ++o) scr[o * 33 + lane] = H[o];
    __syncwarp();
    const int i = lane >> 3, o = lane & 7;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int x = 8 * i - 4 + k;
        const float wk = 1.0f - fabsf((float)k - 7.5f) * 0.125f;
        if (x >= 0 && x < 32) s = fmaf(wk, scr[o * 33 + x], s);
    }
    __syncwarp();
    return s;
}

__global__ void __launch_bounds__(kWarps * 32) sift_kernel(const uint8_t* __restrict__ patches, int64_t n,
                                                           float* __restrict__ sift) {
    __shared__ __align__(16) uint8_t s_patch[kWarps][1024];
    __shared__ float s_scr[kWarps][kScratch];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* P = s_patch[warp];
    float* scr = s_scr[warp];
    const float gxw = expf(-((float)lane - 15.5f) * ((float)lane - 15.5f) / 512.0f);  // g(x), also g(y=lane)
    const int xl = lane > 0 ? lane - 1 : 0, xr = lane < 31 ? lane + 1 : 31;
    const float k4pi = 1.27323954473516268f;  // 4/pi
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    for (int64_t p = (int64_t)blockIdx.x * kWarps + warp; p < n; p += nwarps) {
        const uint4* src = reinterpret_cast<const uint4*>(patches + p * 1024);
        const uint4 q0 = __ldg(src + lane), q1 = __ldg(src + 32 + lane);
        reinterpret_cast<uint4*>(P)[lane] = q0;
        reinterpret_cast<uint4*>(P)[32 + lane] = q1;
        __syncwarp();
        float Ha[8], Hb[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) Ha[o] = Hb[o] = 0.f;
        float h0 = 0.f, h1 = 0.f, h2 = 0.f, h3 = 0.f;
        float prev = (float)P[lane], cur = prev;
#pragma unroll
        for (int y = 0; y < 32; ++y) {
            const float next = (float)P[(y < 31 ? y + 1 : 31) * 32 + lane];
            const float left = __shfl_sync(0xffffffffu, cur, xl);
            const float right = __shfl_sync(0xffffffffu, cur, xr);
            const float gx = right - left, gy = next - prev;
            const float m = sqrtf(fmaf(gx, gx, gy * gy));
            float th = atan2f(gy, gx);
            if (th < 0.f) th += 6.28318530717958648f;
            const float co = th * k4pi;
            const float gyw = __shfl_sync(0xffffffffu, gxw, y);
            const float w = m * gxw * gyw;
            // cell rows: cy = (y - 3.5)/8, j0 = floor(cy), fy = cy - j0   (compile-time per y)
            const float cy = ((float)y - 3.5f) * 0.125f;
            const int j0 = (y < 4) ? -1 : (y - 4) / 8;
            const float fy = cy - (float)j0;
            const float wa = w * (1.0f - fy), wb = w * fy;
            float wo[8];
            wo[0] = __saturatef(1.0f - fabsf(co)) + __saturatef(1.0f - fabsf(co - 8.0f));
#pragma unroll
            for (int o = 1; o < 8; ++o) wo[o] = __saturatef(1.0f - fabsf(co - (float)o));
#pragma unroll
            for (int o = 0; o < 8; ++o) {
                if (j0 >= 0) Ha[o] = fmaf(wa, wo[o], Ha[o]);
                if (j0 + 1 <= 3) Hb[o] = fmaf(wb, wo[o], Hb[o]);
            }
            prev = cur;
            cur = next;
            // leaving cell row j0 at y = 11, 19, 27 (next y starts a new band) and at y = 31
            if (y == 3 || y == 11 || y == 19 || y == 27 || y == 31) {
                if (j0 >= 0) {
                    const float s = flush_row(Ha, scr, lane);
                    if (j0 == 0) h0 = s;
                    if (j0 == 1) h1 = s;
                    if (j0 == 2) h2 = s;
                    if (j0 == 3) h3 = s;
                }
#pragma unroll
                for (int o = 0; o < 8; ++o) {
                    Ha[o] = Hb[o];
                    Hb[o] = 0.f;
                }
            }
        }
        // normalise, clip 0.2, renormalise (R10); the zero histogram stays zero
        float n2 = warp_sum(h0 * h0 + h1 * h1 + h2 * h2 + h3 * h3);
        float* o = sift + p * 128 + lane;
        if (n2 > 0.f) {
            const float inv = 1.0f / sqrtf(n2);
            h0 = fminf(h0 * inv, 0.2f);
            h1 = fminf(h1 * inv, 0.2f);
            h2 = fminf(h2 * inv, 0.2f);
            h3 = fminf(h3 * inv, 0.2f);
            const float inv2 = 1.0f / sqrtf(warp_sum(h0 * h0 + h1 * h1 + h2 * h2 + h3 * h3));
            h0 *= inv2;
            h1 *= inv2;
            h2 *= inv2;
            h3 *= inv2;
        } else {
            h0 = h1 = h2 = h3 = 0.f;
        }
        o[0] = h0;
        o[32] = h1;
        o[64] = h2;
        o[96] = h3;
        __syncwarp();
    }
}

}  // namespace kern

using namespace kern;
cudaError_t launch_sift(const uint8_t* patches, int64_t n, float* sift, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    int64_t blocks = (n + kWarps - 1) / kWarps;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (blocks > cap) blocks = cap;
    ProfScope ps("sift", s);
    sift_kernel<<<(unsigned)blocks, kWarps * 32, 0, s>>>(patches, n, sift);
    return cudaGetLastError();
}

}  // namespace bd
