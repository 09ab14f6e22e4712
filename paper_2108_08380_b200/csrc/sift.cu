// sift.cu — §8(a) rows a6-a8: SIFT 4x4x8 histogram of a normalised 32x32 patch
// ("the vector of real valued features provided by SIFT"; conventions R10).
//
// One warp per patch, lane = pixel column x; the warp walks the 32 rows.  BJ.ns (3):
// "fuses the gradient and orientation binning with a warp-level histogram reduction".
// Per pixel (instruction diet):
//  * gx, gy: the lane keeps column pixels of rows y-1, y, y+1 in registers; x-1, x+1 come by
//    shuffle (replicate border);
//  * m = sqrt(gx^2+gy^2) by MUFU rsqrt; the orientation in units of 45 degrees,
//    co = atan2(gy, gx) * 4/pi in [0, 8), by octant reduction: r = min/max (MUFU rcp),
//    atan(r)*4/pi by a degree-11 odd polynomial (|err| < 2.3e-6 bin), then 3 reflections;
//  * trilinear binning: the pixel adds m*g(x)g(y)*(1-fy or fy)*(1-fo or fo) to orientation
//    bins o0, o0+1 of cell rows j0, j0+1 in a per-lane PRIVATE 2x9-bin histogram in shared
//    memory (layout [row][bin][lane]: bank = lane, conflict-free whatever o0 is; bin 8 is
//    the wrap of bin 0);
//  * when the walk leaves cell row j0 (after y = 11, 19, 27, 31) the private row is folded
//    (bin 8 -> 0) and reduced across lanes with the spatial x-weights 1 - |k - 7.5|/8
//    through a 33-word-padded transpose (conflict-free), landing in lane (i, o) = (L/8, L%8);
//  * the 4 registers per lane are the 128 entries j*32 + L: L2-normalise, clip at 0.2,
//    renormalise (zero stays zero) with two warp all-reductions.
#include <math.h>

#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kWarps = 8;
constexpr int kBins = 9;                 // 8 orientation bins + wrap
constexpr int kPriv = 2 * kBins * 32;    // floats: [row a/b][bin][lane]
constexpr int kScr = 8 * 33;             // floats: [o][x] padded

// g(y) (1 - fy) and g(y) fy per row y, g(t) = exp(-(t-15.5)^2 / 512), fy = frac((y-3.5)/8)
__constant__ float c_gy[32][2];

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// fold the private row (bins 0..8, bin 8 -> 0) and zero it, transpose through scr, reduce
// with the spatial x-weights: lane L gets cell (i = L/8, o = L%8) of this cell row.
__device__ __forceinline__ float flush_row(float* row, float* scr, int lane) {
    float h[kBins];
#pragma unroll
    for (int o = 0; o < kBins; ++o) {
        h[o] = row[o * 32 + lane];
        row[o * 32 + lane] = 0.f;
    }
    h[0] += h[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) scr[o * 33 + lane] = h[o];
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
    __shared__ float s_priv[kWarps][kPriv];
    __shared__ float s_scr[kWarps][kScr];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* P = s_patch[warp];
    float* priv = s_priv[warp];
    float* scr = s_scr[warp];
#pragma unroll
    for (int o = 0; o < 2 * kBins; ++o) priv[o * 32 + lane] = 0.f;
    const float gxw = expf(-((float)lane - 15.5f) * ((float)lane - 15.5f) / 512.0f);
    const int xl = lane > 0 ? lane - 1 : 0, xr = lane < 31 ? lane + 1 : 31;
    float* const rowA = priv;               // the two private cell-row histograms
    float* const rowB = priv + kBins * 32;
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    for (int64_t p = (int64_t)blockIdx.x * kWarps + warp; p < n; p += nwarps) {
        const uint4* src = reinterpret_cast<const uint4*>(patches + p * 1024);
        const uint4 q0 = __ldg(src + lane), q1 = __ldg(src + 32 + lane);
        __syncwarp();
        reinterpret_cast<uint4*>(P)[lane] = q0;
        reinterpret_cast<uint4*>(P)[32 + lane] = q1;
        __syncwarp();
        float h0 = 0.f, h1 = 0.f, h2 = 0.f, h3 = 0.f;
        float prev = (float)P[lane], cur = prev;
#pragma unroll
        for (int y = 0; y < 32; ++y) {
            const float next = (float)P[(y < 31 ? y + 1 : 31) * 32 + lane];
            const float left = __shfl_sync(0xffffffffu, cur, xl);
            const float right = __shfl_sync(0xffffffffu, cur, xr);
            const float gx = right - left, gy = next - prev;
            const float ax = fabsf(gx), ay = fabsf(gy);
            const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
            const float m2 = fmaf(gx, gx, gy * gy);
            const float m = m2 * rsqrt_approx(fmaxf(m2, 1e-30f));
            const float r = mn * rcp_approx(fmaxf(mx, 1e-30f));
            const float s = r * r;
            float a = fmaf(s, -0.014921262860298157f, 0.06703268736600876f);
            a = fmaf(s, a, -0.14823880791664124f);
            a = fmaf(s, a, 0.24642325937747955f);
            a = fmaf(s, a, -0.42350855469703674f);
            a = fmaf(s, a, 1.2732105255126953f);
            a *= r;                                   // atan(r) * 4/pi in [0, 1]
            float co = (ay > ax) ? 2.0f - a : a;      // reflections: first octant -> [0, 8)
            co = (gx < 0.f) ? 4.0f - co : co;
            co = (gy < 0.f) ? 8.0f - co : co;
            const float fl = floorf(co);
            const float fo = co - fl;
            const int o0 = (int)fl;
            const float mg = m * gxw;
            // cell rows: j0 = floor((y - 3.5)/8); bands [0,4) [4,12) [12,20) [20,28) [28,32);
            // the band index parity decides which private buffer holds row j0 (compile time)
            const int j0 = (y < 4) ? -1 : (y - 4) / 8;
            float* ra = ((j0 + 1) & 1) ? rowB : rowA;   // row j0
            float* rb = ((j0 + 1) & 1) ? rowA : rowB;   // row j0 + 1
            if (j0 >= 0) {
                const float wa = mg * c_gy[y][0];
                float* q = ra + o0 * 32 + lane;
                const float t0 = q[0], t1 = q[32];
                q[0] = fmaf(wa, 1.0f - fo, t0);
                q[32] = fmaf(wa, fo, t1);
            }
            if (j0 + 1 <= 3) {
                const float wb = mg * c_gy[y][1];
                float* q = rb + o0 * 32 + lane;
                const float t0 = q[0], t1 = q[32];
                q[0] = fmaf(wb, 1.0f - fo, t0);
                q[32] = fmaf(wb, fo, t1);
            }
            prev = cur;
            cur = next;
            if (j0 >= 0 && (y == 11 || y == 19 || y == 27 || y == 31)) {
                const float sres = flush_row(ra, scr, lane);  // row j0 complete; zeroed for reuse
                if (j0 == 0) h0 = sres;
                if (j0 == 1) h1 = sres;
                if (j0 == 2) h2 = sres;
                if (j0 == 3) h3 = sres;
            }
        }
        // normalise, clip 0.2, renormalise (R10); the zero histogram stays zero
        const float n2 = warp_sum(h0 * h0 + h1 * h1 + h2 * h2 + h3 * h3);
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
    }
}

}  // namespace kern

using namespace kern;
cudaError_t launch_sift(const uint8_t* patches, int64_t n, float* sift, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    static bool init = false;
    if (!init) {
        float t[32][2];
        for (int y = 0; y < 32; ++y) {
            const double g = exp(-((y - 15.5) * (y - 15.5)) / 512.0);
            const double cy = (y - 3.5) / 8.0;
            const double fy = cy - floor(cy);
            t[y][0] = (float)(g * (1.0 - fy));
            t[y][1] = (float)(g * fy);
        }
        cudaError_t e = cudaMemcpyToSymbol(c_gy, t, sizeof t);
        if (e != cudaSuccess) return e;
        init = true;
    }
    int64_t blocks = (n + kWarps - 1) / kWarps;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    ProfScope ps("sift", s);
    sift_kernel<<<(unsigned)blocks, kWarps * 32, 0, s>>>(patches, n, sift);
    return cudaGetLastError();
}

}  // namespace bd
