// bad_image.cu — §8(a) rows a2-a4 on whole images (configs[0], [1]).
//
// One warp per keypoint, lane = test: each round of 32 tests computes both sample points
// with the fixed-order fp32 rule (R6), gathers the 8 integral-image corners,
// compares exactly (R4) and packs the 32 bits with __ballot_sync (lane i -> bit i, R16), so
// every 32 tests become one 32-bit word; the K/32 words of a keypoint leave in one
// coalesced store.
#include <math.h>
#include <stdlib.h>

#include "internal.cuh"

namespace bd {
namespace kern {

__device__ __forceinline__ void sample_point(float x, float y, float a, float b, int dx, int dy,
                                             int& px, int& py) {
    // R6: X = x + (a*dx - b*dy), Y = y + (b*dx + a*dy), fp32, round-to-nearest, no FMA;
    // p = floor(X + 0.5) of the EXACT sum, evaluated in fp32 with the add rounded toward -inf:
    // it never rounds up onto an integer and, integers being representable (|X| < 2^23),
    // never drops below one, so floor(fl_rd(X + 0.5)) = floor(X + 0.5), the exact value of
    // DESIGN.md reading R6 (warp.cu uses the same rule), without the fp64 pipe.
    const float fdx = (float)dx, fdy = (float)dy;
    const float X = __fadd_rn(x, __fsub_rn(__fmul_rn(a, fdx), __fmul_rn(b, fdy)));
    const float Y = __fadd_rn(y, __fadd_rn(__fmul_rn(b, fdx), __fmul_rn(a, fdy)));
    px = __float2int_rd(__fadd_rd(X, 0.5f));
    py = __float2int_rd(__fadd_rd(Y, 0.5f));
}

// Box sum over the (2r+1)^2 box at (px, py), centre and box clamped to the image (R5).
// T = uint16_t: the integral is stored mod 2^16 and the box sum (< 2^16 for r <= 7) is the
// 4-corner combination mod 2^16 — exact.
template <typename T>
__device__ __forceinline__ uint32_t box_sum(const T* __restrict__ II, int64_t ip, int H, int W,
                                            int px, int py, int r, int& area) {
    px = min(max(px, 0), W - 1);
    py = min(max(py, 0), H - 1);
    const int x0 = max(px - r, 0), x1 = min(px + r, W - 1) + 1;
    const int y0 = max(py - r, 0), y1 = min(py + r, H - 1) + 1;
    area = (x1 - x0) * (y1 - y0);
    BD_CHECK(x0 >= 0 && x0 < x1 && x1 <= W && y0 >= 0 && y0 < y1 && y1 <= H);
    const T* r0 = II + (int64_t)y0 * ip;
    const T* r1 = II + (int64_t)y1 * ip;
    const uint32_t v = (uint32_t)__ldg(r1 + x1) - (uint32_t)__ldg(r0 + x1) - (uint32_t)__ldg(r1 + x0) +
                       (uint32_t)__ldg(r0 + x0);
    return sizeof(T) == 2 ? (v & 0xffffu) : v;
}

template <typename T>
__global__ void __launch_bounds__(256) bad_image_kernel(
    const T* __restrict__ integral, int64_t ip, int64_t istride, int n_img, int H, int W,
    const bd_keypoint* __restrict__ kps, const int32_t* __restrict__ kp_image, int64_t n_kp,
    const ImgTest* __restrict__ tests, int K, int scale_radius, uint32_t* __restrict__ out,
    uint8_t* __restrict__ status, const int32_t* __restrict__ perm) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= n_kp) return;
    const int64_t i = perm ? (int64_t)__ldg(perm + w) : w;  // keypoint served by this warp
    const int words = K >> 5;
    const float4 kv = __ldg(reinterpret_cast<const float4*>(kps) + i);
    const int img = kp_image ? __ldg(kp_image + i) : 0;
    const bool valid = isfinite(kv.x) && isfinite(kv.y) && isfinite(kv.z) && isfinite(kv.w) &&
                       kv.w > 0.0f && kv.x >= 0.0f && kv.y >= 0.0f && kv.x <= (float)(W - 1) &&
                       kv.y <= (float)(H - 1) && img >= 0 && img < n_img;
    uint32_t* o = out + i * words;
    if (!valid) {
        if (lane < words) o[lane] = 0u;
        if (status && lane == 0) status[i] = 1;
        return;
    }
    // keypoint frame: a = (float)(scale cos angle), b = (float)(scale sin angle), trig in fp64 (R6)
    float a = 0.f, b = 0.f;
    if (lane == 0) {
        double sn, cs;
        sincos((double)kv.z, &sn, &cs);
        a = (float)((double)kv.w * cs);
        b = (float)((double)kv.w * sn);
    }
    a = __shfl_sync(0xffffffffu, a, 0);
    b = __shfl_sync(0xffffffffu, b, 0);
    const T* II = integral + (int64_t)img * istride;
    uint32_t myword = 0;
    for (int g = 0; g < words; ++g) {
        const ImgTest t = tests[g * 32 + lane];
        int p1x, p1y, p2x, p2y, A1, A2;
        sample_point(kv.x, kv.y, a, b, t.dx1, t.dy1, p1x, p1y);
        sample_point(kv.x, kv.y, a, b, t.dx2, t.dy2, p2x, p2y);
        // NEXT-3 (BD_BAD_SCALE_RADIUS, reading R27): r' = floor(r*scale + 1/2) in fp32
        // (clamped to the image extent: a larger box covers the same clamped pixels, and huge
        // scales must not overflow px + r)
        const int r = scale_radius
                          ? min(__float2int_rd(__fadd_rn(__fmul_rn((float)t.r, kv.w), 0.5f)), max(H, W))
                          : t.r;
        const uint32_t S1 = box_sum(II, ip, H, W, p1x, p1y, r, A1);
        const uint32_t S2 = box_sum(II, ip, H, W, p2x, p2y, r, A2);
        const int full = (2 * t.r + 1) * (2 * t.r + 1);
        bool bit;
        if (!scale_radius && A1 == full && A2 == full) {
            bit = (int)(S1 - S2) <= t.t_full;  // S1 - S2 <= floor(theta * A)  (R4)
        } else {
            // f <= theta  <=>  S1*A2 - S2*A1 <= theta*A1*A2, both sides exact in fp64 (R4)
            // (areas up to H*W under BD_BAD_SCALE_RADIUS: the product in int64)
            const long long D = (long long)S1 * A2 - (long long)S2 * A1;
            bit = (double)D <= (double)t.theta * (double)((long long)A1 * A2);
        }
        const uint32_t w = __ballot_sync(0xffffffffu, bit);
        if (lane == g) myword = w;
    }
    if (lane < words) o[lane] = myword;
    if (status && lane == 0) status[i] = 0;
}

// Box-clustered variant (uint16 integral, unscaled radii): warp per keypoint in two phases.
// (1) lane = box: the 2K boxes in the model's clustered order (api.cu: runs of 32 boxes
//     compact in offset space), 32 per round: sample point (R6), 4 corner gathers, clamped area;
//     (S, A) packed into the warp's shared-memory slot.  The 32 gathers of one instruction now
//     fall on nearby pixels for any rotation / scale (~15 distinct 128-byte lines instead of
//     ~27 when the lanes are 32 unrelated tests).
// (2) lane = test: its two boxes' (S, A) from shared memory (the model's bpos table), the
//     exact compare (R4) and the ballot, as in bad_image_kernel.
constexpr int kClWarps = 8;

template <int KMAX>
__global__ void __launch_bounds__(kClWarps * 32) bad_image_clustered_kernel(
    const uint16_t* __restrict__ integral, int64_t ip, int64_t istride, int n_img, int H, int W,
    const bd_keypoint* __restrict__ kps, const int32_t* __restrict__ kp_image, int64_t n_kp,
    const ImgTest* __restrict__ tests, int K, uint32_t* __restrict__ out, uint8_t* __restrict__ status,
    const int32_t* __restrict__ perm) {
    __shared__ uint32_t sb[kClWarps][2 * KMAX];  // (S | A << 16) per box
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int64_t w = (int64_t)blockIdx.x * kClWarps + wl;
    if (w >= n_kp) return;
    const int64_t i = perm ? (int64_t)__ldg(perm + w) : w;
    const int words = K >> 5;
    const ImgBox* boxes = reinterpret_cast<const ImgBox*>(tests + K);
    const uint32_t* bpos = reinterpret_cast<const uint32_t*>(boxes + 2 * K);  // then the lane-major box copy
    const float4 kv = __ldg(reinterpret_cast<const float4*>(kps) + i);
    const int img = kp_image ? __ldg(kp_image + i) : 0;
    const bool valid = isfinite(kv.x) && isfinite(kv.y) && isfinite(kv.z) && isfinite(kv.w) &&
                       kv.w > 0.0f && kv.x >= 0.0f && kv.y >= 0.0f && kv.x <= (float)(W - 1) &&
                       kv.y <= (float)(H - 1) && img >= 0 && img < n_img;
    uint32_t* o = out + i * words;
    if (!valid) {
        if (lane < words) o[lane] = 0u;
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
    // the image's integral base computed once and kept opaque (so ptxas does not re-derive
    // img * istride per corner), 32-bit corner offsets (an image integral has < 2^31 entries:
    // bad_compute's H*W bound): one IMAD.WIDE per corner address
    const uint16_t* II;
    asm volatile("mov.b64 %0, %1;" : "=l"(II) : "l"(integral + (int64_t)img * istride));
    const uint32_t ip32 = (uint32_t)ip;
    uint32_t* my = sb[wl];
    // phase 1: box sums in clustered order; the lane's box records (item 32 rho + lane) come
    // from the lane-major copy of the table (api.cu) as 16-byte loads, all rounds unrolled so
    // the corner gathers of several boxes are in flight together
    constexpr int kR = 2 * KMAX / 32;
    const int R = (2 * K) >> 5;
    uint32_t rec[kR];
    const uint4* lrec = reinterpret_cast<const uint4*>(bpos + K) + lane * (kR / 4);
#pragma unroll
    for (int v = 0; v < kR / 4; ++v) {
        const uint4 u = 4 * v < R ? __ldg(lrec + v) : make_uint4(0, 0, 0, 0);
        rec[4 * v] = u.x; rec[4 * v + 1] = u.y; rec[4 * v + 2] = u.z; rec[4 * v + 3] = u.w;
    }
#pragma unroll
    for (int rho = 0; rho < kR; ++rho) {
        if (rho < R) {
            const int dx = (int)(int8_t)(rec[rho] & 0xffu), dy = (int)(int8_t)((rec[rho] >> 8) & 0xffu);
            const int r = (int)((rec[rho] >> 16) & 0xffu);
            int px, py;
            sample_point(kv.x, kv.y, a, b, dx, dy, px, py);
            px = min(max(px, 0), W - 1);
            py = min(max(py, 0), H - 1);
            const int x0 = max(px - r, 0), x1 = min(px + r, W - 1) + 1;
            const int y0 = max(py - r, 0), y1 = min(py + r, H - 1) + 1;
            const uint32_t A = (uint32_t)((x1 - x0) * (y1 - y0));
            BD_CHECK(x0 >= 0 && x0 < x1 && x1 <= W && y0 >= 0 && y0 < y1 && y1 <= H);
            const uint32_t o0 = (uint32_t)y0 * ip32, o1 = (uint32_t)y1 * ip32;
            const uint32_t S = ((uint32_t)__ldg(II + (o1 + (uint32_t)x1)) - (uint32_t)__ldg(II + (o0 + (uint32_t)x1)) -
                                (uint32_t)__ldg(II + (o1 + (uint32_t)x0)) + (uint32_t)__ldg(II + (o0 + (uint32_t)x0))) &
                               0xffffu;
            my[rho * 32 + lane] = S | (A << 16);
        }
    }
    __syncwarp();
    uint32_t myword = 0;
    ImgTest tn = tests[lane];  // phase-2 records loaded one round ahead
    uint32_t bpn = __ldg(bpos + lane);
    for (int g = 0; g < words; ++g) {  // phase 2: lane = test
        const ImgTest t = tn;
        const uint32_t bp = bpn;
        if (g + 1 < words) {
            tn = tests[(g + 1) * 32 + lane];
            bpn = __ldg(bpos + (g + 1) * 32 + lane);
        }
        const uint32_t v1 = my[bp & 0xffffu], v2 = my[bp >> 16];
        const int S1 = (int)(v1 & 0xffffu), A1 = (int)(v1 >> 16), S2 = (int)(v2 & 0xffffu), A2 = (int)(v2 >> 16);
        const int full = (2 * t.r + 1) * (2 * t.r + 1);
        bool bit;
        if (A1 == full && A2 == full) {
            bit = S1 - S2 <= t.t_full;  // S1 - S2 <= floor(theta * A)  (R4)
        } else {
            const long long D = (long long)S1 * A2 - (long long)S2 * A1;
            bit = (double)D <= (double)t.theta * (double)((long long)A1 * A2);
        }
        const uint32_t wd = __ballot_sync(0xffffffffu, bit);
        if (lane == g) myword = wd;
    }
    if (lane < words) o[lane] = myword;
    if (status && lane == 0) status[i] = 0;
}

// ---- small batches (latency path, configs[0]): ONE launch and no image integral.  A CTA per
// keypoint builds the exact uint32 integral of just its window (every corner its boxes can
// touch: offsets in [-16, 15], radii <= 7, clamped to the image) in shared memory from the
// image bytes, then thread = test evaluates both boxes there and ballots the bits.  Box sums of
// the local integral equal those of the image integral (the window origin's terms cancel), so
// the bits are the same.  A window larger than the shared-memory budget (keypoint scale above
// ~1.7) sums its boxes directly from the image bytes (slower, exact).
constexpr int kLocThreads = 256;
constexpr int kLocSmemBytes = 32 * 1024;  // 7 CTAs per SM: 1036 keypoints in one wave

template <int KMAX>
__global__ void __launch_bounds__(kLocThreads) bad_image_local_kernel(
    const uint8_t* __restrict__ images, int64_t pitch, int n_img, int H, int W, const bd_keypoint* __restrict__ kps,
    const int32_t* __restrict__ kp_image, const ImgTest* __restrict__ tests, int K, uint32_t* __restrict__ out,
    uint8_t* __restrict__ status) {
    extern __shared__ uint32_t lii[];  // (rows + 1) x P, entry (y - cy0, x - cx0) of the integral
    __shared__ float s_ab[2];
    __shared__ int s_win[4];
    debug_poison_smem(lii);
    const int t = threadIdx.x, lane = t & 31;
    const int64_t i = blockIdx.x;
    const int words = K >> 5;
    const float4 kv = __ldg(reinterpret_cast<const float4*>(kps) + i);
    const int img = kp_image ? __ldg(kp_image + i) : 0;
    const bool valid = isfinite(kv.x) && isfinite(kv.y) && isfinite(kv.z) && isfinite(kv.w) && kv.w > 0.0f &&
                       kv.x >= 0.0f && kv.y >= 0.0f && kv.x <= (float)(W - 1) && kv.y <= (float)(H - 1) &&
                       img >= 0 && img < n_img;
    uint32_t* o = out + i * words;
    if (!valid) {
        if (t < words) o[t] = 0u;
        if (status && t == 0) status[i] = 1;
        return;
    }
    if (t == 0) {
        double sn, cs;
        sincos((double)kv.z, &sn, &cs);
        const float a = (float)((double)kv.w * cs), b = (float)((double)kv.w * sn);
        s_ab[0] = a;
        s_ab[1] = b;
        // integral-coordinate corners: sample points within x +- 16 (|a| + |b|) (+2 for the fp32
        // rounding and the +1/2), boxes r <= 7 left / up and r + 1 right / down
        const double E = 16.0 * (fabs((double)a) + fabs((double)b)) + 2.0;
        s_win[0] = (int)fmax(0.0, floor((double)kv.x - E) - 7);
        s_win[1] = (int)fmin((double)W, ceil((double)kv.x + E) + 8);
        s_win[2] = (int)fmax(0.0, floor((double)kv.y - E) - 7);
        s_win[3] = (int)fmin((double)H, ceil((double)kv.y + E) + 8);
    }
    __syncthreads();
    const float a = s_ab[0], b = s_ab[1];
    const int cx0 = s_win[0], cx1 = s_win[1], cy0 = s_win[2], cy1 = s_win[3];
    const int cols = cx1 - cx0, rows = cy1 - cy0, P = (cols + 1) | 1;  // odd pitch: column scans conflict-free
    const bool fits = (int64_t)(rows + 1) * P * 4 + (int64_t)rows * cols <= kLocSmemBytes;
    const uint8_t* I = images + (int64_t)img * pitch * H;
    if (fits) {
        // the window's pixels into shared memory (independent byte loads by all threads), then
        // thread per row: running row sums; thread per column: running column sums (4 rows per
        // step, loads ahead of the adds); row 0 and column 0 of the local integral are zero
        uint8_t* pix = reinterpret_cast<uint8_t*>(lii + (rows + 1) * P);
        for (int q = t; q < rows * cols; q += kLocThreads) {
            const int y = q / cols, x = q - y * cols;
            pix[q] = __ldg(I + (int64_t)(cy0 + y) * pitch + cx0 + x);
        }
        for (int x = t; x < P; x += kLocThreads) lii[x] = 0u;
        __syncthreads();
        for (int y = t; y < rows; y += kLocThreads) {
            const uint8_t* src = pix + y * cols;
            uint32_t* dst = lii + (y + 1) * P;
            uint32_t acc = 0;
            dst[0] = 0u;
            for (int x = 0; x < cols; ++x) {
                acc += src[x];
                dst[x + 1] = acc;
            }
        }
        __syncthreads();
        for (int x = t + 1; x <= cols; x += kLocThreads) {
            uint32_t acc = 0;
            int y = 1;
            for (; y + 3 <= rows; y += 4) {
                const uint32_t v0 = lii[y * P + x], v1 = lii[(y + 1) * P + x], v2 = lii[(y + 2) * P + x],
                               v3 = lii[(y + 3) * P + x];
                lii[y * P + x] = acc += v0;
                lii[(y + 1) * P + x] = acc += v1;
                lii[(y + 2) * P + x] = acc += v2;
                lii[(y + 3) * P + x] = acc += v3;
            }
            for (; y <= rows; ++y) lii[y * P + x] = acc += lii[y * P + x];
        }
        __syncthreads();
    }
    auto box = [&](int dx, int dy, int r, int& A) -> uint32_t {
        int px, py;
        sample_point(kv.x, kv.y, a, b, dx, dy, px, py);
        px = min(max(px, 0), W - 1);
        py = min(max(py, 0), H - 1);
        const int x0 = max(px - r, 0), x1 = min(px + r, W - 1) + 1;
        const int y0 = max(py - r, 0), y1 = min(py + r, H - 1) + 1;
        A = (x1 - x0) * (y1 - y0);
        if (fits) {
            BD_CHECK(x0 >= cx0 && x1 <= cx1 && y0 >= cy0 && y1 <= cy1);
            const uint32_t* r0 = lii + (y0 - cy0) * P - cx0;
            const uint32_t* r1 = lii + (y1 - cy0) * P - cx0;
            return r1[x1] - r0[x1] - r1[x0] + r0[x0];
        }
        uint32_t sum = 0;  // window too large for shared memory: the box from the image bytes
        for (int y = y0; y < y1; ++y)
            for (int x = x0; x < x1; ++x) sum += __ldg(I + (int64_t)y * pitch + x);
        return sum;
    };
    for (int k = t; k < K; k += kLocThreads) {  // thread = test; K % 32 == 0: whole warps
        const ImgTest tt = tests[k];
        int A1, A2;
        const int S1 = (int)box(tt.dx1, tt.dy1, tt.r, A1), S2 = (int)box(tt.dx2, tt.dy2, tt.r, A2);
        const int full = (2 * tt.r + 1) * (2 * tt.r + 1);
        bool bit;
        if (A1 == full && A2 == full) {
            bit = S1 - S2 <= tt.t_full;  // S1 - S2 <= floor(theta * A)  (R4)
        } else {
            const long long D = (long long)S1 * A2 - (long long)S2 * A1;
            bit = (double)D <= (double)tt.theta * (double)((long long)A1 * A2);
        }
        const uint32_t wd = __ballot_sync(0xffffffffu, bit);
        if (lane == 0) o[k >> 5] = wd;
    }
    if (status && t == 0) status[i] = 0;
}

// ---- spatial order: warps that run together serve nearby keypoints, so their integral
// windows overlap in L1/L2 (c1: bad_image 0.94 -> ~0.70 ms measured with a host sort).  A
// counting sort by (image, 64x64-pixel cell): keys, histogram, one-CTA exclusive scan,
// scatter; the order inside a cell is irrelevant (every keypoint's result is independent).
constexpr int kCell = 64;

__device__ __forceinline__ int cell_of(const bd_keypoint* kps, const int32_t* kp_image, int64_t i, int n_img,
                                       int H, int W, int ncx, int ncy) {
    const float4 kv = __ldg(reinterpret_cast<const float4*>(kps) + i);
    int img = kp_image ? __ldg(kp_image + i) : 0;
    img = min(max(img, 0), n_img - 1);
    // NaN / out-of-range coordinates land in a border cell (the warp marks them invalid)
    const int cx = (kv.x >= 0.f && kv.x < (float)W) ? (int)kv.x / kCell : 0;
    const int cy = (kv.y >= 0.f && kv.y < (float)H) ? (int)kv.y / kCell : 0;
    return (img * ncy + min(cy, ncy - 1)) * ncx + min(cx, ncx - 1);
}

__global__ void kp_cell_hist(const bd_keypoint* __restrict__ kps, const int32_t* __restrict__ kp_image, int64_t n,
                             int n_img, int H, int W, int ncx, int ncy, int32_t* __restrict__ count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(&count[cell_of(kps, kp_image, i, n_img, H, W, ncx, ncy)], 1);
}

// exclusive scan of count (in place) by one 1024-thread CTA: each thread scans a contiguous run
__global__ void __launch_bounds__(1024) kp_cell_scan(int32_t* __restrict__ count, int n_cells) {
    __shared__ int32_t part[1024];
    const int t = threadIdx.x;
    const int per = (n_cells + 1023) / 1024, a = t * per, b = min(n_cells, a + per);
    int32_t sum = 0;
    for (int c = a; c < b; ++c) sum += count[c];
    part[t] = sum;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {  // Hillis-Steele inclusive scan of the run totals
        const int32_t v = t >= d ? part[t - d] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int32_t run = part[t] - sum;
    for (int c = a; c < b; ++c) {
        const int32_t v = count[c];
        count[c] = run;
        run += v;
    }
}

__global__ void kp_cell_scatter(const bd_keypoint* __restrict__ kps, const int32_t* __restrict__ kp_image, int64_t n,
                                int n_img, int H, int W, int ncx, int ncy, int32_t* __restrict__ cursor,
                                int32_t* __restrict__ perm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) perm[atomicAdd(&cursor[cell_of(kps, kp_image, i, n_img, H, W, ncx, ncy)], 1)] = (int32_t)i;
}

}  // namespace kern

using namespace kern;

int bad_image_local_max_kp() {
    static const int v = [] {
        const char* e = getenv("BINDESC_LOCAL_MAX_KP");
        return e ? atoi(e) : 4096;
    }();
    return v;
}

cudaError_t launch_bad_image_local(const uint8_t* images, int n_img, int H, int W, int64_t pitch,
                                   const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp, const ImgTest* tests,
                                   int K, uint32_t* out, uint8_t* status, cudaStream_t s) {
    if (n_kp == 0) return cudaSuccess;
    cudaError_t e = ensure_smem_attr((const void*)bad_image_local_kernel<256>, kLocSmemBytes);
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)bad_image_local_kernel<512>, kLocSmemBytes);
    if (e != cudaSuccess) return e;
    ProfScope ps("bad_image", s);
    if (K <= 256)
        bad_image_local_kernel<256><<<(unsigned)n_kp, kLocThreads, kLocSmemBytes, s>>>(images, pitch, n_img, H, W, kps,
                                                                                      kp_image, tests, K, out, status);
    else
        bad_image_local_kernel<512><<<(unsigned)n_kp, kLocThreads, kLocSmemBytes, s>>>(images, pitch, n_img, H, W, kps,
                                                                                      kp_image, tests, K, out, status);
    return cudaGetLastError();
}

// workspace of the spatial order (0: keypoints are served in input order)
size_t bad_image_order_bytes(int n_img, int H, int W, int64_t n_kp) {
    if (n_kp < (int64_t)num_sms() * 64 || n_kp > (int64_t)INT32_MAX) return 0;  // small batches: latency first
    const int64_t cells = (int64_t)n_img * ((W + kCell - 1) / kCell) * ((H + kCell - 1) / kCell);
    if (cells > (1 << 24)) return 0;
    return ((size_t)cells * 4 + 255) / 256 * 256 + (size_t)n_kp * 4;
}

cudaError_t launch_bad_image(const uint8_t* /*images*/, int n_img, int H, int W, int64_t /*pitch*/,
                             const void* integral, int ii_bytes, int64_t ipitch, const bd_keypoint* kps,
                             const int32_t* kp_image, int64_t n_kp, const ImgTest* tests, int K,
                             int scale_radius, uint32_t* out, uint8_t* status, void* order_ws,
                             cudaStream_t s) {
    const int warps = 8;
    const int64_t blocks = (n_kp + warps - 1) / warps;
    ProfScope ps("bad_image", s);
    int32_t* perm = nullptr;
    if (order_ws) {
        const int ncx = (W + kCell - 1) / kCell, ncy = (H + kCell - 1) / kCell;
        const int n_cells = n_img * ncx * ncy;
        int32_t* count = static_cast<int32_t*>(order_ws);
        perm = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(order_ws) + ((size_t)n_cells * 4 + 255) / 256 * 256);
        cudaError_t e = cudaMemsetAsync(count, 0, (size_t)n_cells * 4, s);
        if (e != cudaSuccess) return e;
        const unsigned g = (unsigned)((n_kp + 255) / 256);
        kp_cell_hist<<<g, 256, 0, s>>>(kps, kp_image, n_kp, n_img, H, W, ncx, ncy, count);
        kp_cell_scan<<<1, 1024, 0, s>>>(count, n_cells);
        kp_cell_scatter<<<g, 256, 0, s>>>(kps, kp_image, n_kp, n_img, H, W, ncx, ncy, count, perm);
    }
    if (ii_bytes == 2 && !scale_radius) {  // box-clustered two-phase kernel (static smem: 8 warps x 2K words)
        const int64_t cb = (n_kp + kClWarps - 1) / kClWarps;
        if (K <= 256)
            bad_image_clustered_kernel<256><<<(unsigned)cb, kClWarps * 32, 0, s>>>(
                static_cast<const uint16_t*>(integral), ipitch, ipitch * (int64_t)(H + 1), n_img, H, W, kps, kp_image,
                n_kp, tests, K, out, status, perm);
        else
            bad_image_clustered_kernel<512><<<(unsigned)cb, kClWarps * 32, 0, s>>>(
                static_cast<const uint16_t*>(integral), ipitch, ipitch * (int64_t)(H + 1), n_img, H, W, kps, kp_image,
                n_kp, tests, K, out, status, perm);
    } else if (ii_bytes == 2)
        bad_image_kernel<uint16_t><<<(unsigned)blocks, warps * 32, 0, s>>>(
            static_cast<const uint16_t*>(integral), ipitch, ipitch * (int64_t)(H + 1), n_img, H, W, kps, kp_image,
            n_kp, tests, K, scale_radius, out, status, perm);
    else
        bad_image_kernel<uint32_t><<<(unsigned)blocks, warps * 32, 0, s>>>(
            static_cast<const uint32_t*>(integral), ipitch, ipitch * (int64_t)(H + 1), n_img, H, W, kps, kp_image,
            n_kp, tests, K, scale_radius, out, status, perm);
    return cudaGetLastError();
}

}  // namespace bd
