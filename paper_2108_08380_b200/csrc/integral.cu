// integral.cu — §8(a) row a1: integral image II(r, c) = sum_{y<r, x<c} I(y, x)
// ("efficiently computed using integral images").
//
// Two HBM passes over uint32 (sums < 2^32 for H*W*255 < 2^32), both fully coalesced
// (DESIGN.md §5.1):
//   1. column pass: one thread per image column walks down the rows with a register running
//      sum, 8 rows of independent byte loads in flight per thread, and writes the vertical
//      prefix V(y, x) = sum_{y' <= y} I(y', x) to II(y+1, x+1) (row/column 0 of II are
//      written as zeros here too);
//   2. row pass (BJ.ns (1): "warp-shuffle row scans"): one warp per row, 32 consecutive
//      entries per step, a 5-step shuffle inclusive scan plus a running carry, in place.
// 13 B/px of HBM traffic (1 read + 4 write, 4 read + 4 write).
#include <algorithm>

#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kColThreads = 128;
constexpr int kRowWarps = 8;

template <typename T>
__global__ void __launch_bounds__(kColThreads) integral_cols_kernel(const uint8_t* __restrict__ img, int H, int W,
                                                                    int64_t pitch, int64_t img_stride,
                                                                    T* __restrict__ out, int64_t op,
                                                                    int64_t out_stride) {
    const int x = blockIdx.x * kColThreads + threadIdx.x;
    if (x > W) return;
    T* o = out + (int64_t)blockIdx.y * out_stride;
    if (x == W) {  // column 0 of II (one thread per image)
        for (int r = 0; r <= H; ++r) o[(int64_t)r * op] = 0u;
        return;
    }
    const uint8_t* src = img + (int64_t)blockIdx.y * img_stride + x;
    T* dst = o + x + 1;
    dst[0] = 0u;  // row 0
    uint32_t acc = 0;
    int y = 0;
    for (; y + 8 <= H; y += 8) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(src + (int64_t)(y + k) * pitch);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc += v[k];
            dst[(int64_t)(y + k + 1) * op] = (T)acc;
        }
    }
    for (; y < H; ++y) {
        acc += __ldg(src + (int64_t)y * pitch);
        dst[(int64_t)(y + 1) * op] = (T)acc;
    }
}

template <typename T>
__global__ void __launch_bounds__(kRowWarps * 32) integral_rows_kernel(int H, int W, T* __restrict__ out,
                                                                       int64_t op, int64_t out_stride) {
    const int lane = threadIdx.x & 31;
    const int y = blockIdx.x * kRowWarps + (threadIdx.x >> 5) + 1;  // rows 1..H
    if (y > H) return;
    T* row = out + (int64_t)blockIdx.y * out_stride + (int64_t)y * op + 1;
    uint32_t carry = 0;
    for (int x0 = 0; x0 < W; x0 += 32) {
        const int x = x0 + lane;
        uint32_t v = x < W ? row[x] : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += t;
        }
        if (x < W) row[x] = (T)(carry + v);
        carry += __shfl_sync(0xffffffffu, v, 31);
    }
}

// ---- small-image path (configs[0]: one 640x480 image): a thread per column has far too little
// parallelism (641 threads walking 480 rows is ~20 us of latency), so the column pass is split
// into row BANDS: (1) thread (x, band) writes the band-local vertical prefix and the band total,
// (2) thread per column turns the band totals into carries (exclusive prefix over bands),
// (3) the row pass adds the carry of the row's band before its shuffle scan.
template <typename T>
__global__ void __launch_bounds__(kColThreads) integral_cols_banded_kernel(const uint8_t* __restrict__ img, int H,
                                                                           int W, int64_t pitch, int64_t img_stride,
                                                                           T* __restrict__ out, int64_t op,
                                                                           int64_t out_stride, int R,
                                                                           uint32_t* __restrict__ tot, int nb) {
    const int x = blockIdx.x * kColThreads + threadIdx.x;
    const int b = blockIdx.y, i = blockIdx.z;
    if (x > W) return;
    T* o = out + (int64_t)i * out_stride;
    const int y0 = b * R, y1 = min(H, y0 + R);
    if (x == W) {  // column 0 of II
        for (int r = y0 + 1; r <= y1; ++r) o[(int64_t)r * op] = 0u;
        if (b == 0) o[0] = 0u;
        return;
    }
    if (b == 0) o[x + 1] = 0u;  // row 0
    const uint8_t* src = img + (int64_t)i * img_stride + x;
    uint32_t acc = 0;
    for (int y = y0; y < y1; ++y) {
        acc += __ldg(src + (int64_t)y * pitch);
        o[(int64_t)(y + 1) * op + x + 1] = (T)acc;
    }
    tot[((int64_t)i * nb + b) * W + x] = acc;
}

// one warp per column: lanes over bands, shuffle scan (a serial loop over bands would be a
// chain of dependent global round trips)
__global__ void integral_band_carry_kernel(uint32_t* __restrict__ tot, int W, int nb) {
    const int lane = threadIdx.x & 31;
    const int x = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (x >= W) return;
    uint32_t* t = tot + (int64_t)blockIdx.y * nb * W + x;
    uint32_t carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {  // in place: total -> exclusive carry
        const int b = b0 + lane;
        const uint32_t v = b < nb ? t[(int64_t)b * W] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += u;
        }
        if (b < nb) t[(int64_t)b * W] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

template <typename T>
__global__ void __launch_bounds__(kRowWarps * 32) integral_rows_banded_kernel(int H, int W, T* __restrict__ out,
                                                                              int64_t op, int64_t out_stride, int R,
                                                                              const uint32_t* __restrict__ carry_tab,
                                                                              int nb) {
    const int lane = threadIdx.x & 31;
    const int y = blockIdx.x * kRowWarps + (threadIdx.x >> 5) + 1;  // rows 1..H
    if (y > H) return;
    T* row = out + (int64_t)blockIdx.y * out_stride + (int64_t)y * op + 1;
    const uint32_t* cb = carry_tab + ((int64_t)blockIdx.y * nb + (y - 1) / R) * W;
    uint32_t carry = 0;
    for (int x0 = 0; x0 < W; x0 += 32) {
        const int x = x0 + lane;
        uint32_t v = x < W ? row[x] + cb[x] : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += t;
        }
        if (x < W) row[x] = (T)(carry + v);
        carry += __shfl_sync(0xffffffffu, v, 31);
    }
}

// ---- vectorised uint16 path (the integral inside bad_compute: W, pitch multiples of 8): three
// short kernels, 4 B/px of HBM traffic (pixels read twice, the integral written once) instead of
// 7 B/px for the column + row passes:
//   (A) band column totals: CTA (band of kBandRows rows, image), thread = 8 columns (8-byte
//       loads), sums its columns over the band;
//   (C) integral_band_carry_kernel: totals -> exclusive prefix over bands (the column prefix V
//       at each band's top row);
//   (B) CTA (band, image): thread = 8 columns, V of its columns in registers (start: the band
//       carry), per row: V += pixels, an in-thread prefix over its 8 columns, a block-wide
//       exclusive scan of the thread totals (warp shuffles + 8 warp totals in shared memory), one
//       16-byte store of the 8 uint16 integral entries.  The output is stored with its column 0 at
//       index 7 (row pitch a multiple of 8), so image columns 8t..8t+7 land 16-byte aligned.
constexpr int kBandRows = 32;
constexpr int kVecThreads = 256;

__global__ void __launch_bounds__(kVecThreads) integral16_band_totals(const uint8_t* __restrict__ img, int H, int W,
                                                                     int64_t pitch, int64_t img_stride,
                                                                     uint32_t* __restrict__ tot, int nb) {
    const int b = blockIdx.x, i = blockIdx.y;
    const int y0 = b * kBandRows, y1 = min(H, y0 + kBandRows);
    for (int x = 8 * threadIdx.x; x < W; x += 8 * kVecThreads) {
        const uint8_t* src = img + (int64_t)i * img_stride + x;
        uint32_t a[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        for (int y = y0; y < y1; ++y) {
            const uint2 w = __ldg(reinterpret_cast<const uint2*>(src + (int64_t)y * pitch));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                a[k] += (w.x >> (8 * k)) & 0xffu;
                a[k + 4] += (w.y >> (8 * k)) & 0xffu;
            }
        }
        uint4* t = reinterpret_cast<uint4*>(tot + ((int64_t)i * nb + b) * W + x);
        t[0] = make_uint4(a[0], a[1], a[2], a[3]);
        t[1] = make_uint4(a[4], a[5], a[6], a[7]);
    }
}

// (C) for the vectorised path: thread per column, the band totals of its column loaded 8 at a
// time (coalesced across the threads) and turned into exclusive carries in place
__global__ void __launch_bounds__(256) integral16_band_carry(uint32_t* __restrict__ tot, int W, int nb) {
    const int x = blockIdx.x * 256 + threadIdx.x;
    if (x >= W) return;
    uint32_t* t = tot + (int64_t)blockIdx.y * nb * W + x;
    uint32_t run = 0;
    for (int b0 = 0; b0 < nb; b0 += 8) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = b0 + k < nb ? t[(int64_t)(b0 + k) * W] : 0u;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (b0 + k < nb) t[(int64_t)(b0 + k) * W] = run;
            run += v[k];
        }
    }
}

__global__ void __launch_bounds__(kVecThreads) integral16_band_rows(const uint8_t* __restrict__ img, int H, int W,
                                                                   int64_t pitch, int64_t img_stride,
                                                                   uint16_t* __restrict__ out, int64_t op,
                                                                   int64_t out_stride,
                                                                   const uint32_t* __restrict__ carry, int nb) {
    __shared__ uint32_t wtot[2][kVecThreads / 32];
    const int b = blockIdx.x, i = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int y0 = b * kBandRows, y1 = min(H, y0 + kBandRows);
    uint16_t* o = out + (int64_t)i * out_stride;  // column c of II at index c + 7
    if (b == 0)
        for (int c = threadIdx.x; c <= W; c += kVecThreads) o[c + 7] = 0u;  // row 0
    const int x = 8 * threadIdx.x;  // W <= 8 * kVecThreads (launch guard)
    const bool act = x < W;
    const uint8_t* src = img + (int64_t)i * img_stride + x;
    uint32_t v[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // column prefix V of this thread's 8 columns
    if (act) {
        const uint4* c4 = reinterpret_cast<const uint4*>(carry + ((int64_t)i * nb + b) * W + x);
        const uint4 c0 = c4[0], c1 = c4[1];
        v[0] = c0.x; v[1] = c0.y; v[2] = c0.z; v[3] = c0.w; v[4] = c1.x; v[5] = c1.y; v[6] = c1.z; v[7] = c1.w;
    }
    uint2 nxt = act && y0 < y1 ? __ldg(reinterpret_cast<const uint2*>(src + (int64_t)y0 * pitch)) : make_uint2(0, 0);
    for (int y = y0; y < y1; ++y) {
        const int pb = y & 1;
        const uint2 w = nxt;
        if (act && y + 1 < y1) nxt = __ldg(reinterpret_cast<const uint2*>(src + (int64_t)(y + 1) * pitch));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] += (w.x >> (8 * k)) & 0xffu;
            v[k + 4] += (w.y >> (8 * k)) & 0xffu;
        }
        uint32_t p[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) p[k] = (k ? p[k - 1] : 0u) + v[k];
        // block-wide exclusive scan of the thread totals p[7]
        uint32_t incl = p[7];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) wtot[pb][warp] = incl;
        __syncthreads();
        uint32_t base = incl - p[7];
#pragma unroll
        for (int w2 = 0; w2 < kVecThreads / 32; ++w2)
            if (w2 < warp) base += wtot[pb][w2];
        uint16_t* row = o + (int64_t)(y + 1) * op;
        if (act) {
            uint4 st;
            st.x = ((base + p[0]) & 0xffffu) | ((base + p[1]) << 16);
            st.y = ((base + p[2]) & 0xffffu) | ((base + p[3]) << 16);
            st.z = ((base + p[4]) & 0xffffu) | ((base + p[5]) << 16);
            st.w = ((base + p[6]) & 0xffffu) | ((base + p[7]) << 16);
            *reinterpret_cast<uint4*>(row + x + 8) = st;
        }
        if (threadIdx.x == 0) row[7] = 0u;  // column 0
    }
}

}  // namespace kern

using namespace kern;

// bands for the small-image path: enough (column, band) threads to fill the GPU, >= 8 rows each
static int integral_bands(int n, int H, int W) {
    const int64_t cols = (int64_t)n * (W + 1);
    const int64_t want = (int64_t)num_sms() * 512;
    if (cols >= want / 4 || H < 32) return 1;
    int nb = (int)std::min<int64_t>((want + cols - 1) / cols, (H + 7) / 8);
    return nb < 2 ? 1 : nb;
}

size_t integral_workspace_bytes(int n, int H, int W) {
    const int nb = integral_bands(n, H, W);
    return nb > 1 ? (size_t)n * nb * W * 4 : 0;
}

// T = uint32_t: the exact integral (sums < 2^32); T = uint16_t: the integral mod 2^16, enough
// for box sums < 2^16 (boxes of radius <= 7 over 8-bit pixels) at half the HBM traffic
template <typename T>
static cudaError_t launch_integral_t(const uint8_t* img, int n, int H, int W, int64_t pitch, T* out,
                                     int64_t out_pitch, cudaStream_t s, void* ws) {
    const int64_t out_stride = out_pitch * (int64_t)(H + 1);
    ProfScope ps("integral", s);
    const int nb = ws ? integral_bands(n, H, W) : 1;
    if (nb > 1) {
        const int R = (H + nb - 1) / nb;
        const int nbr = (H + R - 1) / R;
        uint32_t* tot = reinterpret_cast<uint32_t*>(ws);
        dim3 g1((W + 1 + kColThreads - 1) / kColThreads, nbr, n);
        integral_cols_banded_kernel<T><<<g1, kColThreads, 0, s>>>(img, H, W, pitch, pitch * (int64_t)H, out, out_pitch,
                                                                  out_stride, R, tot, nbr);
        dim3 gc((W + 7) / 8, n);
        integral_band_carry_kernel<<<gc, 256, 0, s>>>(tot, W, nbr);
        dim3 g2((H + kRowWarps - 1) / kRowWarps, n);
        integral_rows_banded_kernel<T><<<g2, kRowWarps * 32, 0, s>>>(H, W, out, out_pitch, out_stride, R, tot, nbr);
        return cudaGetLastError();
    }
    dim3 g1((W + 1 + kColThreads - 1) / kColThreads, n);
    integral_cols_kernel<T><<<g1, kColThreads, 0, s>>>(img, H, W, pitch, pitch * (int64_t)H, out, out_pitch,
                                                       out_stride);
    dim3 g2((H + kRowWarps - 1) / kRowWarps, n);
    integral_rows_kernel<T><<<g2, kRowWarps * 32, 0, s>>>(H, W, out, out_pitch, out_stride);
    return cudaGetLastError();
}

cudaError_t launch_integral(const uint8_t* img, int n, int H, int W, int64_t pitch, uint32_t* out,
                            int64_t out_pitch, cudaStream_t s, void* ws) {
    return launch_integral_t<uint32_t>(img, n, H, W, pitch, out, out_pitch, s, ws);
}

cudaError_t launch_integral16(const uint8_t* img, int n, int H, int W, int64_t pitch, uint16_t* out,
                              int64_t out_pitch, cudaStream_t s, void* ws) {
    return launch_integral_t<uint16_t>(img, n, H, W, pitch, out, out_pitch, s, ws);
}

bool integral16_vec_ok(const uint8_t* img, int n, int H, int W, int64_t pitch) {
    // enough (band, image) CTAs to fill the GPU twice; smaller batches keep the banded path
    const int64_t ctas = (int64_t)n * ((H + kBandRows - 1) / kBandRows);
    return W % 8 == 0 && W <= 8 * kVecThreads && pitch % 8 == 0 && ((uintptr_t)img & 7) == 0 && H >= 1 &&
           ctas >= 2 * num_sms();
}
size_t integral16_vec_workspace_bytes(int n, int H, int W) {
    const int nb = (H + kBandRows - 1) / kBandRows;
    return (size_t)n * nb * W * 4;
}
// out: the integral with column c at out[y * out_pitch + c + 7]; out_pitch % 8 == 0, out 16-byte
// aligned; ws: integral16_vec_workspace_bytes(n, H, W)
cudaError_t launch_integral16_vec(const uint8_t* img, int n, int H, int W, int64_t pitch, uint16_t* out,
                                  int64_t out_pitch, cudaStream_t s, void* ws) {
    const int nb = (H + kBandRows - 1) / kBandRows;
    uint32_t* tot = reinterpret_cast<uint32_t*>(ws);
    ProfScope ps("integral", s);
    integral16_band_totals<<<dim3(nb, n), kVecThreads, 0, s>>>(img, H, W, pitch, pitch * (int64_t)H, tot, nb);
    integral16_band_carry<<<dim3((W + 255) / 256, n), 256, 0, s>>>(tot, W, nb);
    integral16_band_rows<<<dim3(nb, n), kVecThreads, 0, s>>>(img, H, W, pitch, pitch * (int64_t)H, out, out_pitch,
                                                            out_pitch * (int64_t)(H + 1), tot, nb);
    return cudaGetLastError();
}

}  // namespace bd
