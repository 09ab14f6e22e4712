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

}  // namespace bd
