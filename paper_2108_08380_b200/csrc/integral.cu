// integral.cu — §8(a) row a1: integral image II(r, c) = sum_{y<r, x<c} I(y, x)
// ("efficiently computed using integral images").
//
// Two passes over uint32 (sums < 2^32 for H*W*255 < 2^32):
//   1. row pass: one warp per image row; each lane owns 16 consecutive pixels, forms
//      their local prefix, a warp-shuffle exclusive scan joins the lanes (BJ.ns (1):
//      "warp-shuffle row scans"), a running carry joins 512-pixel segments.
//   2. column pass: one thread per column walks down the rows (coalesced across the
//      warp) accumulating the row prefixes (BJ.ns (1): "plus a column pass").
#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kRowWarps = 8;

__global__ void __launch_bounds__(kRowWarps * 32) integral_rows_kernel(
    const uint8_t* __restrict__ img, int H, int W, int64_t pitch, int64_t img_stride,
    uint32_t* __restrict__ out, int64_t op, int64_t out_stride) {
    const int lane = threadIdx.x & 31;
    const int y = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
    if (y >= H) return;
    const uint8_t* row = img + (int64_t)blockIdx.y * img_stride + (int64_t)y * pitch;
    uint32_t* o = out + (int64_t)blockIdx.y * out_stride + (int64_t)(y + 1) * op;
    if (lane == 0) o[0] = 0u;
    uint32_t carry = 0;
    for (int seg = 0; seg < W; seg += 512) {
        const int x0 = seg + lane * 16;
        uint32_t v[16];
        uint32_t run = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int x = x0 + k;
            run += (x < W) ? (uint32_t)__ldg(row + x) : 0u;
            v[k] = run;
        }
        // exclusive scan of the lane totals
        uint32_t incl = run;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
        }
        const uint32_t base = carry + incl - run;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int x = x0 + k;
            if (x < W) o[x + 1] = base + v[k];
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

__global__ void __launch_bounds__(256) integral_cols_kernel(int H, int W, uint32_t* __restrict__ out,
                                                            int64_t op, int64_t out_stride) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > W) return;
    uint32_t* o = out + (int64_t)blockIdx.y * out_stride + c;
    o[0] = 0u;
    uint32_t acc = 0;
    for (int r = 1; r <= H; ++r) {
        uint32_t* p = o + (int64_t)r * op;
        acc += *p;
        *p = acc;
    }
}

}  // namespace kern

using namespace kern;
cudaError_t launch_integral(const uint8_t* img, int n, int H, int W, int64_t pitch, uint32_t* out,
                            int64_t out_pitch, cudaStream_t s) {
    const int64_t out_stride = out_pitch * (int64_t)(H + 1);
    dim3 g1((H + kRowWarps - 1) / kRowWarps, n);
    ProfScope ps("integral", s);
    integral_rows_kernel<<<g1, kRowWarps * 32, 0, s>>>(img, H, W, pitch, pitch * (int64_t)H, out, out_pitch,
                                                        out_stride);
    dim3 g2((W + 1 + 255) / 256, n);
    integral_cols_kernel<<<g2, 256, 0, s>>>(H, W, out, out_pitch, out_stride);
    return cudaGetLastError();
}

}  // namespace bd
