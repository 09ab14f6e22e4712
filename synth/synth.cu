// synth.cu — CUDA twin of synth/__init__.py (seeded integer-exact smoothed noise).
// TEST / BENCH INFRASTRUCTURE: generates the synthetic images / patches of BASELINE.json
// configs directly in HBM (68 GB for configs[4] cannot come from the host).  Holds none of
// the method's arithmetic.  Must stay byte-identical to the numpy generator (checked by
// tests/test_gpu_synth.py).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

__device__ __forceinline__ uint64_t hash64(uint64_t key, int64_t a, int64_t b, int64_t c) {
    uint64_t h = mix64(key + 0x9E3779B97F4A7C15ull);
    h = mix64(h ^ ((uint64_t)a * 0x9E3779B97F4A7C15ull + 1ull));
    h = mix64(h ^ ((uint64_t)b * 0xBF58476D1CE4E5B9ull + 2ull));
    h = mix64(h ^ ((uint64_t)c * 0x94D049BB133111EBull + 3ull));
    return h;
}

__device__ __forceinline__ int noise(uint64_t key, int64_t unit, int64_t r, int64_t c) {
    const uint64_t h = hash64(key, unit, r, c);
    return (int)((h & 0xFF) + ((h >> 8) & 0xFF) + ((h >> 16) & 0xFF) + ((h >> 24) & 0xFF)) - 510;
}

__constant__ int c_w[13] = {3, 11, 35, 83, 155, 226, 256, 226, 155, 83, 35, 11, 3};

constexpr int TX = 32, TY = 16, R = 6;

// One CTA = a 32x16 output tile of one unit (image or patch).  Noise for the tile plus a
// 6-pixel apron is generated into smem, blurred horizontally then vertically (int32, exact).
__global__ void __launch_bounds__(TX * TY) synth_kernel(uint64_t key, int64_t unit0, int H, int W,
                                                        int64_t pitch, int64_t unit_stride, long long g1,
                                                        int gain_mode, uint64_t gain_key, uint8_t* out) {
    __shared__ int z[TY + 2 * R][TX + 2 * R];
    __shared__ int t[TY + 2 * R][TX];
    const int64_t unit = unit0 + blockIdx.z;
    const int r0 = blockIdx.y * TY, c0 = blockIdx.x * TX;
    for (int idx = threadIdx.x; idx < (TY + 2 * R) * (TX + 2 * R); idx += blockDim.x) {
        const int rr = idx / (TX + 2 * R), cc = idx % (TX + 2 * R);
        z[rr][cc] = noise(key, unit, r0 + rr - R, c0 + cc - R);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < (TY + 2 * R) * TX; idx += blockDim.x) {
        const int rr = idx / TX, cc = idx % TX;
        int s = 0;
#pragma unroll
        for (int k = 0; k < 13; ++k) s += c_w[k] * z[rr][cc + k];
        t[rr][cc] = s;
    }
    __syncthreads();
    const int ty = threadIdx.x / TX, tx = threadIdx.x % TX;
    const int r = r0 + ty, c = c0 + tx;
    if (r >= H || c >= W) return;
    long long f = 0;
#pragma unroll
    for (int k = 0; k < 13; ++k) f += (long long)c_w[k] * t[ty + k][tx];
    long long gq = 1024;
    if (gain_mode) gq = 512 + (long long)(hash64(gain_key, unit, 0, 0) % 1537ull);
    const long long g = g1 * gq;
    long long v = ((f * g + (1ll << 41)) >> 42) + 128;
    v = v < 0 ? 0 : (v > 255 ? 255 : v);
    out[blockIdx.z * unit_stride + (int64_t)r * pitch + c] = (uint8_t)v;
}

uint64_t stream_key(uint64_t seed, uint64_t stream) { return seed * 0x100000001B3ull + stream * 0x9E37ull; }

}  // namespace

extern "C" {

// n smoothed-noise images of H x W (row pitch `pitch`), units unit0 .. unit0+n-1.
int synth_images(uint64_t seed, int64_t unit0, int n, int H, int W, int64_t pitch, long long g1, uint8_t* out,
                 void* stream) {
    for (int z0 = 0; z0 < n; z0 += 65535) {
        const int nz = n - z0 < 65535 ? n - z0 : 65535;
        dim3 grid((W + TX - 1) / TX, (H + TY - 1) / TY, nz);
        synth_kernel<<<grid, TX * TY, 0, (cudaStream_t)stream>>>(stream_key(seed, 1), unit0 + z0, H, W, pitch,
                                                                  pitch * H, g1, 0, 0,
                                                                  out + (int64_t)z0 * pitch * H);
    }
    return (int)cudaGetLastError();
}

// n 32x32 patches (units unit0 ..), each with its own gain q/1024, q in 512..2048.
int synth_patches(uint64_t seed, int64_t unit0, int64_t n, long long g1, uint8_t* out, void* stream) {
    for (int64_t z0 = 0; z0 < n; z0 += 65535) {
        const int nz = (int)(n - z0 < 65535 ? n - z0 : 65535);
        dim3 grid(1, 2, nz);
        synth_kernel<<<grid, TX * TY, 0, (cudaStream_t)stream>>>(stream_key(seed, 1), unit0 + z0, 32, 32, 32, 1024,
                                                                  g1, 1, stream_key(seed, 6),
                                                                  out + z0 * 1024);
    }
    return (int)cudaGetLastError();
}

}
