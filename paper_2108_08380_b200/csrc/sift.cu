// sift.cu — §8(a) rows a6-a8: SIFT 4x4x8 histogram of a normalised 32x32 patch
// ("the vector of real valued features provided by SIFT"; conventions R10).
//
// One warp per patch, lane = pixel ROW y; the lane walks the 32 columns of its row.
// BJ.ns (3): "fuses the gradient and orientation binning with a warp-level histogram
// reduction".  Design — the kernel is bound by shared-memory traffic and
// issue slots, so every choice below removes one or the other:
//  * the lane's row arrives straight from HBM as two 16-byte loads (no smem staging); rows
//    y-1 and y+1 come as 8+8 word shuffles (replicate border at lanes 0 / 31);
//  * pixels become exact biased floats 2^23 + p with one PRMT (no I2F); gx, gy are exact
//    differences of biased floats;
//  * m = m2 * rsqrt(m2) and the first-octant angle from t = min(|gx|,|gy|) / m = sin(phi)
//    via a degree-11 odd polynomial of asin (|err| < 7e-7 bin): ONE MUFU per pixel; the
//    octant (3 sign/compare bits) picks the base bin o0 and the direction through an 8-entry
//    nibble LUT (no FRND / F2I);
//  * the x-direction Gaussian x trilinear weights are compile-time immediates (unrolled x):
//    a pixel adds (m*wx*(1-fo), m*wx*fo) to the PAIR ENTRY e[o0] = (part of bin o0, part of
//    bin o0+1) of cell columns i0 and i0+1 in a per-lane private histogram
//    e[i][o][y] (float2; bank pair = y, conflict-free for any o0): one 8-byte load + store
//    per cell instead of two 4-byte ones, and no wrap bin (e[7].y is bin 8 = bin 0);
//  * when the walk leaves cell column i (after x = 11, 19, 27, 31) the column is reduced
//    over rows with the y-direction tent weights: lane (j, o) reads e[o] of the 8 rows of
//    BAND j (between the centres of cell rows j and j+1) once, DIRECTLY from the histogram,
//    in the rotated order r = (o + k) & 7 (conflict-free 8-byte loads), into two sums (for
//    cell rows j and j+1); cell row j, bin o = own sums + band j-1's sums + the e[o-1].y
//    parts (three shuffles).  Each histogram entry is read exactly once (the earlier
//    per-cell-row reduction read every row twice: 128 -> 64 wavefronts per patch), with an
//    ATOMIC EXCHANGE against zero: ATOMS.EXCH.64 costs the shared-memory bandwidth of one
//    LDS.64 (tools/lab/atoms_lab.cu), so the histogram is left clear for the next patch and
//    the separate clear (64 wavefronts per patch) is gone.  The per-lane addresses and
//    weights of the 8 steps are loop invariants;
//  * the 128 entries are j*32 + i*8 + o with lane = (j, o): L2-normalise, clip at 0.2,
//    renormalise (zero stays zero) with warp all-reductions.
#include <math.h>

#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kWarps = 8;
constexpr int kColF2 = 8 * 32;                 // one cell column: [pair entry o][row] float2
constexpr int kHistF2 = 4 * kColF2;            // 1024 float2 = 8 KB per warp

// compile-time exp for the weight tables (|x| <= 0.5, 24 Taylor terms: exact to fp64)
constexpr double cexp(double x) {
    double s = 1.0, t = 1.0;
    for (int k = 1; k < 24; ++k) {
        t *= x / k;
        s += t;
    }
    return s;
}
constexpr double gauss(int t) { return cexp(-((t - 15.5) * (t - 15.5)) / 512.0); }  // sigma 16 (R10)
constexpr int cell0(int x) { return x < 4 ? -1 : (x - 4) / 8; }                   // floor((x-3.5)/8)
constexpr double frac8(int x) { return (x - 3.5) / 8.0 - cell0(x); }
// weight of pixel column x for cell columns cell0(x) (W0) and cell0(x) + 1 (W1)
constexpr float wx0(int x) { return (float)(gauss(x) * (1.0 - frac8(x))); }
constexpr float wx1(int x) { return (float)(gauss(x) * frac8(x)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// packed fp32x2 helpers (Blackwell FADD2 / FMUL2 / FFMA2; each half is an fp32 op)
__device__ __forceinline__ uint64_t pk2(float x, float y) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& x, float& y) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// byte k (0..3) of w as the exact float 2^23 + byte
__device__ __forceinline__ float bfloat(uint32_t w, int k) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7650u | (uint32_t)k));
}

__global__ void __launch_bounds__(kWarps * 32, 3) sift_kernel(const uint8_t* __restrict__ patches, int64_t n,
                                                           float* __restrict__ sift, int root) {
    extern __shared__ __align__(16) float2 s_hist[];  // kWarps x kHistF2 (64 KB, dynamic)
    debug_poison_smem(s_hist);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float2* hist = s_hist + warp * kHistF2;
    for (int i = lane; i < kHistF2; i += 32) hist[i] = make_float2(0.f, 0.f);

    // reduction-phase lane role: band j = lane / 8 = the 8 rows between the centres of cell
    // rows j and j+1 (y = 8j+4 .. 8j+11; band 3 also takes rows 0..3, the part of band -1 that
    // feeds cell row 0), o = lane % 8.  Every histogram row is read exactly once; a row of
    // band j adds g(y)(1 - fy) to cell row j and g(y) fy to cell row j+1 (mod 4), with
    // fy = (y - 8j - 3.5)/8 — the tent weights of R10.  Rows are visited in the rotated order
    // r = (o + k) & 7, so each half-warp reads 16 distinct rows (conflict-free 8-byte loads).
    const int gj = lane >> 3, go = lane & 7;
    // final combination (see the column reduction): bin go reads octant lanes (band base) |
    // {0,1,3,2,6,7,5,4}[go] and | {4,0,1,3,2,6,7,5}[go], packed in one register (5 bits each)
    const uint32_t gsrc12 = (uint32_t)(lane & ~7) | ((0x45762310u >> (4 * go)) & 7u) |
                            (((uint32_t)(lane & ~7) | ((0x57623104u >> (4 * go)) & 7u)) << 5);
    uint32_t gsrc[8];  // shared-window byte addresses (32-bit: half the registers of pointers)
    float gwa[8], gwb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int r = (go + k) & 7;
        int y;
        float wa, wb;
        if (gj < 3 || r < 4) {  // band gj proper (band 3: rows 28..31, no cell row 4)
            y = 8 * gj + 4 + r;
            const float fy = ((float)r + 0.5f) * 0.125f;
            const float dy = (float)y - 15.5f;
            const float g = expf(-dy * dy * (1.0f / 512.0f));
            wa = g * (1.0f - fy);
            wb = gj < 3 ? g * fy : 0.f;
        } else {  // band -1 (rows 0..3) -> cell row 0, carried as band 3's "next" cell row
            y = r - 4;
            const float dy = (float)y - 15.5f;
            const float g = expf(-dy * dy * (1.0f / 512.0f));
            wa = 0.f;
            wb = g * (1.0f - (3.5f - (float)y) * 0.125f);
        }
        gwa[k] = wa;
        gwb[k] = wb;
        gsrc[k] = (uint32_t)__cvta_generic_to_shared(hist + go * 32 + y);
    }
    float2* const hrow = hist + lane;  // this lane's row: e[i][o][lane]
    // the same as a 32-bit shared-window byte address: entry e[i][q][lane] at + 256 q + 2048 i
    const uint32_t hrow_s = (uint32_t)__cvta_generic_to_shared(hrow);
    const int yu = lane > 0 ? lane - 1 : 0, yd = lane < 31 ? lane + 1 : 31;
    __syncwarp();

    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    int64_t p = (int64_t)blockIdx.x * kWarps + warp;
    uint4 qa = make_uint4(0, 0, 0, 0), qb = qa;
    if (p < n) {
        const uint4* src = reinterpret_cast<const uint4*>(patches + p * 1024 + lane * 32);
        qa = __ldg(src);
        qb = __ldg(src + 1);
    }
    for (; p < n; p += nwarps) {
        const uint32_t w[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        if (p + nwarps < n) {  // prefetch the next patch's row
            const uint4* src = reinterpret_cast<const uint4*>(patches + (p + nwarps) * 1024 + lane * 32);
            qa = __ldg(src);
            qb = __ldg(src + 1);
        }
        uint32_t up[8], dn[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            up[k] = __shfl_sync(0xffffffffu, w[k], yu);
            dn[k] = __shfl_sync(0xffffffffu, w[k], yd);
        }
        float h[4];
        // pixel x as an exact biased float (2^23 + p) of this lane's row, x clamped to [0, 31]
        auto px = [&](int x) { x = x < 0 ? 0 : (x > 31 ? 31 : x); return bfloat(w[x >> 2], x & 3); };
        // Pixels in PAIRS (x, x+1), x even: the element-wise float math of both pixels runs as
        // packed fp32x2 (FADD2 / FMUL2 / FFMA2, each half an ordinary fp32 op); cell boundaries
        // (x = 4, 12, 20, 28) are even, so both pixels of a pair share their cell columns.
#pragma unroll
        for (int x = 0; x < 32; x += 2) {
            // gx = P[x+1] - P[x-1], gy = P_down[x] - P_up[x] (replicate borders; exact)
            const uint64_t GX = sub2(pk2(px(x + 1), px(x + 2)), pk2(px(x - 1), px(x)));
            const uint64_t GY = sub2(pk2(bfloat(dn[x >> 2], x & 3), bfloat(dn[(x + 1) >> 2], (x + 1) & 3)),
                                     pk2(bfloat(up[x >> 2], x & 3), bfloat(up[(x + 1) >> 2], (x + 1) & 3)));
            float gx[2], gy[2];
            upk2(GX, gx[0], gx[1]);
            upk2(GY, gy[0], gy[1]);
            const uint64_t M2 = fma2(GX, GX, mul2(GY, GY));
            float m2[2];
            upk2(M2, m2[0], m2[1]);
            const float rs0 = rsqrt_approx(fmaxf(m2[0], 1e-30f)), rs1 = rsqrt_approx(fmaxf(m2[1], 1e-30f));
            const uint64_t RS = pk2(rs0, rs1);
            const uint64_t MM = mul2(M2, RS);                                   // m (0 when m2 == 0)
            const uint64_t T = mul2(pk2(fminf(fabsf(gx[0]), fabsf(gy[0])), fminf(fabsf(gx[1]), fabsf(gy[1]))), RS);
            const uint64_t S = mul2(T, T);                                      // t = sin(phi)
            // asin(t)*4/pi = t*P(t^2), degree-9 odd fit on [0, 1/sqrt(2)]: |err| < 4e-6 bin
            uint64_t A = fma2(S, pk2(0.13525834679603577f, 0.13525834679603577f),
                              pk2(-0.0037576095201075077f, -0.0037576095201075077f));
            A = fma2(S, A, pk2(0.11007487773895264f, 0.11007487773895264f));
            A = fma2(S, A, pk2(0.21086856722831726f, 0.21086856722831726f));
            A = fma2(S, A, pk2(1.2732713222503662f, 1.2732713222503662f));
            float c1[2], mm[2];
            upk2(mul2(A, T), c1[0], c1[1]);                                     // phi * 4/pi in [0, 1]
            upk2(MM, mm[0], mm[1]);
            const int i0 = cell0(x);
            uint32_t hb[2];  // shared byte addresses of the pixels' pair entries (column 0)
            float fo[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                // octant: theta = atan2(gy, gx) in [0, 2pi) (y down) -> co = K + sigma*c1; the
                // base bin o0 and sigma come from (ay > ax, gx < 0, gy < 0)
                const uint32_t q = (uint32_t)(fabsf(gy[k]) > fabsf(gx[k])) | ((__float_as_uint(gx[k]) >> 30) & 2u) |
                                   ((__float_as_uint(gy[k]) >> 29) & 4u);  // gx, gy exact: never -0
                // The pair entry is indexed by the OCTANT q, not by the base bin o0(q), and always
                // receives (w (1 - c1), w c1): for the octants where the angle runs backwards
                // (fo = 1 - c1) that is (part of bin o0 + 1, part of bin o0) — the reduction
                // knows each octant's two target bins, so no bin lookup and no flip per pixel
                fo[k] = c1[k];
                hb[k] = hrow_s + q * 256u;  // pair entry e[q] of this lane's row
            }
            if (i0 >= 0) {  // cell column i0, weight g(x)(1 - fx)
                // scalar FMULs with immediate weights (a packed FMUL2 needs the weight pair
                // materialised in registers: 2 extra moves per use)
                const float wa[2] = {mm[0] * wx0(x), mm[1] * wx0(x + 1)};
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const uint32_t q0 = hb[k] + (uint32_t)(i0 * kColF2 * 8);
                    uint64_t v;
                    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(q0) : "memory");
                    v = fma2(pk2(wa[k], wa[k]), pk2(1.0f - fo[k], fo[k]), v);
                    asm volatile("st.shared.b64 [%0], %1;" ::"r"(q0), "l"(v) : "memory");
                }
            }
            if (i0 + 1 <= 3) {  // cell column i0 + 1, weight g(x) fx
                const float wb[2] = {mm[0] * wx1(x), mm[1] * wx1(x + 1)};
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const uint32_t q1 = hb[k] + (uint32_t)((i0 + 1) * kColF2 * 8);
                    uint64_t v;
                    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(q1) : "memory");
                    v = fma2(pk2(wb[k], wb[k]), pk2(1.0f - fo[k], fo[k]), v);
                    asm volatile("st.shared.b64 [%0], %1;" ::"r"(q1), "l"(v) : "memory");
                }
            }
            if (x + 1 == 11 || x + 1 == 19 || x + 1 == 27 || x + 1 == 31) {
                // cell column ci complete: reduce over rows (reading every entry once, with an
                // atomic exchange that leaves it zero for the next patch: ATOMS.EXCH.64 costs
                // one LDS.64 of shared-memory bandwidth, so the clear is free —
                // tools/lab/atoms_lab.cu), combine pair halves
                const int ci = x + 1 == 11 ? 0 : (x + 1 == 19 ? 1 : (x + 1 == 27 ? 2 : 3));
                __syncwarp();
                // (xa, ya) and (xb, yb) as packed pairs: one FFMA2 per weight and row (the
                // weight broadcast to both halves), half the FFMAs of the scalar form
                uint64_t AXY = pk2(0.f, 0.f), BXY = pk2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    uint64_t v;
                    asm volatile("atom.shared.exch.b64 %0, [%1], 0;" : "=l"(v) : "r"(gsrc[k] + (uint32_t)(ci * kColF2 * 8))
                                 : "memory");
                    AXY = fma2(pk2(gwa[k], gwa[k]), v, AXY);
                    BXY = fma2(pk2(gwb[k], gwb[k]), v, BXY);
                }
                float xa, ya, xb, yb;
                upk2(AXY, xa, ya);
                upk2(BXY, xb, yb);
                // cell row j, bin o = xa(j, o) + xb(j-1, o) + ya(j, o-1) + yb(j-1, o-1)
                // (pair entry e[o] = (part of bin o, part of bin o+1); indices mod 4 and mod 8)
                const int below = (((gj - 1) & 3) << 3) | go;
                // cell row j, octant q = go: the (w (1 - c1), w c1) halves, both bands
                const float ua = xa + __shfl_sync(0xffffffffu, xb, below);
                const float ub = ya + __shfl_sync(0xffffffffu, yb, below);
                // bin o of cell row j = two octants' halves (o0(q) = {0,1,3,2,7,6,4,5}, the halves
                // reversed for q in {1,2,4,7}):  bin 0 = A0 + A4, 1 = B0 + B1, 2 = A1 + A3,
                // 3 = B2 + B3, 4 = A2 + A6, 5 = B6 + B7, 6 = A5 + A7, 7 = B4 + B5 (A = first half,
                // B = second).  Two shuffles: every octant lane is read once per shuffle, by one
                // even bin (wanting A) in one and one odd bin (wanting B) in the other, so it
                // sends A in the shuffle where an even bin reads it: octants {0, 3, 5, 6} in the
                // first, {1, 2, 4, 7} in the second.
                const bool a_first = (0x69u >> go) & 1u;  // q in {0, 3, 5, 6}
                const float s1 = __shfl_sync(0xffffffffu, a_first ? ua : ub, (int)(gsrc12 & 31u));
                const float s2 = __shfl_sync(0xffffffffu, a_first ? ub : ua, (int)(gsrc12 >> 5));
                h[ci] = s1 + s2;
            }
        }
        // normalise, clip 0.2, renormalise (R10); the zero histogram stays zero
        const float n2 = warp_sum(h[0] * h[0] + h[1] * h[1] + h[2] * h[2] + h[3] * h[3]);
        if (n2 > 0.f) {
            const float inv = 1.0f / sqrtf(n2);
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = fminf(h[i] * inv, 0.2f);
            const float inv2 = 1.0f / sqrtf(warp_sum(h[0] * h[0] + h[1] * h[1] + h[2] * h[2] + h[3] * h[3]));
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] *= inv2;
            if (root) {  // NEXT-3 RootSIFT: sqrt(v / sum v)
                const float l1 = warp_sum(h[0] + h[1] + h[2] + h[3]);
                const float il1 = 1.0f / l1;
#pragma unroll
                for (int i = 0; i < 4; ++i) h[i] = sqrtf(h[i] * il1);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = 0.f;
        }
        float* o = sift + p * 128 + gj * 32 + go;
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i * 8] = h[i];
    }
}

}  // namespace kern

using namespace kern;
cudaError_t launch_sift(const uint8_t* patches, int64_t n, float* sift, int root, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    constexpr int smem = kWarps * kHistF2 * 8;  // 64 KB: 3 CTAs (24 warps) per SM at <= 80 registers
    cudaError_t ea = ensure_smem_attr((const void*)sift_kernel, smem);
    if (ea != cudaSuccess) return ea;
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sift_kernel, kWarps * 32, smem);
    if (e != cudaSuccess) return e;
    int64_t blocks = (n + kWarps - 1) / kWarps;
    const int64_t cap = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
    if (blocks > cap) blocks = cap;
    ProfScope ps("sift", s);
    sift_kernel<<<(unsigned)blocks, kWarps * 32, smem, s>>>(patches, n, sift, root);
    return cudaGetLastError();
}

}  // namespace bd
