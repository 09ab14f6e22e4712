// bad_patch.cu — §8(a) rows a1, a3, a4 on 32x32 patches (configs[2]; configs[4] BAD on the
// warped patch, R20).  Fixed geometry (centre (16,16), scale 1, angle 0, R7), so every
// test's 8 integral-image corners, both clamped areas and the exact integer threshold
// floor(theta*A1*A2) are known at bad_create (PatchTable, passed by value as a kernel
// parameter -> constant bank).
//
// Design:
//  * Persistent CTAs, 1 per SM (201 KB smem), 8 warps; a tile is 64 patches = 32 PAIRS.
//  * Packed pair integral: the integral image of A + 65536*B (A, B two patches) is built
//    with plain 32-bit adds.  Box sums are linear, so S_packed = S_A + 65536*S_B exactly,
//    and since 0 <= S < 2^16 (<= 121*255) both halves separate without ambiguity: one
//    32-bit shared-memory load serves two patches (halves the smem wavefronts).
//  * smem integral layout [entry e][pair p] with 33 words per entry: entry e = (y-1)*32 +
//    (x-1) for y, x in 1..32 plus a zero entry 1024 (row/column 0 of an integral is zero).
//    Word (e*33 + p) -> bank (e + p) mod 32: the test phase (lane = pair, uniform entry)
//    and the build phase (8 lanes per pair on 8 column groups) are both conflict-free.
//  * Staging: the 64 KB tile arrives by 32 bulk copies (TMA engine, cp.async.bulk, one
//    2 KB pair each) into a 2080-byte-pitch buffer (conflict-free pixel reads) tracked by
//    an mbarrier; the next tile's copy is issued as soon as the build has consumed the
//    staging buffer, so it overlaps the test phase.
//  * Build: warp w builds pairs 4w..4w+3; lane (q = lane/8, column group cg = lane%8) owns
//    4 columns; per row a 3-step shuffle scan over the 8 lanes of a pair gives the row
//    prefix, a running register sum gives the column prefix.
//  * Tests: warp w evaluates 32-test groups w, w+8, ...; lane = pair; 8 corner loads,
//    packed S1, S2, unpacked halves, two IMADs per patch, sign bit -> bit j of the word.
#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kPairs = 32;                 // pairs per tile (64 patches)
constexpr int kWarps = 8;
constexpr int kEntryWords = 33;            // 32 pairs + 1 pad word
constexpr int kEntries = 1025;             // 32x32 nonzero entries + zero entry
constexpr int kIIBytes = kEntries * kEntryWords * 4;             // 135300
constexpr int kIIBytesAligned = (kIIBytes + 127) / 128 * 128;    // 135424
constexpr int kStgPitch = 2080;            // bytes per pair in the staging buffer
constexpr int kStgBytes = kPairs * kStgPitch;                    // 66560
constexpr int kSmemBytes = kIIBytesAligned + kStgBytes + 64;     // + mbarrier

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Thread 0: issue the bulk copies of tile `t` (patches [64t, 64t+64) ∩ [0, n)).
__device__ __forceinline__ void issue_tile(const uint8_t* __restrict__ patches, int64_t n, int64_t t,
                                           uint8_t* stg, uint64_t* bar) {
    const int64_t first = t * 64;
    const int64_t cnt = min((int64_t)64, n - first);
    mbar_expect_tx(bar, (uint32_t)(cnt * 1024));
    for (int q = 0; 2 * q < cnt; ++q) {
        const uint32_t bytes = (2 * q + 1 < cnt) ? 2048u : 1024u;
        bulk_g2s(stg + q * kStgPitch, patches + (first + 2 * q) * 1024, bytes, bar);
    }
}

__global__ void __launch_bounds__(kWarps * 32, 1)
    bad_patch_kernel(const uint8_t* __restrict__ patches, int64_t n, uint32_t* __restrict__ out, int K,
                     const __grid_constant__ PatchTable tab) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* II = reinterpret_cast<uint32_t*>(smem);
    uint8_t* stg = smem + kIIBytesAligned;
    uint64_t* bar = reinterpret_cast<uint64_t*>(stg + kStgBytes);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_tiles = (n + 63) / 64;
    const int words = K >> 5;

    if (threadIdx.x < kEntryWords) II[1024 * kEntryWords + threadIdx.x] = 0u;  // zero entry
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && (int64_t)blockIdx.x < n_tiles) issue_tile(patches, n, blockIdx.x, stg, bar);

    // build-phase lane roles
    const int q = warp * 4 + (lane >> 3);  // pair built by this lane
    const int cg = lane & 7;               // column group: columns 4cg .. 4cg+3
    const uint8_t* src = stg + q * kStgPitch + cg * 4;
    uint32_t* dst = II + (4 * cg) * kEntryWords + q;   // entry (y-1)*32 + 4cg + j

    uint32_t parity = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, parity ^= 1u) {
        mbar_wait(bar, parity);
        // ---------------- build the packed pair integrals (a1, on chip) ----------------
        {
            uint32_t col0 = 0, col1 = 0, col2 = 0, col3 = 0;
#pragma unroll 4
            for (int y = 0; y < 32; ++y) {
                const uint32_t wa = *reinterpret_cast<const uint32_t*>(src + 32 * y);
                const uint32_t wb = *reinterpret_cast<const uint32_t*>(src + 1024 + 32 * y);
                const uint32_t lo = __byte_perm(wa, wb, 0x5410);  // [A0 A1 B0 B1]
                const uint32_t hi = __byte_perm(wa, wb, 0x7632);  // [A2 A3 B2 B3]
                const uint32_t v0 = __byte_perm(lo, 0u, 0x4240);  // A0 + 65536*B0
                const uint32_t v1 = __byte_perm(lo, 0u, 0x4341);
                const uint32_t v2 = __byte_perm(hi, 0u, 0x4240);
                const uint32_t v3 = __byte_perm(hi, 0u, 0x4341);
                const uint32_t c0 = v0, c1 = c0 + v1, c2 = c1 + v2, c3 = c2 + v3;
                uint32_t s = c3;
#pragma unroll
                for (int d = 1; d < 8; d <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xffffffffu, s, d, 8);
                    if (cg >= d) s += u;
                }
                const uint32_t ex = s - c3;  // row prefix of the columns left of this group
                col0 += ex + c0;
                col1 += ex + c1;
                col2 += ex + c2;
                col3 += ex + c3;
                uint32_t* d0 = dst + (y * 32) * kEntryWords;
                d0[0] = col0;
                d0[kEntryWords] = col1;
                d0[2 * kEntryWords] = col2;
                d0[3 * kEntryWords] = col3;
            }
        }
        __syncthreads();  // integral complete, staging consumed
        if (threadIdx.x == 0 && t + gridDim.x < n_tiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_tile(patches, n, t + gridDim.x, stg, bar);
        }
        // ---------------- K tests per patch pair (a3) and bit packing (a4) ----------------
        {
            const uint32_t* IIl = II + lane;  // lane = pair
            const int64_t pA = t * 64 + 2 * lane;
            for (int g = warp; g < words; g += kWarps) {
                uint32_t wA = 0, wB = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const PatchTest& T = tab.t[g * 32 + j];
                    const uint32_t c0 = IIl[T.off[0] >> 2], c1 = IIl[T.off[1] >> 2];
                    const uint32_t c2 = IIl[T.off[2] >> 2], c3 = IIl[T.off[3] >> 2];
                    const uint32_t c4 = IIl[T.off[4] >> 2], c5 = IIl[T.off[5] >> 2];
                    const uint32_t c6 = IIl[T.off[6] >> 2], c7 = IIl[T.off[7] >> 2];
                    const uint32_t S1 = c0 - c1 - c2 + c3;  // = S1_A + 65536 * S1_B exactly
                    const uint32_t S2 = c4 - c5 - c6 + c7;
                    const int a1 = T.a1, a2 = T.a2, thr1 = T.thr + 1;
                    // bit = [S1*A2 - S2*A1 <= floor(theta*A1*A2)]  (R4), sign of (D - thr - 1)
                    const int eA = (int)(S1 & 0xffffu) * a2 - (int)(S2 & 0xffffu) * a1 - thr1;
                    const int eB = (int)(S1 >> 16) * a2 - (int)(S2 >> 16) * a1 - thr1;
                    wA |= ((uint32_t)eA >> 31) << j;
                    wB |= ((uint32_t)eB >> 31) << j;
                }
                if (pA < n) out[pA * words + g] = wA;
                if (pA + 1 < n) out[(pA + 1) * words + g] = wB;
            }
        }
        __syncthreads();  // tests done before the next build overwrites the integral
    }
}

}  // namespace kern

using namespace kern;
cudaError_t launch_bad_patches(const uint8_t* patches, int64_t n, const PatchTable& tab, int K, uint32_t* out,
                               cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(bad_patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int64_t tiles = (n + 63) / 64;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    ProfScope ps("bad_patch", s);
    bad_patch_kernel<<<grid, kWarps * 32, kSmemBytes, s>>>(patches, n, out, K, tab);
    return cudaGetLastError();
}

}  // namespace bd
