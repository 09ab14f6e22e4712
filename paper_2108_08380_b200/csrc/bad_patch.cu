// bad_patch.cu — §8(a) rows a1, a3, a4 on 32x32 patches, the CUDA-core build (round 1).  The
// default is the tensor-core build bad_patch_tc.cu; this kernel runs with BINDESC_PATCH_TC=0
// and keeps its own parity run (tests/test_gpu_fuzz.py).  Fixed geometry (centre (16,16), scale 1, angle 0, R7), so every
// test's 8 integral-image corners, both clamped areas and the exact integer threshold
// floor(theta*A1*A2) are known at bad_create (PatchTable, passed by value as a kernel
// parameter -> constant bank).
//
// Design:
//  * Persistent CTAs, 1 per SM (226 KB smem), 16 warps; a tile is 64 patches = 32 PAIRS.
//  * Packed pair integral: the integral image of A + 65536*B (A, B two patches) is built
//    with plain 32-bit adds.  Box sums are linear, so S_packed = S_A + 65536*S_B exactly,
//    and since 0 <= S < 2^16 (<= 225*255) both halves separate without ambiguity: one
//    32-bit shared-memory load serves two patches (halves the smem wavefronts).
//  * smem integral layout [entry e][pair p] with 33 words per entry: entry e = (y-1)*32 +
//    (x-1) for y, x in 1..32 plus a zero entry 1024 (row/column 0 of an integral is zero).
//    Word (e*33 + p) -> bank (e + p) mod 32: the test phase (lane = pair, uniform entry)
//    and the build phase (8 lanes per pair on 8 column groups) are both conflict-free.
//  * Staging: two 32 KB half-tile buffers (16 pairs each, 2080-byte pitch per pair:
//    conflict-free pixel reads), each filled by 16 bulk copies (TMA engine, cp.async.bulk)
//    tracked by its own mbarrier.  The 8 warps that build from half h release it with a
//    256-thread named barrier and immediately refill it with the next tile's half (2 bulk
//    copies per warp, issued in parallel), so the HBM stream runs through the end of the
//    build and the whole test phase.
//  * Build (all 16 warps): warp w builds pairs 4(w%8)..4(w%8)+3, rows 16(w/8)..+15; lane
//    (q = lane/8, column group cg = lane%8) owns 4 columns; 4 rows per step, each with a
//    3-step shuffle scan over the 8 lanes of a pair for the row prefix and a running register
//    sum for the column prefix; the bottom-half warp holds its entries in registers until
//    the top-half warp publishes its column totals (named barrier per pair group).
//  * Tests (all 16 warps): the K tests form units of U = 16 (K <= 256) or 32 (K <= 512)
//    consecutive tests, at most one per warp, so all 16 warps share the test phase at
//    K = 256 and K = 512.  The test records are copied once per CTA from the kernel
//    parameter into shared memory.  For the first 16 tests of every unit the lane's 8 corner
//    ADDRESSES (integral base + its pair word + offset) are written once into TENSOR MEMORY
//    (tcgen05.st; the warp's lane quarter, 128 columns per warp = all 512 columns) and read per
//    test with tcgen05.ld (double-buffered, one test ahead) — no record traffic on the L1 data
//    pipe that the corner loads and the build saturate, no address arithmetic — and, when
//    every clamped area fits a signed byte (radii <= 5), their thresholds and area words stay
//    in registers.  Tests 16..31 (K = 512) read broadcast LDS.128 records.  Per test and lane
//    (= pair): 8 corner loads, packed S1/S2, then either 2 DP2A per patch on the PACKED sums
//    (area bytes select the 16-bit half: PatchTest) or 2 unpacks + 2 IMADs per patch, and a
//    funnel shift that appends the sign bit (tests walked high to low so bit j lands at
//    position j, R16).
#include "internal.cuh"
#include "tc.cuh"

#include <stdlib.h>

namespace bd {
namespace kern {

constexpr int kWarps = 16;
constexpr int kEntryWords = 33;            // 32 pairs + 1 pad word
constexpr int kEntries = 1025;             // 32x32 nonzero entries + zero entry
constexpr int kIIBytes = kEntries * kEntryWords * 4;             // 135300
constexpr int kIIBytesAligned = (kIIBytes + 127) / 128 * 128;    // 135424
constexpr int kStgPitch = 2080;            // bytes per pair in a staging buffer
constexpr int kHalfPairs = 16;
constexpr int kStgHalfBytes = kHalfPairs * kStgPitch;            // 33280
constexpr int kTabBytes = kMaxBits * (int)sizeof(PatchTest);      // 24576
// output tile: the K bits of the tile's 64 patches, unit-major ([unit][patch]), so each warp
// writes its unit's bits with one conflict-free store and the tile leaves in coalesced rows
// (a warp's direct stores hit 64 different descriptor rows: ~20-34 L1 wavefronts each)
constexpr int kO16Stride = 68;             // halfwords per unit row (U = 16): reader banks 4j + p/2
constexpr int kO32Stride = 66;             // words per unit row (U = 32): reader banks 2j + p
constexpr int kOutBytes = kWarps * kO32Stride * 4;               // 4224 (>= 16 * 68 * 2)
constexpr int kSmemBytes = kIIBytesAligned + 2 * kStgHalfBytes + kTabBytes + 128 + kOutBytes;  // + 2 mbarriers

using namespace tc;  // smem_addr, mbarriers, bulk_g2s, named_sync

// Issue the bulk copies q in [q0, q1) (one pair each) of half `h` of tile `t` (patches
// [64t + 32h, +32) ∩ [0, n)); the thread with q0 == 0 also posts the half's expected bytes
// (an empty half still arrives with expect_tx 0 so the phase completes).  Called by one lane
// of each of several warps, so the copies are issued in parallel (a loop in one lane is a
// serial waterfall of ~20 instructions per copy).
__device__ __forceinline__ void issue_half(const uint8_t* __restrict__ patches, int64_t n, int64_t t, int h,
                                           uint8_t* stg, uint64_t* bar, int q0, int q1) {
    const int64_t first = t * 64 + 32 * h;
    const int64_t cnt = max((int64_t)0, min((int64_t)32, n - first));
    if (q0 == 0) mbar_expect_tx(bar, (uint32_t)(cnt * 1024));
    for (int q = q0; q < q1 && 2 * q < cnt; ++q) {
        const uint32_t bytes = (2 * q + 1 < cnt) ? 2048u : 1024u;
        bulk_g2s(stg + q * kStgPitch, patches + (first + 2 * q) * 1024, bytes, bar);
    }
}

// s += value of the lane d below within the 8-lane segment (if any): one SHFL whose
// in-range predicate guards the add (no select)
__device__ __forceinline__ void scan_up8_add(uint32_t& s, int d) {
    asm(
        "{\n.reg .pred p;\n.reg .b32 t;\n"
        "shfl.sync.up.b32 t|p, %0, %1, 0x1800, 0xffffffff;\n"
        "@p add.u32 %0, %0, t;\n}\n"
        : "+r"(s)
        : "r"(d));
}

// packed pixel pair -> A + 65536*B for the 4 columns of a 4-byte word (a: patch A bytes, b: B)
__device__ __forceinline__ void unpack4(uint32_t wa, uint32_t wb, uint32_t (&v)[4]) {
    const uint32_t lo = __byte_perm(wa, wb, 0x5410);  // [A0 A1 B0 B1]
    const uint32_t hi = __byte_perm(wa, wb, 0x7632);  // [A2 A3 B2 B3]
    v[0] = __byte_perm(lo, 0u, 0x4240);               // A0 + 65536*B0
    v[1] = __byte_perm(lo, 0u, 0x4341);
    v[2] = __byte_perm(hi, 0u, 0x4240);
    v[3] = __byte_perm(hi, 0u, 0x4341);
}

// Tensor-memory record store (K <= 256): each warp keeps the 8 corner offsets of its 16
// tests in its TMEM lane quarter (warp % 4), replicated over the 32 lanes, and reads them with
// tcgen05.ld (tc::tmem_ld8) — off the L1 data pipe that the corner loads saturate.

template <int U, bool DP2A>
__global__ void __launch_bounds__(kWarps * 32, 1)
    bad_patch_kernel(const uint8_t* __restrict__ patches, int64_t n, uint32_t* __restrict__ out, int K,
                     const uint8_t* __restrict__ status, const __grid_constant__ PatchTable tab) {
    extern __shared__ __align__(128) uint8_t smem[];
    debug_poison_smem(smem);
    uint32_t* II = reinterpret_cast<uint32_t*>(smem);
    uint8_t* stg0 = smem + kIIBytesAligned;
    PatchTest* stab = reinterpret_cast<PatchTest*>(stg0 + 2 * kStgHalfBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(stg0 + 2 * kStgHalfBytes + kTabBytes);
    uint32_t* otile = reinterpret_cast<uint32_t*>(stg0 + 2 * kStgHalfBytes + kTabBytes + 128);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_tiles = (n + 63) / 64;
    const int words = K >> 5;

    if (threadIdx.x < kEntryWords) II[1024 * kEntryWords + threadIdx.x] = 0u;  // zero entry
    for (int i = threadIdx.x; i < K * (int)(sizeof(PatchTest) / 16); i += blockDim.x)
        reinterpret_cast<uint4*>(stab)[i] = reinterpret_cast<const uint4*>(tab.t)[i];
    const int units = K / U;  // <= kWarps
    // tests 0..15 of each warp's unit read their corner offsets from TMEM (128 columns per
    // warp, 4 warps per lane quarter = the full 512 columns); tests 16..31 (U = 32) from smem
    constexpr bool kTmemRec = true;
    constexpr int kTm = 16;
    __shared__ uint32_t s_tmem_base;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (kTmemRec && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_addr(&s_tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this warp's record columns: lanes 32 (warp % 4) .., columns 128 (warp / 4) + 8 j
    const uint32_t tq = kTmemRec ? s_tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128)
                                 : 0u;
    if (kTmemRec && warp < units) {
        // per-lane ABSOLUTE corner addresses (integral base + this lane's pair word + offset):
        // the test loop loads them straight, with no address arithmetic
        const uint32_t IIl0 = (uint32_t)__cvta_generic_to_shared(II + lane);
#pragma unroll
        for (int j = 0; j < kTm; ++j) {
            const uint4* Tq = reinterpret_cast<const uint4*>(stab + warp * U + j);
            const uint4 o0 = Tq[0], o1 = Tq[1];
            BD_CHECK(o0.x < kIIBytes && o0.y < kIIBytes && o0.z < kIIBytes && o0.w < kIIBytes && o1.x < kIIBytes &&
                     o1.y < kIIBytes && o1.z < kIIBytes && o1.w < kIIBytes && (o0.x & 3) == 0);
            const uint32_t v[8] = {IIl0 + o0.x, IIl0 + o0.y, IIl0 + o0.z, IIl0 + o0.w,
                                   IIl0 + o1.x, IIl0 + o1.y, IIl0 + o1.z, IIl0 + o1.w};
            tmem_st8(tq + 8 * j, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0 && (int64_t)blockIdx.x < n_tiles) {
        issue_half(patches, n, blockIdx.x, 0, stg0, &bars[0], 0, 16);
        issue_half(patches, n, blockIdx.x, 1, stg0 + kStgHalfBytes, &bars[1], 0, 16);
    }

    // build-phase lane roles (all 16 warps): pair group g = warp & 7 (4 pairs), row half
    // rh = warp >> 3 (rows 16 rh .. 16 rh + 15); lane = (pair ql, column group cg of 4 columns)
    const int g = warp & 7, rh = warp >> 3;
    const int h = g >> 2;                           // staging half holding this pair group
    const int ql = 4 * (g & 3) + (lane >> 3);       // pair within the half
    const int cg = lane & 7;                        // column group: columns 4cg .. 4cg+3
    uint8_t* stg_h = stg0 + h * kStgHalfBytes;
    const uint8_t* src = stg_h + ql * kStgPitch + cg * 4 + rh * 16 * 32;
    uint32_t* dst = II + (4 * cg) * kEntryWords + (16 * h + ql) + rh * 16 * 32 * kEntryWords;
    // the bottom half's column carries = the top half's last stored row (integral row 16)
    const uint32_t* carry = II + (15 * 32 + 4 * cg) * kEntryWords + (16 * h + ql);

    // DP2A form: the thresholds and area-byte words of the unit's tests 0..15 stay in registers
    // (m2 = m1 << 8), so those tests read no threshold record from shared memory (at U = 32
    // tests 16..31 keep their shared-memory records)
    constexpr bool kThrRegs = DP2A;
    constexpr int kTr = 16;
    int rn[kTr], rm[kTr];
    if (kThrRegs) {
#pragma unroll
        for (int j = 0; j < kTr; ++j) {
            const PatchTest& T = stab[(warp < units ? warp : 0) * U + j];
            rn[j] = T.nthr1;
            rm[j] = T.m1;
        }
    }

    // coalesced store of tile tp's descriptors from the output tile (all 512 threads, at most
    // two words each; the thread -> (patch, word) map and the shared-memory offsets are loop
    // invariants).  Rows of invalid keypoints (status != 0) are written as zero
    // (bd_describe_warped).
    int f_p[2], f_j[2], f_lo[2], f_hi[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int idx = threadIdx.x + r * kWarps * 32;
        f_p[r] = idx < 64 * words ? idx / words : 64;  // 64: no word for this thread
        f_j[r] = idx - (idx / words) * words;
        f_lo[r] = U == 16 ? (2 * f_j[r]) * kO16Stride + f_p[r] : f_j[r] * kO32Stride + f_p[r];
        f_hi[r] = (2 * f_j[r] + 1) * kO16Stride + f_p[r];
    }
    auto flush = [&](int64_t tp) {
        const int64_t p0 = tp * 64;
        const uint16_t* o16 = reinterpret_cast<const uint16_t*>(otile);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (f_p[r] < 64 && p0 + f_p[r] < n) {
                uint32_t v = U == 16 ? ((uint32_t)o16[f_lo[r]] | ((uint32_t)o16[f_hi[r]] << 16)) : otile[f_lo[r]];
                if (status && status[p0 + f_p[r]]) v = 0u;
                out[(p0 + f_p[r]) * words + f_j[r]] = v;
            }
        }
    };

    uint32_t parity = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, parity ^= 1u) {
        if (t != (int64_t)blockIdx.x) flush(t - gridDim.x);  // the previous tile's bits (overlaps the TMA wait)
        mbar_wait(&bars[h], parity);
        // ------------- build the packed pair integrals (a1, on chip) -------------
        // 16 rows per warp, 4 per step: per row a 3-step shuffle scan over the 8 lanes of a
        // pair gives the row prefix, a running register sum the column prefix.  The bottom
        // half keeps its 64 partial entries in registers until the top half has published
        // its column totals (named barrier per pair group), then adds them and stores.
        uint32_t col[4] = {0u, 0u, 0u, 0u};
        uint32_t keep[4][4][4];  // bottom half: [step][row][column]
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            const int y0 = 4 * st;
            uint32_t wa[4], wb[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                wa[r] = *reinterpret_cast<const uint32_t*>(src + 32 * (y0 + r));
                wb[r] = *reinterpret_cast<const uint32_t*>(src + 1024 + 32 * (y0 + r));
            }
            if (st == 3) {
                // the 8 warps of staging half h have read it: the 4 bottom-half warps (no stores
                // interleaved, they get here first) arrive without waiting; the 4 top-half warps
                // sync and each refill its own 4 pairs with the next tile's bytes, so the copy
                // starts before the stores of this build finish
                if (rh == 1) {
                    asm volatile("bar.arrive %0, 256;" ::"r"(1 + h) : "memory");
                } else {
                    named_sync(1 + h, 256);
                    if (lane == 0 && t + gridDim.x < n_tiles) {
                        const int wi = g & 3;
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        const int64_t first = (t + gridDim.x) * 64 + 32 * h;  // first patch of this half
                        if (first + 32 <= n) {  // full half (all but the last tile): four 2 KB pair copies
                            if (wi == 0) mbar_expect_tx(&bars[h], 32u * 1024u);
                            const uint8_t* gsrc = patches + (first + 8 * wi) * 1024;
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                bulk_g2s(stg_h + (4 * wi + c) * kStgPitch, gsrc + 2048 * c, 2048u, &bars[h]);
                        } else {
                            issue_half(patches, n, t + gridDim.x, h, stg_h, &bars[h], 4 * wi, 4 * wi + 4);
                        }
                    }
                }
            }
            uint32_t c[4][4], s4[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                unpack4(wa[r], wb[r], c[r]);
                c[r][1] += c[r][0];
                c[r][2] += c[r][1];
                c[r][3] += c[r][2];
                s4[r] = c[r][3];
            }
#pragma unroll
            for (int d = 1; d < 8; d <<= 1) {
#pragma unroll
                for (int r = 0; r < 4; ++r) scan_up8_add(s4[r], d);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t ex = s4[r] - c[r][3];  // row prefix of the columns left of this group
                uint32_t* d0 = dst + ((y0 + r) * 32) * kEntryWords;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    col[k] += ex + c[r][k];
                    keep[st][r][k] = col[k];
                    if (rh == 0) d0[k * kEntryWords] = col[k];
                }
            }
        }
        if (rh == 0) {
            asm volatile("bar.arrive %0, 64;" ::"r"(3 + g) : "memory");
        } else {
            asm volatile("bar.sync %0, 64;" ::"r"(3 + g) : "memory");
            uint32_t cyk[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) cyk[k] = carry[k * kEntryWords];
#pragma unroll
            for (int st = 0; st < 4; ++st)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    uint32_t* d0 = dst + ((4 * st + r) * 32) * kEntryWords;
#pragma unroll
                    for (int k = 0; k < 4; ++k) d0[k * kEntryWords] = keep[st][r][k] + cyk[k];
                }
        }
        __syncthreads();  // integral complete
        // ------------- K tests per patch pair (a3) and bit packing (a4) -------------
        if (warp < units) {
            const uint32_t IIl = (uint32_t)__cvta_generic_to_shared(II + lane);  // lane = pair
            uint32_t wA = 0, wB = 0;
            uint32_t ob[2][8];  // TMEM records of one test, double buffered
            if (kTmemRec) tmem_ld8(tq + 8 * (kTm - 1), ob[(kTm - 1) & 1]);
#pragma unroll
            for (int j = U - 1; j >= 0; --j) {
                const uint4* Tq = reinterpret_cast<const uint4*>(stab + warp * U + j);
                uint32_t adr[8];  // shared-window addresses of this lane's 8 corners
                if (kTmemRec && j < kTm) {  // this test's records have landed; fetch the next test's
                    tmem_wait8(ob[j & 1]);
                    if (j > 0) tmem_ld8(tq + 8 * (j - 1), ob[(j - 1) & 1]);
#pragma unroll
                    for (int c = 0; c < 8; ++c) adr[c] = ob[j & 1][c];
                } else {
                    const uint4 o0 = Tq[0], o1 = Tq[1];  // broadcast loads (2 wavefronts each)
                    adr[0] = IIl + o0.x; adr[1] = IIl + o0.y; adr[2] = IIl + o0.z; adr[3] = IIl + o0.w;
                    adr[4] = IIl + o1.x; adr[5] = IIl + o1.y; adr[6] = IIl + o1.z; adr[7] = IIl + o1.w;
                }
                const uint4 q2 = (kThrRegs && j < kTr)
                                     ? make_uint4((uint32_t)rn[j & (kTr - 1)], (uint32_t)rm[j & (kTr - 1)],
                                                  (uint32_t)rm[j & (kTr - 1)] << 8, 0u)
                                          : Tq[2];  // thresholds (broadcast)
                uint32_t cv[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cv[c]) : "r"(adr[c]));
                if (BD_DEBUG) {
                    [[maybe_unused]] const uint32_t lo = (uint32_t)__cvta_generic_to_shared(II), hi = lo + kIIBytes;
#pragma unroll
                    for (int c = 0; c < 8; ++c) BD_CHECK(adr[c] >= lo && adr[c] < hi);
                }
                const uint32_t S1 = cv[0] - cv[1] - cv[2] + cv[3];  // S1_A + 65536*S1_B
                const uint32_t S2 = cv[4] - cv[5] - cv[6] + cv[7];
                const int nthr1 = (int)q2.x, m1 = (int)q2.y, m2 = (int)q2.z;
                // bit = [S1*A2 - S2*A1 <= floor(theta*A1*A2)] (R4) = sign of (D - thr1)
                int eA, eB;
                if (DP2A) {  // areas as signed bytes: two DP2A per patch, halves never unpacked
                    eA = dp2a_hi(S2, m1, dp2a_lo(S1, m1, nthr1));
                    eB = dp2a_hi(S2, m2, dp2a_lo(S1, m2, nthr1));
                } else {     // m1 = -A1, m2 = A2
                    eA = (int)(S1 & 0xffffu) * m2 + ((int)(S2 & 0xffffu) * m1 + nthr1);
                    eB = (int)(S1 >> 16) * m2 + ((int)(S2 >> 16) * m1 + nthr1);
                }
                wA = __funnelshift_l((uint32_t)eA, wA, 1);  // (wA << 1) | sign(eA)
                wB = __funnelshift_l((uint32_t)eB, wB, 1);
            }
            // this unit's bits of patches 2 lane, 2 lane + 1 into the output tile (one store)
            if (U == 32)
                *reinterpret_cast<uint2*>(otile + warp * kO32Stride + 2 * lane) = make_uint2(wA, wB);
            else  // a 16-test unit is half an output word
                otile[(warp * kO16Stride) / 2 + lane] = (wA & 0xffffu) | (wB << 16);
        }
        __syncthreads();  // tests done before the next build overwrites the integral
    }
    if ((int64_t)blockIdx.x < n_tiles) {  // the last tile's bits
        const int64_t last = blockIdx.x + (n_tiles - 1 - blockIdx.x) / gridDim.x * gridDim.x;
        flush(last);
    }
    if (kTmemRec) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem_base));
    }
}

}  // namespace kern

using namespace kern;
cudaError_t launch_bad_patches(const uint8_t* patches, int64_t n, const PatchTable& tab, int K, uint32_t* out,
                               const uint8_t* status, cudaStream_t s) {
    // the tensor-core build (bad_patch_tc.cu) for every K it takes (K % 32 == 0); this
    // CUDA-core build otherwise, or everywhere with BINDESC_PATCH_TC=0 (A/B measurement and
    // its own parity tests, tests/test_gpu_fuzz.py)
    static const int use_tc = [] {
        const char* v = getenv("BINDESC_PATCH_TC");
        return v ? atoi(v) : 1;
    }();
    if (use_tc && K % 32 == 0) return launch_bad_patches_tc(patches, n, tab, K, out, status, s);
    cudaError_t e = ensure_smem_attr((const void*)bad_patch_kernel<16, true>, kSmemBytes);
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)bad_patch_kernel<32, true>, kSmemBytes);
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)bad_patch_kernel<16, false>, kSmemBytes);
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)bad_patch_kernel<32, false>, kSmemBytes);
    if (e != cudaSuccess) return e;
    const int64_t tiles = (n + 63) / 64;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    ProfScope ps("bad_patch", s);
    if (K <= 16 * kWarps) {
        if (tab.dp2a)
            bad_patch_kernel<16, true><<<grid, kWarps * 32, kSmemBytes, s>>>(patches, n, out, K, status, tab);
        else
            bad_patch_kernel<16, false><<<grid, kWarps * 32, kSmemBytes, s>>>(patches, n, out, K, status, tab);
    } else {
        if (tab.dp2a)
            bad_patch_kernel<32, true><<<grid, kWarps * 32, kSmemBytes, s>>>(patches, n, out, K, status, tab);
        else
            bad_patch_kernel<32, false><<<grid, kWarps * 32, kSmemBytes, s>>>(patches, n, out, K, status, tab);
    }
    return cudaGetLastError();
}

}  // namespace bd
