// bad_patch_tc.cu — §8(a) rows a1, a3, a4 on 32x32 patches at K <= 256 (configs[2]) with the
// integral's column prefix on the tensor cores (DESIGN.md §5.3 "tensor-core build").
//
//  * Persistent CTAs, 1 per SM: 16 compute warps + 1 producer warp; a tile is 64 patches =
//    32 PAIRS, built in two halves of 32 patches.
//  * Staging: each half's 32 patches arrive by one TMA tensor load (3-D {32, 32, n}, box
//    32 x 32 x 32, SWIZZLE_32B, out-of-range patches zero-filled) into one of two 32 KB slots;
//    a slot is refilled with the next tile's half as soon as the MMAs that read it complete.
//  * Column prefix C = L * P (L the 32x32 lower-triangular ones matrix) as tcgen05.mma kind::i8
//    (u8 x u8 -> s32) on QUARTER tiles of 16 patches: 4 MMAs (M = 128, N = 128, K = 32), MMA q:
//    A = rows 32q..32q+31 of blockdiag(L) (K-major, a window into one zero-padded 7 KB buffer),
//    B = patches 4q..4q+3 of the quarter tile straight from the staging slot as an MN-major
//    SWIZZLE_32B operand (LBO = 1024 B, SBO = 256 B); TMEM lane quarter q then holds the column
//    prefixes of the quarter tile's pairs 2q, 2q+1.  Two D buffers of 128 columns alternate
//    (quarter tiles 0, 2 -> buffer 0, 1, 3 -> buffer 1), each read by its own 8 warps, so
//    while one group waits for its next MMAs the other group works.
//  * Row prefix in registers: compute warp (q, c) = (warp % 4, warp / 4), group g = c / 2, reads
//    row y = lane of pair 16h + 8g + 2q + c % 2 with tcgen05.ld (32 columns of each patch),
//    releases the buffer, packs A + (B << 16), runs the 32-column prefix with 32-bit adds
//    (mod 2^32; box sums < 2^16 separate exactly) and stores the row's 32 integral entries;
//    rows are 1057 words apart so these stores hit 32 banks.
//  * Tests as in bad_patch.cu (lane = pair, 8 corner loads, packed S1/S2, DP2A or integer
//    compare, funnel shift).  Each warp runs one unit of 16 tests.  The lane's 8 corner
//    ADDRESSES of tests 8..15 live in TMEM columns 256..511 (the warp's lane quarter, 64 columns
//    per warp, written once) and are read with one tcgen05.ld per test; tests 0..7 read a
//    broadcast record of 8 byte offsets from shared memory (two LDS.128) and add the lane base.
//    DP2A thresholds stay in registers.
//  * Output through the unit-major output tile, flushed in coalesced rows (bad_patch.cu).
#include "internal.cuh"
#include "tc.cuh"

#include <string.h>

namespace bd {
namespace kern_tc {

using namespace tc;

constexpr int kWarps = 16;                                   // compute warps (+ 1 producer warp)
constexpr int kThreads = (kWarps + 1) * 32;
constexpr int kRowWords = 32 * 33 + 1;                       // integral row stride (words)
constexpr int kZeroWord = 32 * kRowWords;                    // zero entry of pair 0
constexpr int kIIBytes = (kZeroWord + 33) * 4;
constexpr int kIIBytesAligned = (kIIBytes + 1023) / 1024 * 1024;
constexpr int kSlotBytes = 32 * 1024;                        // half a tile
constexpr int kSlots = 2;
constexpr int kZBytes = 28 * 256;                            // blockdiag(L) window buffer
constexpr int kTmemTests = 8;                                // tests per unit with TMEM addresses
constexpr int kRecBytes = 256 * 32;                          // corner byte offsets
constexpr int kThrBytes = 256 * 16;                          // thresholds
constexpr int kO16Stride = 68;                               // halfwords per unit row
constexpr int kOutBytes = kWarps * kO16Stride * 2;
constexpr int kBarBytes = 256;
constexpr int kSmemBytes =
    1024 + kIIBytesAligned + kSlots * kSlotBytes + kZBytes + kRecBytes + kThrBytes + kOutBytes + kBarBytes;
// instruction descriptor, kind::i8: D s32, A u8 K-major, B u8 MN-major, N = 128, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %4, p;\n}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(acc), "r"(kIdesc)
        : "memory");
}
__device__ __forceinline__ void tma_load_patches(void* dst, const CUtensorMap* map, int p, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(0), "r"(p), "r"(smem_addr(bar))
        : "memory");
}
// producer-side wait (try_wait suspends in hardware for a while before it fails; a nanosleep
// back-off here left the MMAs' issue late by microseconds)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (true) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (done) break;
    }
}
__device__ __forceinline__ int dp2a_lo(uint32_t S, int m, int c) {
    int d;
    asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(S), "r"(m), "r"(c));
    return d;
}
__device__ __forceinline__ int dp2a_hi(uint32_t S, int m, int c) {
    int d;
    asm("dp2a.hi.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(S), "r"(m), "r"(c));
    return d;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16(uint32_t (&v)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                   "+r"(v[15])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait8(uint32_t (&v)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
// table byte offsets (api.cu: entry e = (y-1)*32 + (x-1), 1024 = zero, 33 words per entry) ->
// word offsets of this kernel's layout (row stride kRowWords)
inline uint32_t conv_off(uint32_t byte_off) {
    const uint32_t e = byte_off / 132u;
    return e >= 1024u ? (uint32_t)kZeroWord : (e >> 5) * (uint32_t)kRowWords + (e & 31u) * 33u;
}

// The kernel's own test table (built from the PatchTable at launch): corner byte offsets in this
// kernel's integral layout and the thresholds; copied once per CTA into shared memory (and the
// TMEM address records).  (Read from the constant bank with a warp-uniform index instead —
// LDCU.64 into uniform registers folded into the loads' address — the 10 KB working set
// thrashes the constant cache: 2.39 ms, MIO-throttle bound.)
struct TcTable {
    uint4 off[256][2];  // byte offsets of corners 0..7 (PatchTest order)
    int4 thr[256];      // nthr1, m1, m2, 0 (PatchTest)
};

template <bool DP2A>
__global__ void __launch_bounds__(kThreads, 1)
    bad_patch_tc_kernel(const __grid_constant__ CUtensorMap map, int64_t n, uint32_t* __restrict__ out, int K,
                        const uint8_t* __restrict__ status, const __grid_constant__ TcTable tab) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    debug_poison_smem(smem_raw);
    const uint32_t raw = smem_addr(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint32_t* II = reinterpret_cast<uint32_t*>(smem);
    uint8_t* stg = smem + kIIBytesAligned;
    uint8_t* Z = stg + kSlots * kSlotBytes;
    uint4* crec = reinterpret_cast<uint4*>(Z + kZBytes);
    int4* cthr = reinterpret_cast<int4*>(Z + kZBytes + kRecBytes);
    uint32_t* otile = reinterpret_cast<uint32_t*>(Z + kZBytes + kRecBytes + kThrBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(Z + kZBytes + kRecBytes + kThrBytes + kOutBytes);
    uint64_t* full = bars;        // [2] staging slot landed
    uint64_t* dfull = bars + 2;   // [2] D buffer computed (one phase per use)
    uint64_t* dempty = bars + 4;  // [2] D buffer read out by its 8 warps
    __shared__ uint32_t s_tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = warp == kWarps;
    const int64_t n_tiles = (n + 63) / 64;
    const int words = K >> 5;
    const int units = K / 16;  // <= kWarps

    if (threadIdx.x < 33) II[kZeroWord + threadIdx.x] = 0u;
    for (int i = threadIdx.x; i < kZBytes; i += blockDim.x) {  // L in row groups 12..15 of the window
        const int g = i >> 8, w = i & 255, kc = w >> 7, r = (w & 127) >> 4, kk = w & 15;
        const int m = (g - 12) * 8 + r, kx = kc * 16 + kk;
        Z[i] = (g >= 12 && g < 16 && kx <= m) ? 1 : 0;
    }
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
        crec[2 * i] = tab.off[i][0];
        crec[2 * i + 1] = tab.off[i][1];
        cthr[i] = tab.thr[i];
    }
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&dfull[b], 1);
            mbar_init(&dempty[b], kWarps / 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_addr(&s_tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem_base;  // D buffers at columns 0, 128; address records at 256..511

    if (producer) {
        if (lane == 0) {
            const uint32_t zaddr = smem_addr(Z), saddr = smem_addr(stg);
            const int64_t my_tiles = (int64_t)blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
            const int64_t uses = 2 * my_tiles;  // use u = 2 k + h: half h of the k-th tile, slot h
            auto load = [&](int64_t u) {
                const int sl = (int)(u & 1);
                const int64_t tile = blockIdx.x + (u >> 1) * gridDim.x;
                mbar_expect_tx(&full[sl], (uint32_t)kSlotBytes);
                tma_load_patches(stg + sl * kSlotBytes, &map, (int)(tile * 64 + (u & 1) * 32), &full[sl]);
            };
            for (int64_t u = 0; u < 2 && u < uses; ++u) load(u);
            for (int64_t x = 0; x < 2 * uses; ++x) {  // quarter tile x = 4 k + r
                const int r = (int)(x & 3), b = r & 1, h = r >> 1;
                const int64_t v = x >> 1;  // use of buffer b: 2 k + h
                if (v > 0) mbar_wait_sleep(&dempty[b], (uint32_t)((v - 1) & 1));
                if (b == 0) mbar_wait_sleep(&full[h], (uint32_t)((x >> 2) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const uint64_t ad = umma_desc(zaddr + (uint32_t)(12 - 4 * qq) * 256u, 128, 256, 0);
                    const uint64_t bd =
                        umma_desc(saddr + (uint32_t)(h * kSlotBytes + (16 * b + 4 * qq) * 1024), 1024, 256, 6);
                    mma_u8(tmem + 128u * (uint32_t)b, ad, bd, qq > 0 ? 1u : 0u);
                }
                mma_commit(&dfull[b]);
                const int64_t u = x >> 1;  // half use 2 k + h
                if (b == 1 && u + 2 < uses) {  // slot h is free once this half's MMAs complete
                    mbar_wait_sleep(&dfull[1], (uint32_t)(v & 1));
                    load(u + 2);
                }
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3, c = warp >> 2, g = c >> 1;
        const bool active = warp < units;
        const int ub = (active ? warp : 0) * 16;  // the warp's unit
        const uint32_t IIbase = smem_addr(II);
        // the lane's integral base, opaque to ptxas (no re-association into the record adds)
        uint32_t IIl;
        asm volatile("mov.u32 %0, %1;" : "=r"(IIl) : "r"(IIbase + 4u * (uint32_t)lane));
        // TMEM address records of tests 8..15 of the unit: lane quarter q, columns 256 + 64 c
        const uint32_t trec = tmem + ((uint32_t)(32 * q) << 16) + 256u + 64u * (uint32_t)c;
#pragma unroll
        for (int t = 0; t < kTmemTests; ++t) {
            const int i = ub + 16 - kTmemTests + t;
            uint32_t a[8];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const uint4 r = tab.off[i][cc >> 2];
                a[cc] = IIl + ((cc & 3) == 0 ? r.x : (cc & 3) == 1 ? r.y : (cc & 3) == 2 ? r.z : r.w);
            }
            tmem_st8(trec + 8u * (uint32_t)t, a);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        // DP2A thresholds of the unit in registers (loaded through an asm so they are not
        // re-read from the constant bank inside the loop)
        int rn[16], rm[16];
        if (DP2A) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];"
                             : "=r"(rn[j]), "=r"(rm[j])
                             : "r"(smem_addr(cthr + ub + j)));
            }
        }
        int f_p[2], f_j[2], f_lo[2], f_hi[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int idx = threadIdx.x + r * kWarps * 32;
            f_p[r] = idx < 64 * words ? idx / words : 64;
            f_j[r] = idx - (idx / words) * words;
            f_lo[r] = (2 * f_j[r]) * kO16Stride + f_p[r];
            f_hi[r] = (2 * f_j[r] + 1) * kO16Stride + f_p[r];
        }
        auto flush = [&](int64_t tp) {
            const int64_t p0 = tp * 64;
            const uint16_t* o16 = reinterpret_cast<const uint16_t*>(otile);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (f_p[r] < 64 && p0 + f_p[r] < n) {
                    uint32_t v = (uint32_t)o16[f_lo[r]] | ((uint32_t)o16[f_hi[r]] << 16);
                    if (status && status[p0 + f_p[r]]) v = 0u;
                    out[(p0 + f_p[r]) * words + f_j[r]] = v;
                }
            }
        };
        // one test: 8 corner loads from the lane's addresses, packed sums, threshold compare,
        // append the sign bits (bit j of the unit at position j: tests walked high to low)
        uint32_t wA = 0, wB = 0;
        auto test = [&](const uint32_t (&adr)[8], int j) {
            uint32_t cv[8];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                BD_CHECK(adr[cc] >= IIbase && adr[cc] < IIbase + kIIBytes);
                asm("ld.shared.u32 %0, [%1];" : "=r"(cv[cc]) : "r"(adr[cc]));
            }
            const uint32_t S1 = cv[0] - cv[1] - cv[2] + cv[3];
            const uint32_t S2 = cv[4] - cv[5] - cv[6] + cv[7];
            int eA, eB;
            if (DP2A) {
                const int m1 = rm[j], m2 = rm[j] << 8, nthr1 = rn[j];  // m2: bytes (0, A2, 0, -A1)
                eA = dp2a_hi(S2, m1, dp2a_lo(S1, m1, nthr1));
                eB = dp2a_hi(S2, m2, dp2a_lo(S1, m2, nthr1));
            } else {
                const int4 th = cthr[ub + j];
                eA = (int)(S1 & 0xffffu) * th.z + ((int)(S2 & 0xffffu) * th.y + th.x);
                eB = (int)(S1 >> 16) * th.z + ((int)(S2 >> 16) * th.y + th.x);
            }
            wA = __funnelshift_l((uint32_t)eA, wA, 1);
            wB = __funnelshift_l((uint32_t)eB, wB, 1);
        };
        int k = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
            if (k > 0) flush(t - gridDim.x);
            // ------------- integral (a1): row prefixes of the MMA's column prefixes -------------
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                mbar_wait(&dfull[g], (uint32_t)h);  // use 2k + h of buffer g: parity h
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dg = tmem + ((uint32_t)(32 * q) << 16) + 128u * (uint32_t)g + 64u * (uint32_t)(c & 1);
                uint32_t ca[2][16], cb[2][16];
                tmem_ld16(dg, ca[0]);
                tmem_ld16(dg + 32, cb[0]);
                tmem_ld16(dg + 16, ca[1]);
                tmem_ld16(dg + 48, cb[1]);
                tmem_wait16(ca[0]);
                tmem_wait16(cb[0]);
                tmem_wait16(ca[1]);
                tmem_wait16(cb[1]);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&dempty[g]);  // the buffer's next MMAs overlap the prefixes below
                const int P = 16 * h + 8 * g + 2 * q + (c & 1);  // pair of the tile
                const uint32_t adr = IIbase + 4u * (uint32_t)(lane * kRowWords + P);
                uint32_t run = 0;
#pragma unroll
                for (int x = 0; x < 32; ++x) {
                    run += __byte_perm(ca[x >> 4][x & 15], cb[x >> 4][x & 15], 0x5410);
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(adr + 4u * 33u * (uint32_t)x), "r"(run) : "memory");
                }
            }
            named_sync(1, kWarps * 32);  // integral complete
            // ------------- tests (a3) and bit packing (a4) -------------
            if (active) {
                wA = 0;
                wB = 0;
                // tests 15..8: addresses from TMEM, one test ahead
                uint32_t ta[2][8];
                tmem_ld8(trec + 8u * (kTmemTests - 1), ta[1]);
                tmem_wait8(ta[1]);
#pragma unroll
                for (int j = 15; j >= 16 - kTmemTests; --j) {
                    const int t8 = j - (16 - kTmemTests);
                    if (t8 > 0) tmem_ld8(trec + 8u * (uint32_t)(t8 - 1), ta[(j - 1) & 1]);
                    test(ta[j & 1], j);
                    if (t8 > 0) tmem_wait8(ta[(j - 1) & 1]);
                }
                // tests 7..0: broadcast byte-offset records from shared memory, one test ahead
                const uint4* rec = crec + 2 * ub;
                uint4 r0 = rec[2 * (15 - kTmemTests)], r1 = rec[2 * (15 - kTmemTests) + 1];
#pragma unroll
                for (int j = 15 - kTmemTests; j >= 0; --j) {
                    const uint32_t adr[8] = {IIl + r0.x, IIl + r0.y, IIl + r0.z, IIl + r0.w,
                                             IIl + r1.x, IIl + r1.y, IIl + r1.z, IIl + r1.w};
                    if (j > 0) {
                        r0 = rec[2 * (j - 1)];
                        r1 = rec[2 * (j - 1) + 1];
                    }
                    test(adr, j);
                }
                otile[(warp * kO16Stride) / 2 + lane] = (wA & 0xffffu) | (wB << 16);
            }
            named_sync(1, kWarps * 32);  // tests done before the next integral overwrites this one
        }
        if ((int64_t)blockIdx.x < n_tiles) {
            const int64_t last = blockIdx.x + (n_tiles - 1 - blockIdx.x) / gridDim.x * gridDim.x;
            flush(last);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace kern_tc

using namespace kern_tc;
cudaError_t launch_bad_patches_tc(const uint8_t* patches, int64_t n, const PatchTable& tab, int K, uint32_t* out,
                                  const uint8_t* status, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (K > 256 || K % 16 != 0 || n > ((int64_t)1 << 30)) return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem_attr((const void*)bad_patch_tc_kernel<true>, kSmemBytes);
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)bad_patch_tc_kernel<false>, kSmemBytes);
    if (e != cudaSuccess) return e;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap map;  // {32 columns, 32 rows, n patches}, box 32 x 32 x 32, SWIZZLE_32B, OOB = 0
    const cuuint64_t dims[3] = {32, 32, (cuuint64_t)n};
    const cuuint64_t strides[2] = {32, 1024};
    const cuuint32_t box[3] = {32, 32, 32};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(patches), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    TcTable tt;
    memset(&tt, 0, sizeof(tt));
    for (int k = 0; k < K; ++k) {
        const PatchTest& T = tab.t[k];
        uint32_t w[8];
        for (int c = 0; c < 8; ++c) w[c] = 4u * conv_off(T.off[c]);
        tt.off[k][0] = make_uint4(w[0], w[1], w[2], w[3]);
        tt.off[k][1] = make_uint4(w[4], w[5], w[6], w[7]);
        tt.thr[k] = make_int4(T.nthr1, T.m1, T.m2, 0);
    }
    const int64_t tiles = (n + 63) / 64;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    ProfScope ps("bad_patch", s);
    if (tab.dp2a)
        bad_patch_tc_kernel<true><<<grid, kThreads, kSmemBytes, s>>>(map, n, out, K, status, tt);
    else
        bad_patch_tc_kernel<false><<<grid, kThreads, kSmemBytes, s>>>(map, n, out, K, status, tt);
    return cudaGetLastError();
}

}  // namespace bd
