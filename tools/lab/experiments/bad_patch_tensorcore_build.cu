// EXPERIMENT (not built into the product; DESIGN.md §5.3 "tensor-core integral build"):
// the c2 BAD kernel with the integral's column prefix on the tensor cores (tcgen05.mma kind::i8,
// L * P with L lower-triangular ones, B = TMA SWIZZLE_32B pixels as an MN-major operand), a
// producer warp for TMA + MMA, row prefixes in registers from tcgen05.ld.  Bit-exact (all patch
// parity tests green on B200) but slower than the CUDA-core build: 1.85-2.4 ms vs 1.50 ms for
// configs[2].  Compiled only by tools/lab/bp_timing.cu (phase timestamps).
// bad_patch.cu — §8(a) rows a1, a3, a4 on 32x32 patches (configs[2]; configs[4] BAD on the
// warped patch, R20).  Fixed geometry (centre (16,16), scale 1, angle 0, R7), so every
// test's 8 integral-image corners, both clamped areas and the exact integer threshold
// floor(theta*A1*A2) are known at bad_create (PatchTable, passed by value as a kernel
// parameter).
//
// Design.  The kernel is bound by the SM's L1/shared-memory data pipe:
// the K tests read 8 integral corners each, and building the integral on CUDA cores (pixel
// staging reads, row-scan shuffles, stores) cost as much pipe time as the tests.  Here the
// integral's column prefix runs on the tensor cores, otherwise idle, and the pipe carries
// little more than the corner reads and one store per integral entry:
//  * Persistent CTAs, 1 per SM, 16 warps; a tile is 64 patches = 32 PAIRS = 8 groups of 8.
//  * Packed pair integral: the integral of A + 65536*B (A, B two patches) with 32-bit adds;
//    box sums are linear and every box sum < 2^16 (<= 225*255), so one 32-bit load yields both
//    patches' box sums exactly (S_A = low half, S_B = high half).
//  * Staging: each group's 8 patches arrive by one TMA tensor load (2-D view [n*32 rows][32],
//    box 32 x 256, SWIZZLE_32B) into its own 8 KB slot (8 slots = one tile); a slot is refilled
//    with the next tile's group as soon as the MMAs that read it have completed.
//  * Column prefix on the tensor cores (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM):
//    C = L * P with L the 32x32 lower-triangular ones matrix.  Per group and lane quarter q
//    one MMA (M = 128, N = 64, K = 32): A = rows 32q..32q+31 of blockdiag(L) (K-major, a
//    window into one zero-padded 7 KB buffer), B = the pixels of pair 4g + q straight from the
//    staging slot as an MN-major SWIZZLE_32B operand (N = the 2 x 32 columns of the pair, K =
//    the 32 rows: the natural [patch][y][x] layout, LBO = 1024 B, SBO = 256 B); the 4 MMAs of
//    a group accumulate into one 64-column D, quarter q holding pair q's column prefixes.
//  * Row prefix in registers: tcgen05.ld.32x32b gives thread y of the quarter row y of its
//    pair (32 columns of A and of B); it packs A + (B << 16), runs the 32-column prefix with
//    32-bit adds and stores the row's 32 entries.  Integral rows are 1057 words apart (32 x 33
//    + 1), so the 32 lanes' stores (one row each, same column) hit 32 banks.
//  * A 17th warp is the producer: one lane issues every TMA load and every MMA.  TMEM holds
//    256 columns of test records and 4 D slots of 64 columns; group g of a tile uses slot g % 4,
//    so the MMAs of groups 4..7 run while the 16 compute warps store groups 0..3, and the next
//    tile's groups 0..3 while they store 4..7 and run the tests.  A staging slot is refilled as
//    soon as the MMAs that read it have completed (a ring of 8 groups at K <= 256, 6 at K <= 512:
//    most of a tile of lead for the HBM stream).  Compute warp (q, c) = (warp % 4, warp / 4)
//    builds groups c and c + 4 from TMEM lane quarter q (pair 4g + q).
//  * smem integral layout: word (y-1)*1057 + (x-1)*33 + pair for y, x in 1..32, plus a zero
//    entry (32*1057 + pair) for row / column 0: the test phase (lane = pair, uniform entry) is
//    conflict-free.
//  * Tests (all 16 warps): the K tests form units of U = 16 (K <= 256) or 32 (K <= 512)
//    consecutive tests, at most one per warp.  For the first 8 tests of every unit the lane's 8
//    corner ADDRESSES (integral base + its pair word + offset) sit in TENSOR MEMORY (written once
//    per CTA, read per test with tcgen05.ld one test ahead: no address arithmetic and no record
//    traffic on the L1 data pipe that the corner loads saturate); the other tests read their
//    record by two broadcast LDS.128.  When every clamped area fits a signed byte (radii <= 5)
//    the thresholds of tests 0..15 stay in registers.  Per test and lane (= pair): 8 corner
//    loads, packed S1/S2, then either 2 DP2A per patch on the PACKED sums (area bytes select the
//    16-bit half: PatchTest) or 2 unpacks + 2 IMADs per patch, and a funnel shift that appends
//    the sign bit (tests walked high to low so bit j lands at position j, R16).
//  * Output: each warp writes its unit's bits into a unit-major output tile; the tile leaves
//    in coalesced rows at the start of the next tile.
#include "../../../paper_2108_08380_b200/csrc/internal.cuh"
#include "../../../paper_2108_08380_b200/csrc/tc.cuh"

namespace bd {
namespace kern {

constexpr int kWarps = 16;                                   // compute warps (+ 1 producer warp)
constexpr int kThreads = (kWarps + 1) * 32;
constexpr int kRowWords = 32 * 33 + 1;                       // integral row stride (words)
constexpr int kZeroWord = 32 * kRowWords;                    // 33824: zero entry of pair 0
constexpr int kIIWords = kZeroWord + 33;
constexpr int kIIBytes = kIIWords * 4;                       // 135428
constexpr int kIIBytesAligned = (kIIBytes + 1023) / 1024 * 1024;  // 136192
constexpr int kSlotBytes = 32 * 1024;                        // half a tile: 32 patches
constexpr int kZGroups = 28;                                 // blockdiag(L) window buffer
constexpr int kZBytes = kZGroups * 256;                      // 7168
constexpr int kO16Stride = 68;                               // halfwords per unit row (U = 16)
constexpr int kO32Stride = 66;                               // words per unit row (U = 32)
constexpr int kOutBytes = kWarps * kO32Stride * 4;           // 4224
constexpr int kBarBytes = 256;
// staging ring: a full tile (8 groups) at K <= 256; 6 groups at K <= 512 (the records double)
template <int U>
constexpr int slots_of() { return U == 16 ? 2 : 1; }
template <int U>
constexpr int smem_bytes() {
    return 1024 /* alignment slack */ + kIIBytesAligned + slots_of<U>() * kSlotBytes + kZBytes +
           16 * U * (int)sizeof(PatchTest) + kOutBytes + kBarBytes;  // U=16: 226688, U=32: 222592
}
// instruction descriptor, kind::i8: D s32, A u8 K-major, B u8 MN-major, N = 256, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 16) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

using namespace tc;  // smem_addr, mbarriers, mma_commit, tmem_ld32

// phase timestamps of CTA 0 (tools/lab/bp_timing.cu compiles this file with BD_BP_TIMING)
#ifdef BD_BP_TIMING
__device__ long long g_bp_t[64][16];
__device__ long long g_bp_p[64][8][4];  // producer: per half (dempty done, full done, issued, refill done)
#define BP_PMARK(tile, g, i)                                                           \
    do {                                                                               \
        if (blockIdx.x == 0 && (tile) < 64) g_bp_p[(tile)][(g)][(i)] = clock64();      \
    } while (0)
#define BP_MARK(tile, i)                                                     \
    do {                                                                     \
        if (blockIdx.x == 0 && (tile) < 64) g_bp_t[(tile)][(i)] = clock64(); \
    } while (0)
#else
#define BP_MARK(tile, i) \
    do {                 \
    } while (0)
#define BP_PMARK(tile, g, i) \
    do {                     \
    } while (0)
#endif

// UMMA shared-memory descriptor (sm_100 version 1) with explicit LBO / SBO and layout type
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// producer-side wait: try_wait with a short nanosleep back-off, so the producer warp does not
// take issue slots from the compute warps on its SM sub-partition while it waits
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (true) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (done) break;
        __nanosleep(40);
    }
}

__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %4, p;\n}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(acc), "r"(kIdesc)
        : "memory");
}

// 32 patches [p, p + 32) (3-D tensor {32 columns, 32 rows, n patches}, box 32 x 32 x 32)
__device__ __forceinline__ void tma_load_patches(void* dst, const CUtensorMap* map, int p, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(0), "r"(p), "r"(smem_addr(bar))
        : "memory");
}

// DP2A on the packed box sums: c + S.lo16 * m.byte0 + S.hi16 * m.byte1 (.lo) or
// m.byte2 / m.byte3 (.hi); S halves unsigned, m bytes signed (PatchTest, dp2a form)
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

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
// wait for the outstanding tcgen05.ld; the registers pass through the asm so no use of them
// can be scheduled above the wait
__device__ __forceinline__ void tmem_wait8(uint32_t (&v)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
                 :
                 : "memory");
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
__device__ __forceinline__ void tmem_wait32(uint32_t (&v)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                   "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                   "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                   "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
                 :
                 : "memory");
}

// the table's entry-major byte offsets (api.cu: entry e = (y-1)*32 + (x-1), 1024 = zero entry,
// 33 words x 4 bytes per entry) -> this kernel's word offsets (row stride kRowWords)
__device__ __forceinline__ uint32_t conv_off(uint32_t byte_off) {
    const uint32_t e = byte_off / 132u;
    return e >= 1024u ? (uint32_t)kZeroWord : (e >> 5) * (uint32_t)kRowWords + (e & 31u) * 33u;
}

template <int U, bool DP2A>
__global__ void __launch_bounds__(kThreads, 1)
    bad_patch_kernel(const __grid_constant__ CUtensorMap map, int64_t n, uint32_t* __restrict__ out, int K,
                     const uint8_t* __restrict__ status, const __grid_constant__ PatchTable tab) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    debug_poison_smem(smem_raw);
    const uint32_t raw = smem_addr(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);  // 1024-aligned (SWIZZLE_32B slots)
    uint32_t* II = reinterpret_cast<uint32_t*>(smem);
    uint8_t* stg = smem + kIIBytesAligned;
    constexpr int kSlots = slots_of<U>();
    uint8_t* Z = stg + kSlots * kSlotBytes;
    PatchTest* stab = reinterpret_cast<PatchTest*>(Z + kZBytes);       // [K] records, this layout
    uint32_t* otile = reinterpret_cast<uint32_t*>(Z + kZBytes + 16 * U * sizeof(PatchTest));
    uint64_t* bars = reinterpret_cast<uint64_t*>(Z + kZBytes + 16 * U * sizeof(PatchTest) + kOutBytes);
    uint64_t* full = bars;          // [kSlots] staging slot landed (TMA)
    uint64_t* dfull = bars + 8;     // D (half a tile) computed (tcgen05.commit)
    uint64_t* dempty = bars + 9;    // D read out (16 compute warps)
    __shared__ uint32_t s_tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_tiles = (n + 63) / 64;
    const int words = K >> 5;
    const int units = K / U;  // <= kWarps

    // ---------------- setup ----------------
    const bool producer = warp == kWarps;
    if (threadIdx.x < 33) II[kZeroWord + threadIdx.x] = 0u;  // zero entry (corners in row / column 0)
    for (int i = threadIdx.x; i < kZBytes; i += blockDim.x) {  // blockdiag(L) window: L in groups 12..15
        const int g = i >> 8, w = i & 255, kc = w >> 7, r = (w & 127) >> 4, kk = w & 15;
        const int m = (g - 12) * 8 + r, kx = kc * 16 + kk;  // L[m][kx] = [kx <= m]
        Z[i] = (g >= 12 && g < 16 && kx <= m) ? 1 : 0;
    }
    for (int i = threadIdx.x; i < K; i += blockDim.x) {  // records with byte offsets of this layout
        PatchTest T = tab.t[i];
#pragma unroll
        for (int c = 0; c < 8; ++c) T.off[c] = 4 * conv_off(T.off[c]);
        stab[i] = T;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i) mbar_init(&full[i], 1);
        mbar_init(dfull, 1);
        mbar_init(dempty, kWarps);
        mbar_init(dempty + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_addr(&s_tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // Z visible to the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem_base;
    constexpr int kTm = 8;  // tests per unit with TMEM records
    // this warp's record columns: lanes 32 (warp % 4) .., columns 64 (warp / 4) + 8 j
    const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
    if (warp < units && !producer) {
        // per-lane ABSOLUTE corner addresses (integral base + this lane's pair word + offset)
        const uint32_t IIl0 = smem_addr(II + lane);
#pragma unroll
        for (int j = 0; j < kTm; ++j) {
            const uint4* Tq = reinterpret_cast<const uint4*>(stab + warp * U + j);
            const uint4 o0 = Tq[0], o1 = Tq[1];
            const uint32_t v[8] = {IIl0 + o0.x, IIl0 + o0.y, IIl0 + o0.z, IIl0 + o0.w,
                                   IIl0 + o1.x, IIl0 + o1.y, IIl0 + o1.z, IIl0 + o1.w};
            tmem_st8(tq + 8 * j, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // DP2A form: the thresholds and area-byte words of the unit's tests 0..15 stay in registers
    // (m2 = m1 << 8); tests 16..31 (U = 32) read their broadcast records
    int rn[16], rm[16];
    if (DP2A) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const PatchTest& T = tab.t[(warp < units ? warp : 0) * U + j];
            rn[j] = T.nthr1;
            rm[j] = T.m1;
        }
    }

    const uint32_t zaddr = smem_addr(Z), saddr = smem_addr(stg);
    const uint32_t dbase = tmem + 256u;  // D: columns 256..511 (half a tile)

    // ---------------- producer warp: TMA loads and MMAs (one lane) ----------------
    if (producer) {
        if (lane == 0) {
            // use u = 2 k + h: half h of this CTA's k-th tile; staging slot u % kSlots
            const int64_t my_tiles = (int64_t)blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
            const int64_t uses = 2 * my_tiles;
            auto load = [&](int64_t u) {  // TMA of use u (32 patches) into its slot
                const int sl = (int)(u % kSlots);
                const int64_t tile = blockIdx.x + (u >> 1) * gridDim.x;
                mbar_expect_tx(&full[sl], (uint32_t)kSlotBytes);
                tma_load_patches(stg + sl * kSlotBytes, &map, (int)(tile * 64 + (u & 1) * 32), &full[sl]);
            };
            for (int64_t u = 0; u < kSlots && u < uses; ++u) load(u);
            for (int64_t u = 0; u < uses; ++u) {
                const int sl = (int)(u % kSlots);
                if (u > 0) mbar_wait_sleep(dempty, (uint32_t)((u - 1) & 1));  // previous half read out of TMEM
#ifdef BD_BP_NOOVERLAP
                if (u > 0 && (u & 1) == 0) mbar_wait_sleep(dempty + 1, (uint32_t)(((u >> 1) - 1) & 1));
#endif
                BP_PMARK(u >> 1, u & 1, 0);
                mbar_wait_sleep(&full[sl], (uint32_t)((u / kSlots) & 1));
                BP_PMARK(u >> 1, u & 1, 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {  // patches 8 qq .. 8 qq + 7 of the half -> lane quarter qq
                    const uint64_t ad = umma_desc(zaddr + (uint32_t)(12 - 4 * qq) * 256u, 128, 256, 0);
                    const uint64_t bd = umma_desc(saddr + (uint32_t)(sl * kSlotBytes + 8 * qq * 1024), 1024, 256, 6);
                    mma_u8(dbase, ad, bd, qq > 0 ? 1u : 0u);
                }
                mma_commit(dfull);
                BP_PMARK(u >> 1, u & 1, 2);
                if (u + kSlots < uses) {  // the slot is free once these MMAs complete: use u + kSlots
                    mbar_wait_sleep(dfull, (uint32_t)(u & 1));
                    load(u + kSlots);
                }
                BP_PMARK(u >> 1, u & 1, 3);
            }
        }
        __syncwarp();
    } else {
    // ---------------- 16 compute warps ----------------
    // half h: warp (q, j) = (warp % 4, warp / 4) builds pair 16 h + 4 q + j from TMEM lane
    // quarter q, columns 64 j (the MMA of quarter q covers patches 8 q .. 8 q + 7 of the half)
    const int q = warp & 3, c = warp >> 2;
    const uint32_t dmine = dbase + ((uint32_t)(32 * q) << 16) + 64u * (uint32_t)c;

    // coalesced store of tile tp's descriptors from the output tile (all 512 threads, at most
    // two words each; the thread -> (patch, word) map and the shared-memory offsets are loop
    // invariants).  Rows of invalid keypoints (status != 0) are written as zero.
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

    const uint32_t IIbase = smem_addr(II);
    int k = 0;  // tile iteration of this CTA (staging / D phases)
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        if (warp == 0 && lane == 0) BP_MARK(k, 0);
        if (k > 0) flush(t - gridDim.x);  // the previous tile's bits
        // ------------- build the packed pair integrals (a1, on chip) -------------
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            mbar_wait(dfull, (uint32_t)rr);  // use 2k + rr
            if (warp == 0 && lane == 0) BP_MARK(k, 1 + rr);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // thread y = row y of pair P: column prefixes of patch A (cols 0..31) and B (32..63),
            // in two halves of 16 columns (registers)
            uint32_t ca[2][16], cb[2][16];
            const uint32_t dg = dmine;
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
            if (lane == 0) mbar_arrive(dempty);
            // row prefix of the packed pair A + 65536 B (mod 2^32), stored as integral row y + 1
            const int P = 16 * rr + 4 * q + c;
            const uint32_t adr = IIbase + 4u * (uint32_t)(lane * kRowWords + P);
            uint32_t run = 0;
#pragma unroll
            for (int x = 0; x < 32; ++x) {
                run += __byte_perm(ca[x >> 4][x & 15], cb[x >> 4][x & 15], 0x5410);
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(adr + 4u * 33u * (uint32_t)x), "r"(run) : "memory");
            }
        }
        if (warp == 0 && lane == 0) BP_MARK(k, 3);
        named_sync(1, kWarps * 32);  // integral complete
        if (warp == 0 && lane == 0) BP_MARK(k, 4);
        // ------------- K tests per patch pair (a3) and bit packing (a4) -------------
        if (warp < units) {
            const uint32_t IIl = IIbase + 4u * (uint32_t)lane;  // lane = pair
            uint32_t wA = 0, wB = 0;
            uint32_t ob[2][8];  // TMEM records of one test, double buffered
            tmem_ld8(tq + 8 * (kTm - 1), ob[(kTm - 1) & 1]);
            uint4 so[2][2];     // shared-memory records of one test, loaded one test ahead
            {
                const uint4* T0 = reinterpret_cast<const uint4*>(stab + warp * U + U - 1);
                so[(U - 1) & 1][0] = T0[0];
                so[(U - 1) & 1][1] = T0[1];
            }
#pragma unroll
            for (int j = U - 1; j >= 0; --j) {
                const uint4* Tq = reinterpret_cast<const uint4*>(stab + warp * U + j);
                uint32_t adr[8];  // shared-window addresses of this lane's 8 corners
                if (j < kTm) {  // this test's records have landed; fetch the next test's
                    tmem_wait8(ob[j & 1]);
                    if (j > 0) tmem_ld8(tq + 8 * (j - 1), ob[(j - 1) & 1]);
#pragma unroll
                    for (int c = 0; c < 8; ++c) adr[c] = ob[j & 1][c];
                } else {
                    if (j - 1 >= kTm) {  // next test's broadcast records
                        so[(j - 1) & 1][0] = Tq[-3];
                        so[(j - 1) & 1][1] = Tq[-2];
                    }
                    const uint4 o0 = so[j & 1][0], o1 = so[j & 1][1];
                    adr[0] = IIl + o0.x; adr[1] = IIl + o0.y; adr[2] = IIl + o0.z; adr[3] = IIl + o0.w;
                    adr[4] = IIl + o1.x; adr[5] = IIl + o1.y; adr[6] = IIl + o1.z; adr[7] = IIl + o1.w;
                }
                const uint4 q2 = (DP2A && j < 16) ? make_uint4((uint32_t)rn[j], (uint32_t)rm[j], (uint32_t)rm[j] << 8, 0u)
                                                  : Tq[2];  // thresholds (broadcast)
                if (BD_DEBUG) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) BD_CHECK(adr[c] >= IIbase && adr[c] < IIbase + kIIBytes);
                }
                uint32_t cv[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) asm("ld.shared.u32 %0, [%1];" : "=r"(cv[c]) : "r"(adr[c]));
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
        if (warp == 0 && lane == 0) BP_MARK(k, 5);
#ifdef BD_BP_NOOVERLAP
        if (warp == 0 && lane == 0) mbar_arrive(dempty + 1);
#endif
        named_sync(1, kWarps * 32);  // tests done before the next build overwrites the integral
        if (warp == 0 && lane == 0) BP_MARK(k, 6);
    }
    if ((int64_t)blockIdx.x < n_tiles) {  // the last tile's bits
        const int64_t last = blockIdx.x + (n_tiles - 1 - blockIdx.x) / gridDim.x * gridDim.x;
        flush(last);
    }
    }  // compute warps
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace kern

using namespace kern;
cudaError_t launch_bad_patches(const uint8_t* patches, int64_t n, const PatchTable& tab, int K, uint32_t* out,
                               const uint8_t* status, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (n > ((int64_t)1 << 30)) return cudaErrorInvalidValue;  // TMA patch coordinates are int32
    cudaError_t e = ensure_smem_attr((const void*)bad_patch_kernel<16, true>, smem_bytes<16>());
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)bad_patch_kernel<32, true>, smem_bytes<32>());
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)bad_patch_kernel<16, false>, smem_bytes<16>());
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)bad_patch_kernel<32, false>, smem_bytes<32>());
    if (e != cudaSuccess) return e;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    // the patches as a 3-D u8 tensor {32 columns, 32 rows, n}, box 32 x 32 x 32 (half a tile),
    // SWIZZLE_32B = the MN-major SW32 UMMA operand layout; patches beyond n read as 0
    CUtensorMap map;
    const cuuint64_t dims[3] = {32, 32, (cuuint64_t)n};
    const cuuint64_t strides[2] = {32, 1024};
    const cuuint32_t box[3] = {32, 32, 32};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(patches), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    const int64_t tiles = (n + 63) / 64;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    ProfScope ps("bad_patch", s);
    if (K <= 16 * kWarps) {
        if (tab.dp2a)
            bad_patch_kernel<16, true><<<grid, kThreads, smem_bytes<16>(), s>>>(map, n, out, K, status, tab);
        else
            bad_patch_kernel<16, false><<<grid, kThreads, smem_bytes<16>(), s>>>(map, n, out, K, status, tab);
    } else {
        if (tab.dp2a)
            bad_patch_kernel<32, true><<<grid, kThreads, smem_bytes<32>(), s>>>(map, n, out, K, status, tab);
        else
            bad_patch_kernel<32, false><<<grid, kThreads, smem_bytes<32>(), s>>>(map, n, out, K, status, tab);
    }
    return cudaGetLastError();
}

}  // namespace bd
