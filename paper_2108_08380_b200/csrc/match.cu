// match.cu — SURVEY §8(f) NEXT-1: brute-force Hamming nearest neighbours and mutual NN over
// binary descriptor sets (P:559-560 / P:566-570 "BFMatcher with Mutual Nearest Neighbors";
// S:514-540 tie rule: lowest index).
//
// The paper's similarity S(x, y) = h(x)^T h(y) with h in {-1, +1}^K equals
// K - 2 Hamming(x, y) exactly, so the all-pairs similarity of a query block A (n_a x K) and a
// train block B (n_b x K) is the dense contraction S = A_pm B_pm^T, computed EXACTLY on the
// tensor cores as a block-scaled FP4 GEMM (tcgen05 kind::mxf4): +-1 is an e2m1 value, every
// ue8m0 block scale is 1.0, products are +-1 and the f32 accumulator holds integers
// |S| <= 512 exactly (kind::mxf4 runs at twice the kind::i8 rate on half the operand bytes).
// The nearest neighbour of row i is the argmax of S[i, :] (first maximum = lowest index on
// ties); dist = (K - S)/2.
// Design:
//  * expand: bits -> packed e2m1 rows (bit 1 -> +1.0 = 0x2, bit 0 -> -1.0 = 0xA), one thread
//    per 32-bit word, one 16-byte store;
//  * work list: (direction, pair, 256-row query tile) items, both directions in one launch,
//    built on the device from one small offsets table;
//  * match: persistent CTA PAIRS (tcgen05 cta_group::2) — per 64 values of K one MMA with
//    M = 256, N = 224 issued by the leader; each CTA holds its 128 query rows (double buffered
//    across items) and half of every 224-row train tile (an 8-stage ring of 14 KB K-atoms);
//    8 epilogue warps per CTA read the 128 x 224 f32 accumulator (two TMEM buffers; the last
//    64 TMEM columns hold the block scales) and keep a running (max S, first index) per
//    row — see the kernel's comment;
//  * mutual: nn_ba[nn_ab[i]] == i.
#include <algorithm>
#include <type_traits>
#include <vector>

#include "internal.cuh"
#include "tc.cuh"

namespace bd {
namespace kern {

constexpr int kMT = 128;                  // query rows per CTA (the pair's MMA has M = 256)
constexpr int kEpiWarps = 8;              // 2 per TMEM lane quarter, one per column half
constexpr int kMmaWarp = kEpiWarps, kTmaWarp = kEpiWarps + 1;
constexpr int kMThreads = (kEpiWarps + 2) * 32;
constexpr int kNT = 224;                  // train rows per tile (MMA N), 112 per CTA
constexpr int kHalfCols = kNT / 2;        // accumulator columns per epilogue warp
constexpr int kAtomBytes = kMT * 128;     // one SWIZZLE_128B atom of the query tile: 128 rows x 256 e2m1 values
constexpr int kBAtomBytes = (kNT / 2) * 128;  // one CTA's half of a train-tile atom (14 KB)
constexpr int kBStages = 8;               // train-atom ring (112 KB)
constexpr int kDBufs = 2;                 // TMEM accumulators (2 x 224 columns)
constexpr uint32_t kSfCol = kDBufs * kNT; // TMEM columns 448..511: block scale factors, all 1.0

// bits -> packed e2m1 values, +1.0 (0x2) for a 1 bit and -1.0 (0xA) for a 0 bit, element e
// in nibble e % 2 of byte e / 2 (any consistent order works: the dot product is a sum);
// one thread per 32-bit word, one 16-byte store
__global__ void expand_pm1_kernel(const uint32_t* __restrict__ bits, int64_t n_words, uint8_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_words) return;
    const uint32_t w = __ldg(bits + i);
    uint32_t q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) v |= (((w >> (8 * k + b)) & 1u) ? 0x2u : 0xAu) << (4 * b);
        q[k] = v;
    }
    *reinterpret_cast<uint4*>(out + i * 16) = make_uint4(q[0], q[1], q[2], q[3]);
}

struct MatchWork {
    int32_t a0, na, b0, nb;  // query rows [a0, a0+na) (this tile), train rows [b0, b0+nb)
    int32_t a_pair0;         // first query row of the pair (nn indices are pair-relative)
    int32_t dir;             // 0: queries from a, train from b; 1: the reverse
    int32_t pad[2];
};

struct MatchOut {
    int32_t* nn[2];
    int32_t* dist[2];
};

using tc::smem_addr;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// the address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA 2-D tile load into this CTA's shared memory, completing on an mbarrier of the CTA pair
// (here: always the leader's)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
}
// block-scaled e2m1 MMA (kind::mxf4, one ue8m0 scale per 32 values, read from TMEM)
__device__ __forceinline__ void mma_f4_pair(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc,
                                            uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
        : "memory");
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
// maximum of C (32 or 16) floats held as bits: a 3-input max tree
template <int C>
__device__ __forceinline__ float chunk_max(const uint32_t* v) {
    auto f = [&](int i) { return __uint_as_float(v[i]); };
    if (C == 32) {
        float m[11];
#pragma unroll
        for (int i = 0; i < 10; ++i) m[i] = fmax3(f(3 * i), f(3 * i + 1), f(3 * i + 2));
        m[10] = fmaxf(f(30), f(31));
        const float a = fmax3(m[0], m[1], m[2]), b = fmax3(m[3], m[4], m[5]), c = fmax3(m[6], m[7], m[8]);
        return fmaxf(fmax3(a, b, c), fmaxf(m[9], m[10]));
    } else {
        float m[6];
#pragma unroll
        for (int i = 0; i < 5; ++i) m[i] = fmax3(f(3 * i), f(3 * i + 1), f(3 * i + 2));
        m[5] = f(15);
        return fmaxf(fmax3(m[0], m[1], m[2]), fmax3(m[3], m[4], m[5]));
    }
}
// arrive on the mbarrier at this offset in both CTAs of the pair when the MMAs issued so far complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_addr(bar)),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
#ifdef BD_DEBUG_CHECKS
    // debug build: a lost arrival traps (block, thread, parity) instead of hanging
    uint32_t done = 0;
    for (uint64_t spin = 0; !done; ++spin) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (spin == (1ull << 26)) {
            printf("bindesc debug: cluster mbarrier wait timed out (block %d thread %d parity %u)\n", blockIdx.x,
                   threadIdx.x, parity);
            __trap();
        }
    }
#else
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
#endif
}

// CTA PAIRS (cta_group::2, cluster of 2 on one TPC), persistent: pair c takes work items c,
// c + pairs, ...; both directions in one launch.  A work item is a 256-row query tile against
// the pair's train rows in 224-row tiles: one tcgen05.mma.cta_group::2.kind::mxf4 (M = 256,
// N = 224, K = 64) per 32 bytes of packed K, issued by the leader; each CTA holds its 128 query
// rows and HALF of each train tile (112 rows), so per SM the operand reads and the TMA writes
// stay within the 128 B/cycle of shared memory, where one CTA with M = 128 spends its whole
// shared-memory bandwidth on operand reads and the train-tile writes stretch the MMAs
// (measured with kind::i8: ~1500 cycles per 16-MMA tile at M = N = 128, 1.25x at N = 256).
// Shared memory per CTA: its query rows double buffered (the next item's land under this
// item) and a ring of kBStages 14 KB train atoms (112 rows x 128 bytes of packed K).  TMEM per
// CTA: two 224-column f32 accumulators (its 128 query rows x the tile's 224 train rows) and
// 64 columns of ue8m0 block scales, all 1.0 (written once; read by every MMA).
// Barriers: TMA bytes of both CTAs complete on the LEADER's aready/full; MMA commits arrive
// on afree/empty/dfull in BOTH CTAs (multicast), so each CTA's producer refills its own
// stages and each epilogue reads its own accumulator; dfree (leader) counts the 4 epilogue
// warps of both CTAs.
// NK = ceil(K / 64) MMAs per tile, compile-time: the issue loop adds constant offsets to
// descriptors built once per stage (rebuilding them per MMA in a runtime loop capped the
// issuing lane at ~80 cycles per 64-cycle MMA: tools/lab/mma_tile_lab.cu).  K not a multiple
// of 64: the tensor maps' rows end at K / 2 bytes, so the TMA zero-fills the rest of the last
// 32-byte K step in both operands (e2m1 zero adds nothing).
template <int NK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kMThreads, 1)
    match_kernel(const __grid_constant__ CUtensorMap tq0, const __grid_constant__ CUtensorMap tt0,
                 const __grid_constant__ CUtensorMap tq1, const __grid_constant__ CUtensorMap tt1,
                 const MatchWork* __restrict__ work, int n_items, int K, MatchOut out) {
    // direction 0: query rows of a (tq0), train rows of b (tt0); direction 1: tq1 over b, tt1 over a
    using namespace tc;
    constexpr int kAtoms = (NK + 3) / 4;  // 128-byte K atoms = 256 e2m1 values = 4 MMAs
    constexpr int kABytes = kAtoms * kAtomBytes;
    extern __shared__ uint8_t smem_raw[];
    debug_poison_smem(smem_raw);
    __shared__ uint64_t aready[2], afree[2], full[kBStages], empty[kBStages], dfull[kDBufs], dfree[kDBufs];
    __shared__ uint32_t tmem_base_s;
    __shared__ int2 merge[kMT];
    const uint32_t raw = smem_addr(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = base;                // 2 x this CTA's 128 query rows
    uint8_t* sB = base + 2 * kABytes;  // kBStages train atoms (this CTA's 128 rows of each tile)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int n_local = pair < n_items ? (n_items - 1 - pair) / n_pairs + 1 : 0;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&aready[s], 1);
            mbar_init(&afree[s], 1);
        }
        for (int s = 0; s < kBStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < kDBufs; ++s) {
            mbar_init(&dfull[s], 1);
            mbar_init(&dfree[s], 2 * kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_addr(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA signal
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    if (warp < 4) {  // block scale factors: TMEM columns 448..511 of every lane = ue8m0 1.0
        const uint32_t sf = tmem + ((uint32_t)(warp * 32) << 16) + kSfCol;
#pragma unroll
        for (int c = 0; c < 64; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(sf + c),
                         "r"(0x7F7F7F7Fu));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // scale factors of both CTAs written before the first MMA
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    if (warp == kTmaWarp) {
        // TMA producer (one lane per CTA): this CTA's half of every operand tile
        if (lane == 0) {
            auto loadA = [&](int li) {
                const MatchWork w = work[pair + li * n_pairs];
                const int buf = li & 1;
                if (li >= 2) mbar_wait(&afree[buf], ((li - 2) >> 1) & 1);
                if (rank == 0) mbar_expect_tx(&aready[buf], (uint32_t)(2 * kABytes));
                const uint32_t bar = mapa_rank(smem_addr(&aready[buf]), 0);
                const CUtensorMap* m = w.dir ? &tq1 : &tq0;
#pragma unroll
                for (int a = 0; a < kAtoms; ++a)
                    tma_load_2d_pair(sA + buf * kABytes + a * kAtomBytes, m, 128 * a, w.a0 + (int)rank * kMT, bar);
            };
            if (n_local > 0) loadA(0);
            if (n_local > 1) loadA(1);
            int st = 0, round = 0;
            for (int li = 0; li < n_local; ++li) {
                const MatchWork w = work[pair + li * n_pairs];
                const CUtensorMap* m = w.dir ? &tt1 : &tt0;
                const int n_nt = (w.nb + kNT - 1) / kNT;
                const int a_next_at = n_nt < 3 ? n_nt - 1 : 2;  // the next query tile after this train tile
                for (int nt = 0; nt < n_nt; ++nt) {
#pragma unroll
                    for (int a = 0; a < kAtoms; ++a) {
                        if (round > 0) mbar_wait(&empty[st], (round - 1) & 1);
                        if (rank == 0) mbar_expect_tx(&full[st], (uint32_t)(2 * kBAtomBytes));
                        tma_load_2d_pair(sB + st * kBAtomBytes, m, 128 * a, w.b0 + nt * kNT + (int)rank * (kNT / 2),
                                         mapa_rank(smem_addr(&full[st]), 0));
                        if (++st == kBStages) {
                            st = 0;
                            ++round;
                        }
                    }
                    if (nt == a_next_at && li >= 1 && li + 1 < n_local) loadA(li + 1);
                }
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp) {
        // MMA issuer: one lane of the leader
        if (rank == 0 && lane == 0) {
            // block-scaled instruction descriptor: A, B e2m1 (MXF4 format 1), K-major, N, scale
            // format ue8m0 (bit 23), M = 256, scale-factor ids 0, dense K = 64
            const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(kNT >> 3) << 17) | (1u << 23) |
                                   ((uint32_t)((2 * kMT) >> 4) << 24);
            const uint32_t sfa = tmem + kSfCol, sfb = tmem + kSfCol + 32u;
            int st = 0, round = 0, d = 0, dround = 0;
            for (int li = 0; li < n_local; ++li) {
                const MatchWork w = work[pair + li * n_pairs];
                const int n_nt = (w.nb + kNT - 1) / kNT;
                const int buf = li & 1;
                mbar_wait(&aready[buf], (li >> 1) & 1);
                // smem addresses < 256 KB: the 14-bit address field absorbs the constant offsets
                const uint64_t dA = desc_sw128(smem_addr(sA + buf * kABytes));
                for (int nt = 0; nt < n_nt; ++nt) {
                    if (dround > 0) mbar_wait_cluster(&dfree[d], (dround - 1) & 1);
                    const uint32_t dt = tmem + (uint32_t)(d * kNT);
#pragma unroll
                    for (int a = 0; a < kAtoms; ++a) {
                        mbar_wait(&full[st], round & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint64_t dB = desc_sw128(smem_addr(sB + st * kBAtomBytes));
#pragma unroll
                        for (int k32 = 0; k32 < 4; ++k32) {
                            const int ks = 4 * a + k32;
                            if (ks < NK)
                                mma_f4_pair(dt, dA + (uint64_t)((a * kAtomBytes + k32 * 32) >> 4),
                                            dB + (uint64_t)((k32 * 32) >> 4), idesc, ks > 0 ? 1u : 0u, sfa, sfb);
                        }
                        mma_commit_pair(&empty[st]);
                        if (++st == kBStages) {
                            st = 0;
                            ++round;
                        }
                    }
                    mma_commit_pair(&dfull[d]);
                    if (++d == kDBufs) {
                        d = 0;
                        ++dround;
                    }
                }
                mma_commit_pair(&afree[buf]);
            }
        }
        __syncwarp();
    } else {
        // epilogue: 8 warps per CTA; warp w reads TMEM lane quarter w % 4 (its 32 query rows),
        // columns [112 (w / 4), +112) of each tile (f32 accumulators holding exact integers
        // |S| <= 512), keeping a running (max S, first index) per row; the two column halves
        // merge through shared memory at the end of each item.  Train columns arrive in
        // increasing order within a half, so a strict '>' keeps the lowest index; the merge
        // breaks ties by index.
        const int quarter = warp & 3, half = warp >> 2;
        const int row = (int)rank * kMT + quarter * 32 + lane;  // row of the 256-row query tile
        const uint32_t dfree_leader0 = mapa_rank(smem_addr(&dfree[0]), 0);
        const uint32_t kNegInf = 0xff800000u;
        int d = 0, dround = 0;
        for (int li = 0; li < n_local; ++li) {
            const MatchWork w = work[pair + li * n_pairs];
            const int n_nt = (w.nb + kNT - 1) / kNT;
            float bestk = -INFINITY, bestk_floor = -INFINITY;  // best key; 128 (S_best + 1)
            int bestt = 0;                                      // its tile
            for (int nt = 0; nt < n_nt; ++nt) {
                mbar_wait(&dfull[d], dround & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const int c0 = half * kHalfCols;
                const uint32_t taddr = tmem + (uint32_t)(d * kNT + c0) + ((uint32_t)(quarter * 32) << 16);
                const int jmax = w.nb - nt * kNT - c0;  // valid columns of this half
                // all 112 columns in flight at once, one wait; the accumulator is released to
                // the MMA before the reduction runs
                uint32_t v[kHalfCols];
#pragma unroll
                for (int q = 0; q < 3; ++q) tmem_ld32(taddr + q * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * q));
                tmem_ld16(taddr + 96, v + 96);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                     dfree_leader0 + (uint32_t)(d * sizeof(uint64_t)))
                                 : "memory");
                if (jmax < kHalfCols) {  // ragged last tile: columns >= jmax never win
#pragma unroll
                    for (int c = 0; c < kHalfCols; ++c)
                        if (c >= jmax) v[c] = kNegInf;
                }
                // key = 128 S + (127 - column): exact in f32 (|key| < 2^17), so the maximum key
                // of the tile half is its maximum S at its FIRST column — one FFMA per column
                // with an immediate and a 3-input max tree, no search, no divergence
                float kf[kHalfCols];
#pragma unroll
                for (int c = 0; c < kHalfCols; ++c) kf[c] = fmaf(__uint_as_float(v[c]), 128.0f, (float)(127 - c));
                float m[38];
#pragma unroll
                for (int i = 0; i < 37; ++i) m[i] = fmax3(kf[3 * i], kf[3 * i + 1], kf[3 * i + 2]);
                m[37] = kf[111];
                float m2[13];
#pragma unroll
                for (int i = 0; i < 12; ++i) m2[i] = fmax3(m[3 * i], m[3 * i + 1], m[3 * i + 2]);
                m2[12] = fmaxf(m[36], m[37]);
                const float m3a = fmax3(m2[0], m2[1], m2[2]), m3b = fmax3(m2[3], m2[4], m2[5]);
                const float m3c = fmax3(m2[6], m2[7], m2[8]), m3d = fmax3(m2[9], m2[10], m2[11]);
                const float kmax = fmaxf(fmax3(m3a, m3b, m3c), fmaxf(m3d, m2[12]));
                // a later tile replaces the running best only with a strictly larger S
                // (kmax >= 128 (S_best + 1) <=> S > S_best): earlier tiles win ties
                if (kmax >= bestk_floor) {
                    bestk = kmax;
                    bestt = nt;
                    bestk_floor = 128.0f * (floorf(kmax * (1.0f / 128.0f)) + 1.0f);
                }
                if (++d == kDBufs) {
                    d = 0;
                    ++dround;
                }
            }
            // (S, first index) of this half, then merge the column halves (epilogue warps
            // only: named barrier 1)
            const float sb = floorf(bestk * (1.0f / 128.0f));  // -inf if the half saw no column
            int best = sb > -1e9f ? (int)sb : -0x7fffffff;
            int besti = bestt * kNT + half * kHalfCols + (127 - (int)(bestk - 128.0f * sb));
            if (half == 1) merge[quarter * 32 + lane] = make_int2(best, besti);
            named_sync(1, kEpiWarps * 32);
            if (half == 0) {
                const int2 o = merge[quarter * 32 + lane];
                if (o.x > best || (o.x == best && o.y < besti)) {
                    best = o.x;
                    besti = o.y;
                }
                if (row < w.na) {
                    int32_t* nn = w.dir ? out.nn[1] : out.nn[0];
                    int32_t* dist = w.dir ? out.dist[1] : out.dist[0];
                    nn[w.a0 + row] = besti;
                    if (dist) dist[w.a0 + row] = (K - best) >> 1;
                }
            }
            named_sync(1, kEpiWarps * 32);  // merge slots free for the next item
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // no cross-CTA signal or MMA access after this point
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// offsets table (one small H2D copy): [a_off | b_off | tile prefix of direction 0 | of
// direction 1], n_pairs + 1 entries each
__device__ __forceinline__ int pair_of_row(const int64_t* __restrict__ off, int n_pairs, int64_t i) {
    int lo = 0, hi = n_pairs - 1;  // largest p with off[p] <= i
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void build_work_kernel(const int64_t* __restrict__ tab, int n_pairs, int n_items0, int n_items,
                                  MatchWork* __restrict__ work) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_items) return;
    const int dir = i >= n_items0;
    const int64_t* a_off = tab;
    const int64_t* b_off = tab + (n_pairs + 1);
    const int64_t* tpre = tab + (2 + dir) * (n_pairs + 1);
    const int j = i - dir * n_items0;
    const int p = pair_of_row(tpre, n_pairs, j);
    const int64_t* q_off = dir ? b_off : a_off;
    const int64_t* t_off = dir ? a_off : b_off;
    MatchWork w{};
    w.a0 = (int32_t)(q_off[p] + (int64_t)(j - tpre[p]) * (2 * kMT));
    w.na = (int32_t)min((int64_t)(2 * kMT), q_off[p + 1] - w.a0);
    w.b0 = (int32_t)t_off[p];
    w.nb = (int32_t)(t_off[p + 1] - t_off[p]);
    w.a_pair0 = (int32_t)q_off[p];
    w.dir = dir;
    work[i] = w;
}

__global__ void mutual_kernel(const int32_t* __restrict__ nn_ab, const int32_t* __restrict__ nn_ba,
                              const int64_t* __restrict__ tab, int n_pairs, int64_t n_a, uint8_t* __restrict__ mutual) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_a) return;
    const int p = pair_of_row(tab, n_pairs, i);
    const int64_t local = i - tab[p];
    const int j = nn_ab[i];
    mutual[i] = (uint8_t)(nn_ba[tab[n_pairs + 1 + p] + j] == local);
}

}  // namespace kern

using namespace kern;

// Row-argmax of the +-1 similarity per pair, a against b (direction 0) and, when out.nn[1]
// is set, b against a (direction 1), in one persistent launch over the device work list.
static cudaError_t launch_nn(const uint8_t* a_pm, int64_t n_a, const uint8_t* b_pm, int64_t n_b, int K,
                             const MatchWork* d_work, int n_items, const MatchOut& out, cudaStream_t s) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    // rows of K / 2 bytes (packed e2m1); boxes of 128 bytes of K (a SWIZZLE_128B atom) x 128
    // query rows or 112 train rows (each CTA of a pair loads its half of a tile)
    CUtensorMap mq[2], mt[2];
    const cuuint32_t estr[2] = {1, 1};
    auto encode = [&](CUtensorMap* m, const uint8_t* p, int64_t rows, int box_rows) {
        const cuuint64_t dims[2] = {(cuuint64_t)(K / 2), (cuuint64_t)rows}, strides[1] = {(cuuint64_t)(K / 2)};
        const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(p), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (!encode(&mq[0], a_pm, n_a, kMT) || !encode(&mt[0], b_pm, n_b, kNT / 2) || !encode(&mq[1], b_pm, n_b, kMT) ||
        !encode(&mt[1], a_pm, n_a, kNT / 2))
        return cudaErrorInvalidValue;
    const int grid = 2 * std::min(n_items, num_sms() / 2);  // CTA pairs
    auto go = [&](auto nk) -> cudaError_t {
        constexpr int NK = decltype(nk)::value;
        constexpr int smem = 1024 + 2 * ((NK + 3) / 4) * kAtomBytes + kBStages * kBAtomBytes;
        cudaError_t e2 = ensure_smem_attr((const void*)match_kernel<NK>, smem);
        if (e2 != cudaSuccess) return e2;
        match_kernel<NK><<<(unsigned)grid, kMThreads, smem, s>>>(mq[0], mt[0], mq[1], mt[1], d_work, n_items, K, out);
        return cudaGetLastError();
    };
    switch ((K + 63) >> 6) {  // K = 64-value MMA steps
#define BD_MATCH_K(n) \
    case n: return go(std::integral_constant<int, n>{});
        BD_MATCH_K(1) BD_MATCH_K(2) BD_MATCH_K(3) BD_MATCH_K(4) BD_MATCH_K(5) BD_MATCH_K(6) BD_MATCH_K(7)
        BD_MATCH_K(8)
#undef BD_MATCH_K
        default: return cudaErrorInvalidValue;
    }
}

namespace {
struct MatchWs {  // workspace carve-up (all offsets 256-byte aligned)
    size_t a_pm, b_pm, work, tab, total;
};
size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }
MatchWs match_ws(int64_t n_a, int64_t n_b, int K, int n_pairs) {
    MatchWs w;
    const int64_t max_items = (n_a + n_b) / (2 * kMT) + 2 * (int64_t)n_pairs;
    w.a_pm = 0;
    w.b_pm = up256(w.a_pm + (size_t)n_a * (K / 2));   // packed e2m1 rows
    w.work = up256(w.b_pm + (size_t)n_b * (K / 2));  // both directions' work items
    w.tab = up256(w.work + (size_t)max_items * sizeof(MatchWork));
    w.total = up256(w.tab + (size_t)4 * (n_pairs + 1) * 8);
    return w;
}
}  // namespace

// The one host->device copy (the offsets table, 32 (n_pairs + 1) bytes) comes from a pageable
// std::vector: cudaMemcpyAsync stages pageable sources before returning, so the vector may go
// out of scope (no host synchronisation).  The work list and the row -> pair map are built on
// the device from it.
cudaError_t launch_match(const uint32_t* a, const uint32_t* b, const int64_t* a_off, const int64_t* b_off,
                         int n_pairs, int K, int32_t* nn_ab, int32_t* dist_ab, int32_t* nn_ba, int32_t* dist_ba,
                         uint8_t* mutual, void* ws, cudaStream_t s) {
    const int64_t n_a = a_off[n_pairs], n_b = b_off[n_pairs];
    const int words = K >> 5;
    const MatchWs L = match_ws(n_a, n_b, K, n_pairs);
    uint8_t* W = reinterpret_cast<uint8_t*>(ws);
    uint8_t* a_pm = W + L.a_pm;
    uint8_t* b_pm = W + L.b_pm;
    MatchWork* d_work = reinterpret_cast<MatchWork*>(W + L.work);
    int64_t* d_tab = reinterpret_cast<int64_t*>(W + L.tab);
    const int P1 = n_pairs + 1;
    std::vector<int64_t> tab(4 * (size_t)P1);
    for (int p = 0; p <= n_pairs; ++p) {
        tab[p] = a_off[p];
        tab[P1 + p] = b_off[p];
    }
    tab[2 * P1] = tab[3 * P1] = 0;
    for (int p = 0; p < n_pairs; ++p) {  // query tiles (256 rows) per pair, per direction
        tab[2 * P1 + p + 1] = tab[2 * P1 + p] + (a_off[p + 1] - a_off[p] + 2 * kMT - 1) / (2 * kMT);
        tab[3 * P1 + p + 1] = tab[3 * P1 + p] + (b_off[p + 1] - b_off[p] + 2 * kMT - 1) / (2 * kMT);
    }
    const int n_items0 = (int)tab[3 * P1 - 1], n_items = n_items0 + (nn_ba ? (int)tab[4 * P1 - 1] : 0);
    ProfScope ps("match", s);
    cudaError_t e = cudaMemcpyAsync(d_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    build_work_kernel<<<(unsigned)((n_items + 127) / 128), 128, 0, s>>>(d_tab, n_pairs, n_items0, n_items, d_work);
    expand_pm1_kernel<<<(unsigned)((n_a * words + 255) / 256), 256, 0, s>>>(a, n_a * words, a_pm);
    expand_pm1_kernel<<<(unsigned)((n_b * words + 255) / 256), 256, 0, s>>>(b, n_b * words, b_pm);
    MatchOut out{{nn_ab, nn_ba}, {dist_ab, nn_ba ? dist_ba : nullptr}};
    e = launch_nn(a_pm, n_a, b_pm, n_b, K, d_work, n_items, out, s);
    if (e != cudaSuccess || !nn_ba || !mutual) return e;
    mutual_kernel<<<(unsigned)((n_a + 255) / 256), 256, 0, s>>>(nn_ab, nn_ba, d_tab, n_pairs, n_a, mutual);
    return cudaGetLastError();
}

size_t match_workspace_bytes(int64_t n_a, int64_t n_b, int K, int n_pairs) {
    return match_ws(n_a, n_b, K, n_pairs).total;
}

}  // namespace bd
