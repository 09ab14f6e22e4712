// bad_patch16.cu — §8(a) rows a1, a3, a4 on 32x32 patches for K <= 256 (configs[2]):
// the pipelined variant of bad_patch.cu, in which the integral of one sub-tile is built
// WHILE the tests of the previous sub-tile run.
//
// Why a second kernel: bad_patch.cu keeps one 32-pair integral (135 KB) in shared memory, so
// its build and test phases serialise.  Here a sub-tile is 16 PAIRS (32 patches, packed
// A + 65536*B as in bad_patch.cu) and two integrals (2 x 68 KB) alternate:
//  * layout: entry e(y, x) = 33y + x (y, x in 0..32, row/column 0 are real zero entries),
//    word (e, p) at e*16 + p: bank = 16*(e & 1) + p, and e & 1 = (x + y) & 1 — the entry's
//    COLOUR.  A warp's 32 lanes serve 16 pairs twice: lanes 0-15 one test, lanes 16-31
//    another, so a corner load is conflict-free exactly when the two corners have opposite
//    colours.  An unclamped box's corners (y1,x1), (y0,x1), (y1,x0), (y0,x0) have colours
//    (a, !a, !a, a) (odd side lengths), so two tests whose (box-1, box-2) colour classes are
//    complementary — after optionally swapping a test's two boxes, which only swaps the
//    two area multipliers — load all 8 corners conflict-free.  bad_create pairs the 16 tests
//    of every half-word by an exact minimum-conflict matching (subset DP over 2^16 states).
//  * build (1 warp, lane = (pair p, column half q)): each lane owns 16 columns of one pair for
//    all 32 rows (in-lane row prefix, register column sums, no vertical carry); the q = 1 lane
//    runs ONE ROW BEHIND the q = 0 lane, so the two stores of a pair in every STS instruction
//    have opposite colours (conflict-free), and it receives the q = 0 row total of the
//    previous step by one shuffle (the row-prefix carry);
//  * tests (16 warps, warp w = half-word w of the output: 8 test pairs): per lane the 8 corner
//    byte offsets, the threshold-record address and the bit mask of its test sit in TENSOR
//    MEMORY (tcgen05.ld, one pair ahead), so no record traffic touches the L1 data pipe except
//    one LDS.128 for the thresholds; the two halves' bits meet in one shuffle and leave as
//    16-bit half-words;
//  * staging: 16 bulk copies (TMA engine) per sub-tile into two alternating buffers, issued
//    one per tester warp at the start of the phase that precedes their use.
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace bd {
namespace kern16 {

constexpr int kPairs = 16;                        // pairs per sub-tile (32 patches)
constexpr int kTesters = 16;                      // tester warps (one per output half-word)
constexpr int kBuilders = 4;                      // builder warps (8 rows each)
constexpr int kThreads = (kTesters + kBuilders) * 32;
constexpr int kEntries = 33 * 33;                 // 1089
constexpr int kIIBytes = kEntries * kPairs * 4;   // 69696
constexpr int kStgPitch = 2064;                   // 516 words = 4 mod 32: conflict-free LDS.128
constexpr int kStgBytes = kPairs * kStgPitch;     // 33024
constexpr int kThrBytes = kMaxBits * 2 * 16;      // (test, orientation) threshold records
constexpr int kTmCols = 16;                       // TMEM columns per test pair and lane
constexpr int kVBytes = kBuilders * 32 * 16 * 4;  // per builder lane: 16 column sums of its rows
constexpr int kSmemBytes = 2 * kIIBytes + 2 * kStgBytes + kThrBytes + kVBytes + 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void unpack4(uint32_t wa, uint32_t wb, uint32_t& v0, uint32_t& v1, uint32_t& v2,
                                        uint32_t& v3) {
    const uint32_t lo = __byte_perm(wa, wb, 0x5410);  // [A0 A1 B0 B1]
    const uint32_t hi = __byte_perm(wa, wb, 0x7632);  // [A2 A3 B2 B3]
    v0 = __byte_perm(lo, 0u, 0x4240);                 // A0 + 65536*B0
    v1 = __byte_perm(lo, 0u, 0x4341);
    v2 = __byte_perm(hi, 0u, 0x4240);
    v3 = __byte_perm(hi, 0u, 0x4341);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
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
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    bad_patch16_kernel(const uint8_t* __restrict__ patches, int64_t n, uint16_t* __restrict__ out, int K,
                       const uint8_t* __restrict__ status, const P16Lane* __restrict__ lanes,
                       const int4* __restrict__ thr) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* II0 = reinterpret_cast<uint32_t*>(smem);
    uint8_t* stg0 = smem + 2 * kIIBytes;
    int4* sthr = reinterpret_cast<int4*>(stg0 + 2 * kStgBytes);
    uint4* vbuf = reinterpret_cast<uint4*>(stg0 + 2 * kStgBytes + kThrBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(stg0 + 2 * kStgBytes + kThrBytes + kVBytes);
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int hw_count = K >> 4;  // output half-words per patch = tester warps in use
    const int64_t n_sub = (n + 31) / 32;

    // ---- prologue: zero row/column 0 of both integrals, thresholds, barriers, TMEM ----
    for (int i = tid; i < 2 * 65 * kPairs; i += kThreads) {
        const int b = i / (65 * kPairs), r = i % (65 * kPairs), j = r / kPairs, p = r % kPairs;
        const int e = j < 33 ? j : 33 * (j - 32);  // row 0 (e = 0..32), column 0 (e = 33y)
        II0[b * (kIIBytes / 4) + e * kPairs + p] = 0u;
    }
    for (int i = tid; i < 2 * K; i += kThreads) sthr[i] = thr[i];
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // tester warp w: lane quarter w % 4, columns 128 (w / 4) + 16 i for test pair i
    const uint32_t tq = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
    const bool tester = warp < hw_count;
    if (tester) {
        const int h = lane >> 4;
#pragma unroll 1
        for (int i = 0; i < 8; ++i) {
            const P16Lane& L = lanes[(warp * 8 + i) * 2 + h];
            const uint32_t v[8] = {L.off[0], L.off[1], L.off[2], L.off[3], L.off[4], L.off[5], L.off[6], L.off[7]};
            tmem_st8(tq + kTmCols * i, v);
            tmem_st2(tq + kTmCols * i + 8, L.rec, L.mask);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }

    // sub-tile -> staging buffer (16 bulk copies of one pair each; one per tester warp)
    auto issue = [&](int64_t sub, int b) {
        const int64_t first = sub * 32;
        const int64_t cnt = min((int64_t)32, n - first);
        if (warp == 0 && lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[b])),
                         "r"((uint32_t)(cnt * 1024))
                         : "memory");
        if (warp < kPairs && lane == 0 && 2 * warp < cnt) {
            const uint32_t bytes = (2 * warp + 1 < cnt) ? 2048u : 1024u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(stg0 + b * kStgBytes + warp * kStgPitch)),
                "l"(patches + (first + 2 * warp) * 1024), "r"(bytes), "r"(smem_u32(&bars[b]))
                : "memory");
        }
    };

    // local sub-tiles of this CTA: s_k = blockIdx.x + k * gridDim.x, k = 0 .. n_loc - 1
    const int64_t n_loc = (int64_t)blockIdx.x < n_sub ? (n_sub - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (n_loc > 0) issue(blockIdx.x, 0);
    uint32_t par[2] = {0u, 0u};
    for (int64_t k = 0; k <= n_loc; ++k) {
        // phase k: build sub-tile k into II[k & 1] || test sub-tile k - 1 from II[(k - 1) & 1]
        if (k + 1 < n_loc) issue(blockIdx.x + (k + 1) * gridDim.x, (int)((k + 1) & 1));
        if (warp >= kTesters && k < n_loc) {
            // ------------------------------- build -------------------------------
            // builder bw owns rows 8bw .. 8bw+7; lane = (pair p, column half q)
            const int b = (int)(k & 1), bw = warp - kTesters;
            mbar_wait(&bars[b], par[b]);
            par[b] ^= 1u;
            const int p = lane & 15, q = lane >> 4;
            const uint8_t* src = stg0 + b * kStgBytes + p * kStgPitch + 16 * q;
            uint32_t* II = II0 + b * (kIIBytes / 4) + p;
            // (a) column sums of this builder's 8 rows (bytes summed in 16-bit lanes)
            uint32_t aE[4] = {0u, 0u, 0u, 0u}, aO[4] = {0u, 0u, 0u, 0u}, bE[4] = {0u, 0u, 0u, 0u},
                     bO[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint4 wa = *reinterpret_cast<const uint4*>(src + (8 * bw + r) * 32);
                const uint4 wb = *reinterpret_cast<const uint4*>(src + 1024 + (8 * bw + r) * 32);
                const uint32_t xa[4] = {wa.x, wa.y, wa.z, wa.w}, xb[4] = {wb.x, wb.y, wb.z, wb.w};
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    aE[x] += xa[x] & 0x00ff00ffu;
                    aO[x] += __byte_perm(xa[x], 0u, 0x4341);  // bytes 1, 3 in 16-bit lanes
                    bE[x] += xb[x] & 0x00ff00ffu;
                    bO[x] += __byte_perm(xb[x], 0u, 0x4341);
                }
            }
            {
                uint4* vo = vbuf + bw * 4 * 32 + lane;  // [builder][x][lane]: conflict-free 16-byte rows
#pragma unroll
                for (int x = 0; x < 4; ++x)  // columns 4x .. 4x+3 as packed pairs A + 65536 B
                    vo[x * 32] = make_uint4(__byte_perm(aE[x], bE[x], 0x5410), __byte_perm(aO[x], bO[x], 0x5410),
                                       __byte_perm(aE[x], bE[x], 0x7632), __byte_perm(aO[x], bO[x], 0x7632));
            }
            asm volatile("bar.sync 2, %0;" ::"r"(kBuilders * 32) : "memory");
            // (b) integral at row 8bw for the lane's 16 columns: column sums of the rows above,
            // prefixed over columns (q = 1 adds the q = 0 half's total)
            uint32_t col[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) col[j] = 0u;
            for (int bb = 0; bb < bw; ++bb) {
                const uint4* vi = vbuf + bb * 4 * 32 + lane;
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const uint4 v = vi[x * 32];
                    col[4 * x] += v.x, col[4 * x + 1] += v.y, col[4 * x + 2] += v.z, col[4 * x + 3] += v.w;
                }
            }
#pragma unroll
            for (int j = 1; j < 16; ++j) col[j] += col[j - 1];
            {
                const uint32_t left = __shfl_xor_sync(0xffffffffu, col[15], 16);
                if (q) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) col[j] += left;
                }
            }
            // (c) the 8 rows; the q = 1 lane runs ONE ROW BEHIND (opposite colours per store)
            uint32_t carry_next = 0u;
#pragma unroll 3
            for (int t = 0; t <= 8; ++t) {
                const int rr = t - q;
                const bool act = rr >= 0 && rr < 8;
                const int ry = 8 * bw + rr;
                uint4 wa = make_uint4(0, 0, 0, 0), wb = wa;
                if (act) {
                    wa = *reinterpret_cast<const uint4*>(src + ry * 32);
                    wb = *reinterpret_cast<const uint4*>(src + 1024 + ry * 32);
                }
                uint32_t c[16];
                unpack4(wa.x, wb.x, c[0], c[1], c[2], c[3]);
                unpack4(wa.y, wb.y, c[4], c[5], c[6], c[7]);
                unpack4(wa.z, wb.z, c[8], c[9], c[10], c[11]);
                unpack4(wa.w, wb.w, c[12], c[13], c[14], c[15]);
#pragma unroll
                for (int j = 1; j < 16; ++j) c[j] += c[j - 1];
                // row-prefix carry: q = 1 needs the q = 0 total of ITS row, sent one step ago
                const uint32_t tot = __shfl_xor_sync(0xffffffffu, c[15], 16);
                const uint32_t carry = q ? carry_next : 0u;
                carry_next = tot;
                if (act) {
                    uint32_t* d = II + ((ry + 1) * 33 + 16 * q + 1) * kPairs;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        col[j] += c[j] + carry;
                        d[j * kPairs] = col[j];
                    }
                }
            }
        } else if (tester && k >= 1) {
            // ------------------------------- tests -------------------------------
            const int b = (int)((k - 1) & 1);
            const int64_t base = (blockIdx.x + (k - 1) * gridDim.x) * 32;
            const uint32_t IIl = smem_u32(II0 + b * (kIIBytes / 4) + (lane & 15));
            const uint32_t thr_s = smem_u32(sthr);
            uint32_t wA = 0u, wB = 0u;
            uint32_t ob[2][16];
            tmem_ld16(tq, ob[0]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                tmem_wait16(ob[i & 1]);
                if (i < 7) tmem_ld16(tq + kTmCols * (i + 1), ob[(i + 1) & 1]);
                const uint32_t* r = ob[i & 1];
                uint32_t cv[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cv[c]) : "r"(IIl + r[c]));
                int4 th;
                asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(th.x), "=r"(th.y), "=r"(th.z), "=r"(th.w)
                             : "r"(thr_s + r[8]));
                const uint32_t S1 = cv[0] - cv[1] - cv[2] + cv[3];
                const uint32_t S2 = cv[4] - cv[5] - cv[6] + cv[7];
                // bit = [S1*m1 + S2*m2 + nthr1 < 0] (R4; m1, m2 = A2, -A1, or -A1, A2 when the
                // record's boxes are stored swapped)
                const int eA = (int)(S1 & 0xffffu) * th.y + ((int)(S2 & 0xffffu) * th.z + th.x);
                const int eB = (int)(S1 >> 16) * th.y + ((int)(S2 >> 16) * th.z + th.x);
                wA |= (uint32_t)(eA >> 31) & r[9];
                wB |= (uint32_t)(eB >> 31) & r[9];
            }
            wA |= __shfl_xor_sync(0xffffffffu, wA, 16);
            wB |= __shfl_xor_sync(0xffffffffu, wB, 16);
            if (lane < 16) {
                const int64_t pA = base + 2 * lane;
                if (status) {
                    if (pA < n && status[pA]) wA = 0u;
                    if (pA + 1 < n && status[pA + 1]) wB = 0u;
                }
                if (pA < n) out[pA * hw_count + warp] = (uint16_t)wA;
                if (pA + 1 < n) out[(pA + 1) * hw_count + warp] = (uint16_t)wB;
            }
        }
        __syncthreads();  // phase boundary: integral k done, integral k-1 free, staging k free
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
}

}  // namespace kern16

// ------------------------------------------------------------------------- host --------
// Tables of the 16-pair kernel (bad_create, K <= 256): per half-word (16 tests) an exact
// minimum-conflict pairing, per (pair, half) the lane record, per (test, orientation) the
// threshold record (nthr1, m1, m2).
int patch16_tables(const int8_t* pairs, const uint8_t* radii, const PatchTable& tab, int K,
                   std::vector<P16Lane>& lanes, std::vector<int32_t>& thr) {
    if (K > 256 || K % 32) return -1;
    struct TestGeo {
        uint32_t e[8];  // entries of box 1 (c0..c3) then box 2 (c4..c7)
        int col[8];
    };
    std::vector<TestGeo> g(K);
    thr.assign((size_t)K * 2 * 4, 0);
    for (int k = 0; k < K; ++k) {
        const int r = radii[k];
        for (int j = 0; j < 2; ++j) {
            const int px = 16 + pairs[4 * k + 2 * j], py = 16 + pairs[4 * k + 2 * j + 1];
            const int x0 = std::max(px - r, 0), x1 = std::min(px + r, 31) + 1;
            const int y0 = std::max(py - r, 0), y1 = std::min(py + r, 31) + 1;
            const int ys[4] = {y1, y0, y1, y0}, xs[4] = {x1, x1, x0, x0};  // + - - +
            for (int c = 0; c < 4; ++c) {
                g[k].e[4 * j + c] = (uint32_t)(33 * ys[c] + xs[c]);
                g[k].col[4 * j + c] = (ys[c] + xs[c]) & 1;
            }
        }
        const PatchTest& T = tab.t[k];  // nthr1, na1 = -A1, a2 = A2
        int32_t* n0 = &thr[(size_t)(2 * k) * 4];
        n0[0] = T.nthr1, n0[1] = T.a2, n0[2] = T.na1;  // boxes in order: S1*A2 + S2*(-A1)
        int32_t* n1 = &thr[(size_t)(2 * k + 1) * 4];
        n1[0] = T.nthr1, n1[1] = T.na1, n1[2] = T.a2;  // swapped: S_box2*(-A1) + S_box1*A2
    }
    // conflicts of test a (as stored) against test b in orientation sw
    auto cost = [&](int a, int b, int sw) {
        int c = 0;
        for (int s = 0; s < 8; ++s) c += g[a].col[s] == g[b].col[sw ? (s + 4) & 7 : s];
        return c;
    };
    lanes.assign((size_t)K / 16 * 8 * 2, P16Lane{});
    std::vector<int> dp(1 << 16), choice(1 << 16);
    for (int hw = 0; hw < K / 16; ++hw) {
        const int t0 = 16 * hw;
        // exact min-cost perfect matching over the 16 tests of the half-word: dp[mask] = min
        // conflicts to pair the tests in mask, always pairing the lowest member first
        std::fill(dp.begin(), dp.end(), 1 << 20);
        dp[0] = 0;
        for (int mask = 1; mask < (1 << 16); ++mask) {
            if (__builtin_popcount(mask) & 1) continue;
            const int i = __builtin_ctz(mask);
            const int rest = mask & ~(1 << i);
            for (int j = i + 1; j < 16; ++j) {
                if (!(rest >> j & 1)) continue;
                const int c = std::min(cost(t0 + i, t0 + j, 0), cost(t0 + i, t0 + j, 1));
                const int v = dp[rest & ~(1 << j)] + c;
                if (v < dp[mask]) dp[mask] = v, choice[mask] = j;
            }
        }
        int mask = 0xffff, slot = 0;
        while (mask) {
            const int i = __builtin_ctz(mask), j = choice[mask];
            mask &= ~((1 << i) | (1 << j));
            const int a = t0 + i, b = t0 + j;
            const int sw = cost(a, b, 1) < cost(a, b, 0) ? 1 : 0;
            for (int h = 0; h < 2; ++h) {
                const int t = h ? b : a, s = h ? sw : 0;
                P16Lane& L = lanes[(size_t)(hw * 8 + slot) * 2 + h];
                for (int c = 0; c < 8; ++c) L.off[c] = g[t].e[s ? (c + 4) & 7 : c] * kern16::kPairs * 4u;
                L.rec = (uint32_t)(2 * t + s) * 16u;
                L.mask = 1u << (t - t0);
            }
            ++slot;
        }
    }
    return 0;
}

using namespace kern16;
int patch16_max_bits() { return 256; }

cudaError_t launch_bad_patches16(const uint8_t* patches, int64_t n, const P16Lane* lanes, const int32_t* thr, int K,
                                 uint32_t* out, const uint8_t* status, cudaStream_t s) {
    cudaError_t e = ensure_smem_attr((const void*)bad_patch16_kernel, kSmemBytes);
    if (e != cudaSuccess) return e;
    const int64_t subs = (n + 31) / 32;
    const int grid = (int)std::min<int64_t>(subs, num_sms());
    ProfScope ps("bad_patch", s);
    bad_patch16_kernel<<<grid, kThreads, kSmemBytes, s>>>(patches, n, reinterpret_cast<uint16_t*>(out), K, status,
                                                          lanes, reinterpret_cast<const int4*>(thr));
    return cudaGetLastError();
}

}  // namespace bd
