// match.cu — SURVEY §8(f) NEXT-1: brute-force Hamming nearest neighbours and mutual NN over
// binary descriptor sets (P:559-560 / P:566-570 "BFMatcher with Mutual Nearest Neighbors";
// S:514-540 tie rule: lowest index).
//
// The paper's similarity S(x, y) = h(x)^T h(y) with h in {-1, +1}^K equals
// K - 2 Hamming(x, y) exactly, so the all-pairs similarity of a query block A (n_a x K) and a
// train block B (n_b x K) is the dense contraction S = A_pm B_pm^T — an exact int8 GEMM with
// int32 accumulators on the tensor cores (tcgen05 kind::i8).  The nearest neighbour of row i
// is the argmax of S[i, :] (first maximum = lowest index on ties); dist = (K - S)/2.
// Design:
//  * expand: bits -> +-1 int8 rows (bit 1 -> +1, bit 0 -> -1; any consistent sign works), one
//    thread per 32-bit word, two 16-byte stores;
//  * match: one CTA per (pair, 128-row query tile); the query tile (128 x K int8, K/128
//    SWIZZLE_128B atoms) is TMA-loaded once; the pair's train rows stream through a 2-stage
//    TMA ring of 128-row tiles filled by warp 5 (one lane) one tile ahead of the MMAs (a
//    producer that waited for its own load before issuing MMAs kept the tensor pipe idle
//    during every load); warp 4 (one lane) issues K/32 tcgen05.mma (M = N = 128,
//    K = 32) per tile into a double-buffered TMEM accumulator; warps 0-3 read their 32 rows x
//    128 columns with tcgen05.ld and keep a running (max S, first index) per row — train
//    columns arrive in increasing order, so a strict '>' keeps the lowest index;
//  * mutual: nn_ba[nn_ab[i]] == i.
#include <algorithm>
#include <type_traits>
#include <vector>

#include "internal.cuh"
#include "tc.cuh"

namespace bd {
namespace kern {

constexpr int kMT = 128;                  // rows per tile (M and N)
constexpr int kMThreads = 6 * 32;         // 4 epilogue warps + MMA warp + TMA producer warp
constexpr int kNT = 256;                  // train rows per tile (MMA N)
constexpr int kAtomBytes = kMT * 128;     // one SWIZZLE_128B atom of the query tile: 128 rows x 128 bytes of K
constexpr int kBAtomBytes = kNT * 128;    // one atom of a train tile (32 KB)
constexpr int kBStages = 3;               // train-atom ring (96 KB)
constexpr int kDBufs = 2;                 // TMEM accumulators (2 x 256 columns)

__global__ void expand_pm1_kernel(const uint32_t* __restrict__ bits, int64_t n_words, int8_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_words) return;
    const uint32_t w = __ldg(bits + i);
    uint32_t q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) v |= (((w >> (4 * k + b)) & 1u) ? 0x01u : 0xFFu) << (8 * b);
        q[k] = v;
    }
    uint4* o = reinterpret_cast<uint4*>(out + i * 32);
    o[0] = make_uint4(q[0], q[1], q[2], q[3]);
    o[1] = make_uint4(q[4], q[5], q[6], q[7]);
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

// Persistent: CTA c takes work items c, c + grid, ...; both directions in one launch.
// Shared memory: the query tile double buffered (the next item's tile lands during this
// item's train tiles) and a ring of kBStages 16 KB train ATOMS (128 rows x 128 bytes of K):
// a stage is released after its 4 MMAs, so loads run ~1.5 tiles ahead at K = 512.
// TMEM: kDBufs accumulators of 128 columns, so the epilogue of tile t overlaps the MMAs of
// tiles t+1 and t+2.
// NKS = K / 32 MMAs per tile, a compile-time count: the issue loop adds constant offsets to
// descriptors built once per stage.  Rebuilding both descriptors from addresses per MMA (a
// runtime loop) limited the issuing lane to ~80 cycles per MMA instead of the tensor pipe's 64
// (tools/lab/mma_tile_lab.cu: 1274 vs 1044 cycles per 16-MMA tile).
template <int NKS>
__global__ void __launch_bounds__(kMThreads, 1)
    match_kernel(const __grid_constant__ CUtensorMap tq0, const __grid_constant__ CUtensorMap tt0,
                 const __grid_constant__ CUtensorMap tq1, const __grid_constant__ CUtensorMap tt1,
                 const MatchWork* __restrict__ work, int n_items, MatchOut out) {
    // direction 0: query tiles of a (tq0, 128-row boxes), train tiles of b (tt0, 256-row boxes);
    // direction 1: tq1 over b, tt1 over a
    using namespace tc;
    constexpr int K = NKS * 32;
    constexpr int kAtoms = (NKS + 3) / 4;
    constexpr int kABytes = kAtoms * kAtomBytes;
    extern __shared__ uint8_t smem_raw[];
    debug_poison_smem(smem_raw);
    __shared__ uint64_t aready[2], afree[2], full[kBStages], empty[kBStages], dfull[kDBufs], dfree[kDBufs];
    __shared__ uint32_t tmem_base_s;
    const uint32_t raw = smem_addr(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = base;                // 2 query tiles
    uint8_t* sB = base + 2 * kABytes;  // kBStages train atoms
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_local = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
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
            mbar_init(&dfree[s], 4 * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_addr(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;

    if (warp == 5) {
        // TMA producer (one lane)
        if (lane == 0) {
            auto loadA = [&](int li) {
                const MatchWork w = work[blockIdx.x + li * gridDim.x];
                const int buf = li & 1;
                if (li >= 2) mbar_wait(&afree[buf], ((li - 2) >> 1) & 1);
                mbar_expect_tx(&aready[buf], (uint32_t)kABytes);
                const CUtensorMap* m = w.dir ? &tq1 : &tq0;
#pragma unroll
                for (int a = 0; a < kAtoms; ++a) tma_load_2d(sA + buf * kABytes + a * kAtomBytes, m, 128 * a, w.a0, &aready[buf]);
            };
            if (n_local > 0) loadA(0);
            if (n_local > 1) loadA(1);
            int st = 0, round = 0;
            for (int li = 0; li < n_local; ++li) {
                const MatchWork w = work[blockIdx.x + li * gridDim.x];
                const CUtensorMap* m = w.dir ? &tt1 : &tt0;
                const int n_nt = (w.nb + kNT - 1) / kNT;
                const int a_next_at = n_nt < 3 ? n_nt - 1 : 2;  // the next query tile after this train tile
                for (int nt = 0; nt < n_nt; ++nt) {
#pragma unroll
                    for (int a = 0; a < kAtoms; ++a) {
                        if (round > 0) mbar_wait(&empty[st], (round - 1) & 1);
                        mbar_expect_tx(&full[st], (uint32_t)kBAtomBytes);
                        tma_load_2d(sB + st * kBAtomBytes, m, 128 * a, w.b0 + nt * kNT, &full[st]);
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
    } else if (warp == 4) {
        // MMA issuer (one lane)
        if (lane == 0) {
            const uint32_t idesc = idesc_s8(kMT, kNT);
            int st = 0, round = 0, d = 0, dround = 0;
            for (int li = 0; li < n_local; ++li) {
                const MatchWork w = work[blockIdx.x + li * gridDim.x];
                const int n_nt = (w.nb + kNT - 1) / kNT;
                const int buf = li & 1;
                mbar_wait(&aready[buf], (li >> 1) & 1);
                // smem addresses < 256 KB: the 14-bit address field absorbs the constant offsets
                const uint64_t dA = desc_sw128(smem_addr(sA + buf * kABytes));
                for (int nt = 0; nt < n_nt; ++nt) {
                    if (dround > 0) mbar_wait(&dfree[d], (dround - 1) & 1);
                    const uint32_t dt = tmem + (uint32_t)(d * kNT);
#pragma unroll
                    for (int a = 0; a < kAtoms; ++a) {
                        mbar_wait(&full[st], round & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint64_t dB = desc_sw128(smem_addr(sB + st * kBAtomBytes));
#pragma unroll
                        for (int k32 = 0; k32 < 4; ++k32) {
                            const int ks = 4 * a + k32;
                            if (ks < NKS)
                                mma_s8(dt, dA + (uint64_t)((a * kAtomBytes + k32 * 32) >> 4), dB + (uint64_t)((k32 * 32) >> 4),
                                       idesc, ks > 0 ? 1u : 0u);
                        }
                        mma_commit(&empty[st]);
                        if (++st == kBStages) {
                            st = 0;
                            ++round;
                        }
                    }
                    mma_commit(&dfull[d]);
                    if (++d == kDBufs) {
                        d = 0;
                        ++dround;
                    }
                }
                mma_commit(&afree[buf]);
            }
        }
        __syncwarp();
    } else {
        // epilogue: warps 0-3, thread = query row, running (max S, first index) over train tiles
        const int row = warp * 32 + lane;
        int d = 0, dround = 0;
        for (int li = 0; li < n_local; ++li) {
            const MatchWork w = work[blockIdx.x + li * gridDim.x];
            const int n_nt = (w.nb + kNT - 1) / kNT;
            int best = -0x7fffffff, besti = 0;
            for (int nt = 0; nt < n_nt; ++nt) {
                mbar_wait(&dfull[d], dround & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t taddr = tmem + (uint32_t)(d * kNT) + ((uint32_t)(warp * 32) << 16);
                const int jmax = w.nb - nt * kNT;  // valid columns in this tile
#pragma unroll
                for (int q = 0; q < kNT / 32; ++q) {
                    uint32_t v[32];
                    tmem_ld32(taddr + q * 32, v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    // chunk maximum first (31 IMNMX); the first index of a new maximum is searched
                    // only when it beats the running best — rare after the first few tiles
                    if (q * 32 + 32 > jmax) {  // ragged last tile: columns >= jmax never win
#pragma unroll
                        for (int c = 0; c < 32; ++c)
                            if (q * 32 + c >= jmax) v[c] = 0x80000000u;
                    }
                    int mx = (int)v[0];
#pragma unroll
                    for (int c = 1; c < 32; ++c) mx = max(mx, (int)v[c]);
                    if (mx > best) {
                        int ci = 31;
#pragma unroll
                        for (int c = 31; c >= 0; --c)
                            if ((int)v[c] == mx) ci = c;
                        best = mx;
                        besti = nt * kNT + q * 32 + ci;
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&dfree[d]);
                if (++d == kDBufs) {
                    d = 0;
                    ++dround;
                }
            }
            if (row < w.na) {
                int32_t* nn = w.dir ? out.nn[1] : out.nn[0];
                int32_t* dist = w.dir ? out.dist[1] : out.dist[0];
                nn[w.a0 + row] = besti;
                if (dist) dist[w.a0 + row] = (K - best) >> 1;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 4) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

__global__ void mutual_kernel(const int32_t* __restrict__ nn_ab, const int32_t* __restrict__ nn_ba,
                              const int64_t* __restrict__ pair_a0, const int64_t* __restrict__ pair_b0,
                              const int32_t* __restrict__ pair_of, int64_t n_a, uint8_t* __restrict__ mutual) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_a) return;
    const int p = pair_of[i];
    const int64_t local = i - pair_a0[p];
    const int j = nn_ab[i];
    mutual[i] = (uint8_t)(nn_ba[pair_b0[p] + j] == local);
}

}  // namespace kern

using namespace kern;

// Row-argmax of the +-1 similarity per pair, a against b (direction 0) and, when nn_ba is
// given, b against a (direction 1), in one persistent launch.
static cudaError_t launch_nn(const int8_t* a_pm, int64_t n_a, const int8_t* b_pm, int64_t n_b,
                             const int64_t* a_off, const int64_t* b_off, int n_pairs, int K, MatchWork* d_work,
                             const MatchOut& out, cudaStream_t s) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    // query maps: 128-row boxes; train maps: 256-row boxes; both SWIZZLE_128B, 128 bytes of K
    CUtensorMap mq[2], mt[2];
    const cuuint32_t estr[2] = {1, 1};
    auto encode = [&](CUtensorMap* m, const int8_t* p, int64_t rows, int box_rows) {
        const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)K};
        const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(p), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (!encode(&mq[0], a_pm, n_a, kMT) || !encode(&mt[0], b_pm, n_b, kNT) || !encode(&mq[1], b_pm, n_b, kMT) ||
        !encode(&mt[1], a_pm, n_a, kNT))
        return cudaErrorInvalidValue;
    std::vector<MatchWork> hw;
    for (int dir = 0; dir < (out.nn[1] ? 2 : 1); ++dir) {
        const int64_t* q_off = dir ? b_off : a_off;
        const int64_t* t_off = dir ? a_off : b_off;
        for (int p = 0; p < n_pairs; ++p)
            for (int64_t r = q_off[p]; r < q_off[p + 1]; r += kMT) {
                MatchWork w{};
                w.a0 = (int32_t)r;
                w.na = (int32_t)std::min<int64_t>(kMT, q_off[p + 1] - r);
                w.b0 = (int32_t)t_off[p];
                w.nb = (int32_t)(t_off[p + 1] - t_off[p]);
                w.a_pair0 = (int32_t)q_off[p];
                w.dir = dir;
                hw.push_back(w);
            }
    }
    cudaError_t e = cudaMemcpyAsync(d_work, hw.data(), hw.size() * sizeof(MatchWork), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    const int n_items = (int)hw.size();
    const int grid = std::min(n_items, num_sms());
    auto go = [&](auto nks) -> cudaError_t {
        constexpr int NKS = decltype(nks)::value;
        constexpr int smem = 1024 + 2 * ((NKS + 3) / 4) * kAtomBytes + kBStages * kBAtomBytes;
        cudaError_t e2 = ensure_smem_attr((const void*)match_kernel<NKS>, smem);
        if (e2 != cudaSuccess) return e2;
        match_kernel<NKS><<<(unsigned)grid, kMThreads, smem, s>>>(mq[0], mt[0], mq[1], mt[1], d_work, n_items, out);
        return cudaGetLastError();
    };
    switch (K >> 5) {
#define BD_MATCH_K(n) \
    case n: return go(std::integral_constant<int, n>{});
        BD_MATCH_K(1) BD_MATCH_K(2) BD_MATCH_K(3) BD_MATCH_K(4) BD_MATCH_K(5) BD_MATCH_K(6) BD_MATCH_K(7)
        BD_MATCH_K(8) BD_MATCH_K(9) BD_MATCH_K(10) BD_MATCH_K(11) BD_MATCH_K(12) BD_MATCH_K(13) BD_MATCH_K(14)
        BD_MATCH_K(15) BD_MATCH_K(16)
#undef BD_MATCH_K
        default: return cudaErrorInvalidValue;
    }
}

namespace {
struct MatchWs {  // workspace carve-up (all offsets 256-byte aligned)
    size_t a_pm, b_pm, work, a0, b0, pair_of, total;
};
size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }
MatchWs match_ws(int64_t n_a, int64_t n_b, int K, int n_pairs) {
    MatchWs w;
    const int64_t max_w1 = n_a / kMT + n_pairs, max_w2 = n_b / kMT + n_pairs;
    w.a_pm = 0;
    w.b_pm = up256(w.a_pm + (size_t)n_a * K);
    w.work = up256(w.b_pm + (size_t)n_b * K);  // both directions' work items
    w.a0 = up256(w.work + (size_t)(max_w1 + max_w2) * sizeof(MatchWork));
    w.b0 = up256(w.a0 + (size_t)n_pairs * 8);
    w.pair_of = up256(w.b0 + (size_t)n_pairs * 8);
    w.total = up256(w.pair_of + (size_t)n_a * 4);
    return w;
}
}  // namespace

// Host->device copies below come from pageable std::vectors: cudaMemcpyAsync stages pageable
// sources before returning, so the vectors may go out of scope (no host synchronisation).
cudaError_t launch_match(const uint32_t* a, const uint32_t* b, const int64_t* a_off, const int64_t* b_off,
                         int n_pairs, int K, int32_t* nn_ab, int32_t* dist_ab, int32_t* nn_ba, int32_t* dist_ba,
                         uint8_t* mutual, void* ws, cudaStream_t s) {
    const int64_t n_a = a_off[n_pairs], n_b = b_off[n_pairs];
    const int words = K >> 5;
    const MatchWs L = match_ws(n_a, n_b, K, n_pairs);
    uint8_t* W = reinterpret_cast<uint8_t*>(ws);
    int8_t* a_pm = reinterpret_cast<int8_t*>(W + L.a_pm);
    int8_t* b_pm = reinterpret_cast<int8_t*>(W + L.b_pm);
    ProfScope ps("match", s);
    expand_pm1_kernel<<<(unsigned)((n_a * words + 255) / 256), 256, 0, s>>>(a, n_a * words, a_pm);
    expand_pm1_kernel<<<(unsigned)((n_b * words + 255) / 256), 256, 0, s>>>(b, n_b * words, b_pm);
    MatchOut out{{nn_ab, nn_ba}, {dist_ab, nn_ba ? dist_ba : nullptr}};
    cudaError_t e = launch_nn(a_pm, n_a, b_pm, n_b, a_off, b_off, n_pairs, K, reinterpret_cast<MatchWork*>(W + L.work),
                              out, s);
    if (e != cudaSuccess || !nn_ba || !mutual) return e;
    int64_t* d_a0 = reinterpret_cast<int64_t*>(W + L.a0);
    int64_t* d_b0 = reinterpret_cast<int64_t*>(W + L.b0);
    int32_t* d_pair_of = reinterpret_cast<int32_t*>(W + L.pair_of);
    std::vector<int32_t> pair_of(n_a);
    for (int p = 0; p < n_pairs; ++p)
        for (int64_t i = a_off[p]; i < a_off[p + 1]; ++i) pair_of[i] = p;
    e = cudaMemcpyAsync(d_a0, a_off, n_pairs * 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_b0, b_off, n_pairs * 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_pair_of, pair_of.data(), n_a * 4, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    mutual_kernel<<<(unsigned)((n_a + 255) / 256), 256, 0, s>>>(nn_ab, nn_ba, d_a0, d_b0, d_pair_of, n_a, mutual);
    return cudaGetLastError();
}

size_t match_workspace_bytes(int64_t n_a, int64_t n_b, int K, int n_pairs) {
    return match_ws(n_a, n_b, K, n_pairs).total;
}

}  // namespace bd
