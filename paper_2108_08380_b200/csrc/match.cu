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
constexpr int kMaxK = 512;
constexpr int kTileBytesMax = kMT * kMaxK;  // 64 KB of int8

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
    int32_t pad[3];
};

// NKS = K / 32 MMAs per tile, a compile-time count: the issue loop then adds constant offsets
// to two descriptors built once per tile.  Rebuilding both descriptors from addresses per MMA
// (a runtime loop) limited the issuing lane to ~80 cycles per MMA instead of the tensor pipe's
// 64 (tools/lab/mma_tile_lab.cu: 1274 vs 1044 cycles per 16-MMA tile).
template <int NKS>
__global__ void __launch_bounds__(kMThreads, 1)
    match_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const MatchWork* __restrict__ work, int32_t* __restrict__ nn, int32_t* __restrict__ dist) {
    constexpr int K = NKS * 32;
    using namespace tc;
    extern __shared__ uint8_t smem_raw[];
    debug_poison_smem(smem_raw);
    __shared__ uint64_t barA, full[2], empty[2], dfull[2], dfree[2];
    __shared__ uint32_t tmem_base_s;
    const uint32_t raw = smem_addr(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int n_atoms = K >> 7;       // 128-byte K atoms (K = 128..512); K < 128 uses 1 atom
    const int atoms = n_atoms > 0 ? n_atoms : 1;
    const int tile_bytes = kMT * 128 * atoms;
    uint8_t* sA = base;
    uint8_t* sB = base + tile_bytes;  // 2 stages
    const MatchWork wk = work[blockIdx.x];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_nt = (wk.nb + kMT - 1) / kMT;
    if (tid == 0) {
        mbar_init(&barA, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&dfull[s], 1);
            mbar_init(&dfree[s], 4 * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            smem_addr(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;

    if (warp == 5) {
        // TMA producer (one lane): the query tile once, then train tiles into the 2-stage ring
        // as soon as a stage is released (one tile ahead of the MMAs)
        if (lane == 0) {
            const int atom_bytes = kMT * 128;
            mbar_expect_tx(&barA, (uint32_t)(atoms * atom_bytes));
            for (int a = 0; a < atoms; ++a) tma_load_2d(sA + a * atom_bytes, &tmA, 128 * a, wk.a0, &barA);
            for (int nt = 0; nt < n_nt; ++nt) {
                const int s = nt & 1;
                if (nt >= 2) mbar_wait(&empty[s], ((nt - 2) >> 1) & 1);
                uint8_t* st = sB + s * tile_bytes;
                mbar_expect_tx(&full[s], (uint32_t)(atoms * atom_bytes));
                for (int a = 0; a < atoms; ++a) tma_load_2d(st + a * atom_bytes, &tmB, 128 * a, wk.b0 + nt * kMT, &full[s]);
            }
        }
        __syncwarp();
    } else if (warp == 4) {
        // MMA issuer (one lane)
        if (lane == 0) {
            const uint32_t idesc = idesc_s8(kMT, kMT);
            const int atom_bytes = kMT * 128;
            mbar_wait(&barA, 0);
            for (int nt = 0; nt < n_nt; ++nt) {
                const int s = nt & 1;
                mbar_wait(&full[s], (nt >> 1) & 1);
                if (nt >= 2) mbar_wait(&dfree[s], ((nt - 2) >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                // smem addresses < 256 KB: the 14-bit address field of the descriptor absorbs the
                // constant offsets without a carry
                const uint64_t dA = desc_sw128(smem_addr(sA)), dB = desc_sw128(smem_addr(sB + s * tile_bytes));
                const uint32_t d = tmem + (uint32_t)(s * kMT);
#pragma unroll
                for (int ks = 0; ks < NKS; ++ks) {
                    const uint64_t off = (uint64_t)(((ks >> 2) * atom_bytes + (ks & 3) * 32) >> 4);
                    mma_s8(d, dA + off, dB + off, idesc, ks > 0 ? 1u : 0u);
                }
                mma_commit(&empty[s]);
                mma_commit(&dfull[s]);
            }
        }
        __syncwarp();
    } else {
        const int row = warp * 32 + lane;
        int best = -0x7fffffff, besti = 0;
        for (int nt = 0; nt < n_nt; ++nt) {
            const int s = nt & 1;
            mbar_wait(&dfull[s], (nt >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t taddr = tmem + (uint32_t)(s * kMT) + ((uint32_t)(warp * 32) << 16);
            const int jmax = wk.nb - nt * kMT;  // valid columns in this tile
#pragma unroll
            for (int q = 0; q < 4; ++q) {
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
                int m = (int)v[0];
#pragma unroll
                for (int c = 1; c < 32; ++c) m = max(m, (int)v[c]);
                if (m > best) {
                    int ci = 31;
#pragma unroll
                    for (int c = 31; c >= 0; --c)
                        if ((int)v[c] == m) ci = c;
                    best = m;
                    besti = nt * kMT + q * 32 + ci;
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&dfree[s]);
        }
        if (row < wk.na) {
            nn[wk.a0 + row] = besti;
            if (dist) dist[wk.a0 + row] = (K - best) >> 1;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 4) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
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

// Row-argmax of the +-1 similarity of a (expanded, n_a x K int8) against b per pair.
static cudaError_t launch_nn(const int8_t* a_pm, int64_t n_a, const int8_t* b_pm, int64_t n_b,
                             const int64_t* a_off, const int64_t* b_off, int n_pairs, int K, MatchWork* d_work,
                             std::vector<MatchWork>& hw, int32_t* nn, int32_t* dist, cudaStream_t s) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap ma, mb;
    const cuuint32_t box[2] = {128, (cuuint32_t)kMT};
    const cuuint32_t estr[2] = {1, 1};
    const cuuint64_t da[2] = {(cuuint64_t)K, (cuuint64_t)n_a}, sa[1] = {(cuuint64_t)K};
    const cuuint64_t db[2] = {(cuuint64_t)K, (cuuint64_t)n_b}, sb[1] = {(cuuint64_t)K};
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(a_pm), da, sa, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(b_pm), db, sb, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    hw.clear();
    for (int p = 0; p < n_pairs; ++p)
        for (int64_t r = a_off[p]; r < a_off[p + 1]; r += kMT) {
            MatchWork w{};
            w.a0 = (int32_t)r;
            w.na = (int32_t)std::min<int64_t>(kMT, a_off[p + 1] - r);
            w.b0 = (int32_t)b_off[p];
            w.nb = (int32_t)(b_off[p + 1] - b_off[p]);
            w.a_pair0 = (int32_t)a_off[p];
            hw.push_back(w);
        }
    cudaError_t e = cudaMemcpyAsync(d_work, hw.data(), hw.size() * sizeof(MatchWork), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    const int smem = 3 * kTileBytesMax + 1024;
    auto go = [&](auto nks) -> cudaError_t {
        constexpr int NKS = decltype(nks)::value;
        cudaError_t e2 = ensure_smem_attr((const void*)match_kernel<NKS>, smem);
        if (e2 != cudaSuccess) return e2;
        match_kernel<NKS><<<(unsigned)hw.size(), kMThreads, smem, s>>>(ma, mb, d_work, nn, dist);
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
    size_t a_pm, b_pm, work1, work2, a0, b0, pair_of, total;
};
size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }
MatchWs match_ws(int64_t n_a, int64_t n_b, int K, int n_pairs) {
    MatchWs w;
    const int64_t max_w1 = n_a / kMT + n_pairs, max_w2 = n_b / kMT + n_pairs;
    w.a_pm = 0;
    w.b_pm = up256(w.a_pm + (size_t)n_a * K);
    w.work1 = up256(w.b_pm + (size_t)n_b * K);
    w.work2 = up256(w.work1 + (size_t)max_w1 * sizeof(MatchWork));
    w.a0 = up256(w.work2 + (size_t)max_w2 * sizeof(MatchWork));
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
    std::vector<MatchWork> hw;
    cudaError_t e = launch_nn(a_pm, n_a, b_pm, n_b, a_off, b_off, n_pairs, K,
                              reinterpret_cast<MatchWork*>(W + L.work1), hw, nn_ab, dist_ab, s);
    if (e != cudaSuccess || !nn_ba) return e;
    e = launch_nn(b_pm, n_b, a_pm, n_a, b_off, a_off, n_pairs, K, reinterpret_cast<MatchWork*>(W + L.work2), hw,
                  nn_ba, dist_ba, s);
    if (e != cudaSuccess || !mutual) return e;
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
