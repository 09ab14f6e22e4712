// bad_patch_tc.cu — §8(a) rows a1, a3, a4 on 32x32 patches (configs[2]; configs[4] BAD-512 on
// the warped patch) with the integral's column prefix on the tensor cores — the default patch
// kernel for every K % 32 == 0 (bad_patch.cu, the CUDA-core build, under BINDESC_PATCH_TC=0).
// DESIGN.md §5.3.
//
//  * Persistent CTAs, 1 per SM: 16 compute warps + 1 producer warp; a tile is 64 patches =
//    32 PAIRS, built in two halves of 32 patches.
//  * Staging: each half's 32 patches arrive by one TMA tensor load (3-D {32, 32, n}, box
//    32 x 32 x 32, SWIZZLE_32B, patches past n zero-filled) into one of two 32 KB slots; the
//    producer refills slot h with the next tile's half as soon as the MMAs reading it commit.
//  * Column prefix C = L * P (L the 32x32 lower-triangular ones matrix) as tcgen05.mma kind::i8
//    (u8 x u8 -> s32): per half, 4 MMAs (M = 128, N = 256, K = 32), MMA q: A = rows 32q..32q+31
//    of blockdiag(L) (K-major, a window into one zero-padded 7 KB buffer), B = patches 8q..8q+7
//    of the half straight from the slot as an MN-major SWIZZLE_32B operand (LBO = 1024 B, SBO =
//    256 B); TMEM lane quarter q then holds the column prefixes of pairs 4q..4q+3 of the half.
//    D is double buffered (2 x 256 TMEM columns, one per half): the next tile's MMAs run under
//    this tile's tests.
//  * Row prefix in registers: compute warp (q, c) = (warp % 4, warp / 4) reads row y = lane of
//    pair 16h + 4q + c with two packed-16-bit tcgen05.ld (32 columns of each patch), packs
//    A + (B << 16), runs the 32-column prefix with 32-bit adds (mod 2^32; box sums < 2^16
//    separate exactly) and stores the row's 32 integral entries.  The integral is the full
//    33 x 33 table II(Y, X), Y, X in 0..32, whose zero row Y = 0 and zero column X = 0 are
//    written once: entry (Y, X, pair) at word 1089 Y + 33 X + pair, so every box is a
//    rectangle in word space, the row stores (lane = row; 1089 = 1 mod 32) hit 32 banks and
//    the test loads (lane = pair) stay conflict-free.
//  * Tests as in bad_patch.cu (lane = pair, 8 corner loads, packed S1/S2, DP2A or integer
//    compare, funnel shift), one unit of U = 16 (K <= 256) or 32 (K <= 512) tests per warp, with
//    8-BYTE broadcast records (one LDS.64 = one shared wavefront, loaded one test ahead; a
//    broadcast LDS.128 costs two): per box the word offset of its corner (Y0, X0) (16 bits) and
//    its width and height (bytes), decoded in 7 ops — PRMT + IMAD for each of (Y0, X0),
//    (Y0, X1), (Y1, X0) and one IADD3 for (Y1, X1).  TMEM holds the two D buffers, not the
//    records.  DP2A thresholds in registers at U = 16.
//  * Output through the unit-major output tile, flushed in coalesced rows at the start of the
//    next tile (bad_patch.cu); on the warped path the tile's status bytes are loaded a tile
//    ahead and invalid keypoints' rows written as zero.
#include "internal.cuh"
#include "tc.cuh"

#include <string.h>

namespace bd {
namespace kern_tc {

using namespace tc;

constexpr int kWarps = 16;                                   // compute warps (+ 1 producer warp)
constexpr int kThreads = (kWarps + 1) * 32;
constexpr int kRowWords = 33 * 33;                           // integral row stride (words), = 1 mod 32
constexpr int kIIBytes = 33 * kRowWords * 4;                 // rows Y = 0..32
constexpr int kIIBytesAligned = (kIIBytes + 1023) / 1024 * 1024;
constexpr int kSlotBytes = 32 * 1024;                        // half a tile
constexpr int kSlots = 2;
constexpr int kZBytes = 28 * 256;                            // blockdiag(L) window buffer
constexpr int kRecBytes = kMaxBits * 8;                      // per table (records, thresholds)
// output tile, unit-major (bad_patch.cu): U = 16 halfword rows of 68, U = 32 word rows of 66
constexpr int kO16Stride = 68;
constexpr int kO32Stride = 66;
constexpr int kOutBytes = kWarps * kO32Stride * 4;
constexpr int kBarBytes = 256;
constexpr int kSmemBytes = 1024 + kIIBytesAligned + kSlots * kSlotBytes + kZBytes + 2 * kRecBytes + kOutBytes + kBarBytes;
// instruction descriptor, kind::i8: D s32, A u8 K-major, B u8 MN-major, N = 256, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 16) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

// The kernel's own test table (built from the PatchTable at launch), copied once per CTA into
// shared memory and read as broadcast records (one LDS.64 per test, plus one LDS.64 of
// thresholds at U = 32).
// (Read from the constant bank with a warp-uniform index instead, LDCU.64 into uniform
// registers folded into the loads' address, the 10 KB working set thrashes the constant cache:
// 2.39 ms vs 1.89 ms, MIO-throttle bound — DESIGN.md §5.3.)
struct TcTable {
    // .x: word offsets 1089 Y0 + 33 X0 of box 1 (low half) and box 2 (high half);
    // .y: bytes X1 - X0, Y1 - Y0 of box 1, then of box 2
    uint2 rec[kMaxBits];
    // .x: nthr1; .y: m1 in the DP2A byte form, else (m1 & 0xffff) | (m2 << 16) (PatchTest)
    int2 thr[kMaxBits];
};

// PRMT-select a 16-bit half or a byte of w (zero-extended), times MUL, plus base: 2 ops
template <uint32_t SEL, uint32_t MUL>
__device__ __forceinline__ uint32_t prmt_mad(uint32_t w, uint32_t base) {
    uint32_t r;
    asm("{\n.reg .b32 t;\nprmt.b32 t, %1, 0, %3;\nmad.lo.u32 %0, t, %4, %2;\n}" : "=r"(r) : "r"(w), "r"(base), "n"(SEL), "n"(MUL));
    return r;
}

// the 4 corner values of box B of record cw, (Y1, X1), (Y0, X1), (Y1, X0), (Y0, X0), for the
// lane's pair (IIl = integral base + 4 lane, opaque to ptxas so nothing is re-associated)
template <int B>
__device__ __forceinline__ void box_corners(uint2 cw, uint32_t IIl, uint32_t IIbase, uint32_t* cv) {
    const uint32_t a3 = prmt_mad<B ? 0x4432u : 0x4410u, 4u>(cw.x, IIl);               // (Y0, X0)
    const uint32_t a1 = prmt_mad<B ? 0x4442u : 0x4440u, 4u * 33u>(cw.y, a3);          // (Y0, X1)
    const uint32_t a2 = prmt_mad<B ? 0x4443u : 0x4441u, 4u * (uint32_t)kRowWords>(cw.y, a3);  // (Y1, X0)
    const uint32_t a0 = a1 + a2 - a3;                                                  // (Y1, X1)
    BD_CHECK(a3 >= IIbase && a0 < IIbase + kIIBytes);
    asm("ld.shared.u32 %0, [%1];" : "=r"(cv[0]) : "r"(a0));
    asm("ld.shared.u32 %0, [%1];" : "=r"(cv[1]) : "r"(a1));
    asm("ld.shared.u32 %0, [%1];" : "=r"(cv[2]) : "r"(a2));
    asm("ld.shared.u32 %0, [%1];" : "=r"(cv[3]) : "r"(a3));
}

// U: tests per warp (unit), 16 for K <= 256, 32 for K <= 512
// ST: a status array is passed (the warped path): rows of invalid keypoints are zeroed
template <int U, bool DP2A, bool ST>
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
    uint2* crec = reinterpret_cast<uint2*>(Z + kZBytes);
    int2* cthr = reinterpret_cast<int2*>(Z + kZBytes + kRecBytes);
    uint32_t* otile = reinterpret_cast<uint32_t*>(Z + kZBytes + 2 * kRecBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(Z + kZBytes + 2 * kRecBytes + kOutBytes);
    uint64_t* full = bars;          // [2] staging slot landed
    uint64_t* dfull = bars + 2;     // [2] D buffer computed
    uint64_t* dempty = bars + 4;    // [2] D buffer read out (16 warps)
    __shared__ uint32_t s_tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = warp == kWarps;
    const int64_t n_tiles = (n + 63) / 64;
    const int words = K >> 5;
    const int units = K / U;  // <= kWarps

    // zero row Y = 0 and zero column X = 0 (never overwritten)
    for (int i = threadIdx.x; i < kRowWords; i += blockDim.x) II[i] = 0u;
    for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) II[(1 + i / 33) * kRowWords + i % 33] = 0u;
    for (int i = threadIdx.x; i < kZBytes; i += blockDim.x) {  // L in row groups 12..15 of the window
        const int g = i >> 8, w = i & 255, kc = w >> 7, r = (w & 127) >> 4, kk = w & 15;
        const int m = (g - 12) * 8 + r, kx = kc * 16 + kk;
        Z[i] = (g >= 12 && g < 16 && kx <= m) ? 1 : 0;
    }
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
        crec[i] = tab.rec[i];
        cthr[i] = tab.thr[i];
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&dfull[i], 1);
            mbar_init(&dempty[i], kWarps);
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
    const uint32_t tmem = s_tmem_base;  // D buffer h at columns 256 h

    if (producer) {
        if (lane == 0) {
            const uint32_t zaddr = smem_addr(Z), saddr = smem_addr(stg);
            const int64_t my_tiles = (int64_t)blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
            const int64_t uses = 2 * my_tiles;  // use u = 2 k + h: half h of the k-th tile, slot h
            auto load = [&](int64_t u) {
                const int sl = (int)(u & 1);
                const int64_t tile = blockIdx.x + (u >> 1) * gridDim.x;
                mbar_expect_tx(&full[sl], (uint32_t)kSlotBytes);
                tma_load_3d(stg + sl * kSlotBytes, &map, 0, 0, (int)(tile * 64 + (u & 1) * 32), &full[sl]);
            };
            for (int64_t u = 0; u < 2 && u < uses; ++u) load(u);
            for (int64_t u = 0; u < uses; ++u) {
                const int h = (int)(u & 1);
                const uint32_t kk = (uint32_t)(u >> 1);
                if (kk > 0) mbar_wait_sleep(&dempty[h], (kk - 1) & 1u);  // buffer h read out (tile k-1)
                mbar_wait_sleep(&full[h], kk & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const uint64_t ad = umma_desc(zaddr + (uint32_t)(12 - 4 * qq) * 256u, 128, 256, 0);
                    const uint64_t bd = umma_desc(saddr + (uint32_t)(h * kSlotBytes + 8 * qq * 1024), 1024, 256, 6);
                    mma_s8(tmem + 256u * (uint32_t)h, ad, bd, kIdesc, qq > 0 ? 1u : 0u);
                }
                mma_commit(&dfull[h]);
                if (u + 2 < uses) {  // slot h is free once these MMAs complete: the next tile's half h
                    mbar_wait_sleep(&dfull[h], kk & 1u);
                    load(u + 2);
                }
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3, c = warp >> 2;
        const int wu = __shfl_sync(0xffffffffu, warp, 0);  // warp-uniform unit index
        int f_p[2], f_j[2], f_lo[2], f_hi[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int idx = threadIdx.x + r * kWarps * 32;
            f_p[r] = idx < 64 * words ? idx / words : 64;
            f_j[r] = idx - (idx / words) * words;
            f_lo[r] = U == 16 ? (2 * f_j[r]) * kO16Stride + f_p[r] : f_j[r] * kO32Stride + f_p[r];
            f_hi[r] = (2 * f_j[r] + 1) * kO16Stride + f_p[r];
        }
        // status bytes of the tile flushed next, loaded one tile ahead (a load at flush time
        // put its latency on the critical path: ~10 % of the stall samples in c4)
        uint8_t stv[2] = {0, 0};
        auto load_status = [&](int64_t tp) {
#pragma unroll
            for (int r = 0; r < 2; ++r)
                stv[r] = (ST && f_p[r] < 64 && tp * 64 + f_p[r] < n) ? status[tp * 64 + f_p[r]] : (uint8_t)0;
        };
        auto flush = [&](int64_t tp) {
            const int64_t p0 = tp * 64;
            const uint16_t* o16 = reinterpret_cast<const uint16_t*>(otile);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (f_p[r] < 64 && p0 + f_p[r] < n) {
                    uint32_t v = U == 16 ? ((uint32_t)o16[f_lo[r]] | ((uint32_t)o16[f_hi[r]] << 16)) : otile[f_lo[r]];
                    if (ST && stv[r]) v = 0u;  // invalid keypoint (warped path): zero row
                    out[(p0 + f_p[r]) * words + f_j[r]] = v;
                }
            }
        };
        const uint32_t IIbase = smem_addr(II);
        // U = 16, DP2A: thresholds of the warp's 16 tests in registers (through an asm load so
        // they are not re-read inside the loop); U = 32: one LDS.64 per test, one test ahead
        constexpr bool kRegThr = DP2A && U == 16;
        int rn[16], rm[16];
        if (kRegThr) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];"
                             : "=r"(rn[j]), "=r"(rm[j])
                             : "r"(smem_addr(cthr + (wu < units ? wu : 0) * 16 + j)));
        }
        int k = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
            if (k > 0) flush(t - gridDim.x);
            if (ST) load_status(t);
            // ------------- integral (a1): row prefixes of the MMA's column prefixes -------------
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                mbar_wait(&dfull[h], (uint32_t)(k & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dg = tmem + 256u * (uint32_t)h + ((uint32_t)(32 * q) << 16) + 64u * (uint32_t)c;
                uint32_t pa[16], pb[16];  // column prefixes of patch A / B, x = 2i, 2i+1 packed
                tmem_ld32p(dg, pa);
                tmem_ld32p(dg + 32, pb);
                tmem_wait16(pa);
                tmem_wait16(pb);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&dempty[h]);
                const int P = 16 * h + 4 * q + c;  // pair of the tile
                const uint32_t adr = IIbase + 4u * (uint32_t)((lane + 1) * kRowWords + 33 + P);  // (Y, X) = (y + 1, 1)
                uint32_t run = 0;
#pragma unroll
                for (int x = 0; x < 32; ++x) {
                    run += __byte_perm(pa[x >> 1], pb[x >> 1], (x & 1) ? 0x7632 : 0x5410);  // A_x + 65536 B_x
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(adr + 4u * 33u * (uint32_t)x), "r"(run) : "memory");
                }
            }
            named_sync(1, kWarps * 32);  // integral complete
            // ------------- tests (a3) and bit packing (a4) -------------
            if (wu < units) {
                // the lane's integral base, opaque to ptxas so each corner decodes in 2 ops
                // (PRMT zero-extend, IMAD onto IIl) instead of being re-associated into 3
                uint32_t IIl;
                asm volatile("mov.u32 %0, %1;" : "=r"(IIl) : "r"(IIbase + 4u * (uint32_t)lane));
                uint32_t wA = 0, wB = 0;
                const uint2* rec = crec + wu * U;
                const int2* thr = cthr + wu * U;
                uint2 nrec = rec[U - 1];
                int2 nthr = kRegThr ? make_int2(0, 0) : thr[U - 1];
#pragma unroll
                for (int j = U - 1; j >= 0; --j) {
                    const uint2 cw = nrec;  // this test's record; the next one's is loaded now
                    const int2 th = nthr;
                    if (j > 0) {
                        nrec = rec[j - 1];
                        if (!kRegThr) nthr = thr[j - 1];
                    }
                    uint32_t cv[8];
                    box_corners<0>(cw, IIl, IIbase, cv);
                    box_corners<1>(cw, IIl, IIbase, cv + 4);
                    const uint32_t S1 = cv[0] - cv[1] - cv[2] + cv[3];
                    const uint32_t S2 = cv[4] - cv[5] - cv[6] + cv[7];
                    int eA, eB;
                    if (DP2A) {
                        const int n1 = kRegThr ? rn[j & 15] : th.x, m1 = kRegThr ? rm[j & 15] : th.y;
                        const int m2 = m1 << 8;  // bytes (0, A2, 0, -A1)
                        eA = dp2a_hi(S2, m1, dp2a_lo(S1, m1, n1));
                        eB = dp2a_hi(S2, m2, dp2a_lo(S1, m2, n1));
                    } else {
                        const int m1 = (int)(int16_t)(th.y & 0xffff), m2 = th.y >> 16;  // -A1, A2
                        eA = (int)(S1 & 0xffffu) * m2 + ((int)(S2 & 0xffffu) * m1 + th.x);
                        eB = (int)(S1 >> 16) * m2 + ((int)(S2 >> 16) * m1 + th.x);
                    }
                    wA = __funnelshift_l((uint32_t)eA, wA, 1);
                    wB = __funnelshift_l((uint32_t)eB, wB, 1);
                }
                if (U == 32)
                    *reinterpret_cast<uint2*>(otile + warp * kO32Stride + 2 * lane) = make_uint2(wA, wB);
                else  // a 16-test unit is half an output word
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
    if (K > kMaxBits || K % 32 != 0 || n > ((int64_t)1 << 30)) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    for (const void* f : {(const void*)bad_patch_tc_kernel<16, true, false>, (const void*)bad_patch_tc_kernel<16, false, false>,
                          (const void*)bad_patch_tc_kernel<32, true, false>, (const void*)bad_patch_tc_kernel<32, false, false>,
                          (const void*)bad_patch_tc_kernel<16, true, true>, (const void*)bad_patch_tc_kernel<16, false, true>,
                          (const void*)bad_patch_tc_kernel<32, true, true>, (const void*)bad_patch_tc_kernel<32, false, true>})
        if (e == cudaSuccess) e = ensure_smem_attr(f, kSmemBytes);
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
    // records from the PatchTable's corner entries (api.cu: corners (Y1,X1), (Y0,X1), (Y1,X0),
    // (Y0,X0) of each box as byte offsets e * 132, e = 32 (Y - 1) + X - 1, or e = 1024 when
    // Y = 0 or X = 0): Y1, X1 >= 1 come from the first corner, Y0 from the second, X0 from the third
    TcTable tt;
    memset(&tt, 0, sizeof(tt));
    for (int k = 0; k < K; ++k) {
        const PatchTest& T = tab.t[k];
        uint32_t base[2], dims[2];
        for (int b = 0; b < 2; ++b) {
            const uint32_t e0 = T.off[4 * b] / 132u, e1 = T.off[4 * b + 1] / 132u, e2 = T.off[4 * b + 2] / 132u;
            if (e0 >= 1024u) return cudaErrorInvalidValue;
            const uint32_t Y1 = e0 / 32u + 1u, X1 = e0 % 32u + 1u;
            const uint32_t Y0 = e1 >= 1024u ? 0u : e1 / 32u + 1u, X0 = e2 >= 1024u ? 0u : e2 % 32u + 1u;
            if (Y0 >= Y1 || X0 >= X1) return cudaErrorInvalidValue;
            base[b] = Y0 * (uint32_t)kRowWords + X0 * 33u;
            dims[b] = (X1 - X0) | ((Y1 - Y0) << 8);
        }
        tt.rec[k] = make_uint2(base[0] | (base[1] << 16), dims[0] | (dims[1] << 16));
        tt.thr[k] = make_int2(T.nthr1, tab.dp2a ? T.m1 : (int)(((uint32_t)T.m1 & 0xffffu) | ((uint32_t)T.m2 << 16)));
    }
    const int64_t tiles = (n + 63) / 64;
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    ProfScope ps("bad_patch", s);
    auto go = [&](auto kern) { kern<<<grid, kThreads, kSmemBytes, s>>>(map, n, out, K, status, tt); };
    const bool st = status != nullptr;
    if (K <= 16 * kWarps) {
        if (tab.dp2a)
            st ? go(bad_patch_tc_kernel<16, true, true>) : go(bad_patch_tc_kernel<16, true, false>);
        else
            st ? go(bad_patch_tc_kernel<16, false, true>) : go(bad_patch_tc_kernel<16, false, false>);
    } else {
        if (tab.dp2a)
            st ? go(bad_patch_tc_kernel<32, true, true>) : go(bad_patch_tc_kernel<32, true, false>);
        else
            st ? go(bad_patch_tc_kernel<32, false, true>) : go(bad_patch_tc_kernel<32, false, false>);
    }
    return cudaGetLastError();
}

}  // namespace bd
