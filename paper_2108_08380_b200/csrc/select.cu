// select.cu — SURVEY §8(f) NEXT-4: one iteration of the BAD feature-selection hot loop
// (Algorithm 1 lines 4-12) with Algorithm 2's integer-sort threshold search
// ("integer sorting, that is O(P+m) ... m = 5110 possible values for theta").
// Readings R29-R31: integer Eq. 2 losses, exact rational feature values
// f = num/den, buckets b = floor((f + 255) * 10) computed exactly, events at the distinct
// member values of each triplet with exact jumps; L* and b* per candidate.
//
// Design:
//  * patch_integral_em: one thread per patch builds its 33x33 integral image in registers and
//    stores it ENTRY-MAJOR as uint16 (box sums < 2^16 for r <= 7, mod-2^16 arithmetic is
//    exact), so the 32 lanes of a warp that read entry e of 32 consecutive patches issue one
//    coalesced 64-byte load;
//  * select_kernel: persistent CTAs (512 threads) loop over candidates; per candidate
//    (a) num = S1*A2 - S2*A1 for every patch (8 coalesced entry loads) into shared memory,
//    (b) every triplet: its three values from smem, L_i(-inf), the exact jumps at its distinct
//        values, bucket by exact double division, integer atomicAdd into a 5111-bin smem
//        histogram (Algorithm 2's counting sort), (c) a block-wide scan of the histogram with
//        the first-minimum rule -> L*, b*.  All arithmetic is integer or exact, so results are
//        independent of thread order.
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace bd {
namespace kern {

constexpr int kSelThreads = 512;
constexpr int kBins = 5111;
constexpr int kMaxSelPatches = 40000;

struct SelCand {
    uint32_t e[8];   // entry indices (y*33 + x) of the 8 corners: S1 = e0 - e1 - e2 + e3, S2 = ...
    int32_t a1, a2;  // clamped areas
    int32_t pad[2];
};

__global__ void patch_integral_em(const uint8_t* __restrict__ patches, int M, uint16_t* __restrict__ II) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    const uint4* src = reinterpret_cast<const uint4*>(patches + (int64_t)m * 1024);
    uint32_t col[32];
#pragma unroll
    for (int x = 0; x < 32; ++x) col[x] = 0;
    for (int x = 0; x <= 32; ++x) II[(int64_t)x * M + m] = 0;  // row 0
    for (int y = 0; y < 32; ++y) {
        const uint4 q0 = __ldg(src + 2 * y), q1 = __ldg(src + 2 * y + 1);
        const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        uint32_t row = 0;
        II[(int64_t)((y + 1) * 33) * M + m] = 0;  // column 0
#pragma unroll
        for (int x = 0; x < 32; ++x) {
            row += (w[x >> 2] >> (8 * (x & 3))) & 0xffu;
            col[x] += row;
            II[(int64_t)((y + 1) * 33 + x + 1) * M + m] = (uint16_t)col[x];
        }
    }
}

__device__ __forceinline__ long long trip_loss(int tau, int sap, int san, int ha, int hp, int hn) {
    const int v = tau - sap - ha * hp + san + ha * hn;
    return v > 0 ? v : 0;
}

__global__ void __launch_bounds__(kSelThreads, 1)
    select_kernel(const uint16_t* __restrict__ II, int M, const int32_t* __restrict__ trip, int N,
                  const int32_t* __restrict__ sap, const int32_t* __restrict__ san, int tau,
                  const SelCand* __restrict__ cand, int J, long long* __restrict__ out_loss,
                  int32_t* __restrict__ out_bucket) {
    extern __shared__ __align__(16) uint8_t smem[];
    debug_poison_smem(smem);
    int32_t* num = reinterpret_cast<int32_t*>(smem);              // M
    int32_t* hist = num + ((M + 3) & ~3);                         // kBins (+ pad)
    __shared__ long long s_red[kSelThreads / 32];
    __shared__ int s_min[kSelThreads / 32], s_arg[kSelThreads / 32];
    __shared__ int s_carry[kSelThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int j = blockIdx.x; j < J; j += gridDim.x) {
        const SelCand c = cand[j];
        const long long den = (long long)c.a1 * c.a2;
        const double dden = (double)den;
        // (a) feature numerators of every patch
        for (int m = tid; m < M; m += kSelThreads) {
            uint32_t v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldg(II + (int64_t)c.e[k] * M + m);
            const int S1 = (int)((v[0] - v[1] - v[2] + v[3]) & 0xffffu);
            const int S2 = (int)((v[4] - v[5] - v[6] + v[7]) & 0xffffu);
            num[m] = S1 * c.a2 - S2 * c.a1;
        }
        for (int b = tid; b < kBins; b += kSelThreads) hist[b] = 0;
        __syncthreads();
        // (b) events of every triplet (R31) into the bucket histogram (Algorithm 2 counting sort)
        long long L0 = 0;
        for (int i = tid; i < N; i += kSelThreads) {
            const int ia = __ldg(trip + 3 * i), ip = __ldg(trip + 3 * i + 1), in = __ldg(trip + 3 * i + 2);
            const int s_ap = __ldg(sap + i), s_an = __ldg(san + i);
            const int v[3] = {num[ia], num[ip], num[in]};
            L0 += trip_loss(tau, s_ap, s_an, -1, -1, -1);
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                bool first = true;
#pragma unroll
                for (int q = 0; q < m; ++q) first = first && (v[q] != v[m]);
                if (!first) continue;
                int hb[3], ha[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    hb[q] = v[q] < v[m] ? 1 : -1;
                    ha[q] = v[q] <= v[m] ? 1 : -1;
                }
                const int d = (int)(trip_loss(tau, s_ap, s_an, ha[0], ha[1], ha[2]) -
                                    trip_loss(tau, s_ap, s_an, hb[0], hb[1], hb[2]));
                if (d != 0) {
                    // b = floor((10 num + 2550 den) / den): exact (operands < 2^53, quotient
                    // never within rounding of an integer from below, |gap| >= 1/den)
                    const double q = (double)(10LL * v[m] + 2550LL * den);
                    const int b = (int)floor(q / dden);
                    BD_CHECK(b >= 0 && b < kBins);
                    atomicAdd(&hist[b], d);
                }
            }
        }
        // block-reduce L0
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L0 += __shfl_xor_sync(0xffffffffu, L0, o);
        if (lane == 0) s_red[warp] = L0;
        __syncthreads();
        // (c) prefix over the histogram: thread t owns bins [10t, 10t+10) (512*10 >= 5111)
        int local[10];
        int run = 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            const int b = tid * 10 + k;
            run += b < kBins ? hist[b] : 0;
            local[k] = run;
        }
        // exclusive scan of the thread totals
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t2 = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t2;
        }
        if (lane == 31) s_carry[warp] = incl;
        __syncthreads();
        int wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += s_carry[w];
        const int base = wbase + incl - run;
        int bmin = 0x7fffffff, barg = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            const int b = tid * 10 + k;
            const int pv = base + local[k];
            if (b < kBins && pv < bmin) {
                bmin = pv;
                barg = b;
            }
        }
        // first minimum: smallest value, then smallest bin
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int om = __shfl_xor_sync(0xffffffffu, bmin, o), oa = __shfl_xor_sync(0xffffffffu, barg, o);
            if (om < bmin || (om == bmin && oa < barg)) {
                bmin = om;
                barg = oa;
            }
        }
        if (lane == 0) {
            s_min[warp] = bmin;
            s_arg[warp] = barg;
        }
        __syncthreads();
        if (tid == 0) {
            long long l0 = 0;
            int m = 0x7fffffff, a = 0x7fffffff;
            for (int w = 0; w < kSelThreads / 32; ++w) {
                l0 += s_red[w];
                if (s_min[w] < m || (s_min[w] == m && s_arg[w] < a)) {
                    m = s_min[w];
                    a = s_arg[w];
                }
            }
            // theta = -inf (all bits -1) comes first in sweep order: a bucket wins only if
            // strictly better
            out_loss[j] = m < 0 ? l0 + m : l0;
            out_bucket[j] = m < 0 ? a : -1;
        }
        __syncthreads();  // smem reused by the next candidate
    }
}

}  // namespace kern

using namespace kern;

int select_max_patches() { return kMaxSelPatches; }

cudaError_t launch_select(const uint8_t* patches, int M, const int32_t* trip, int N, const int32_t* sap,
                          const int32_t* san, int tau, const int8_t* cand_pairs, const uint8_t* cand_radii, int J,
                          long long* loss, int32_t* bucket, void* ws, cudaStream_t s) {
    // candidate records (host): the same clamped-box construction as bad_create's patch path
    std::vector<SelCand> hc(J);
    for (int j = 0; j < J; ++j) {
        const int r = cand_radii[j];
        int area[2];
        for (int q = 0; q < 2; ++q) {
            const int px = 16 + cand_pairs[4 * j + 2 * q], py = 16 + cand_pairs[4 * j + 2 * q + 1];
            const int x0 = std::max(px - r, 0), x1 = std::min(px + r, 31) + 1;
            const int y0 = std::max(py - r, 0), y1 = std::min(py + r, 31) + 1;
            area[q] = (x1 - x0) * (y1 - y0);
            hc[j].e[4 * q + 0] = (uint32_t)(y1 * 33 + x1);
            hc[j].e[4 * q + 1] = (uint32_t)(y0 * 33 + x1);
            hc[j].e[4 * q + 2] = (uint32_t)(y1 * 33 + x0);
            hc[j].e[4 * q + 3] = (uint32_t)(y0 * 33 + x0);
        }
        hc[j].a1 = area[0];
        hc[j].a2 = area[1];
    }
    uint16_t* II = reinterpret_cast<uint16_t*>(ws);
    SelCand* dc = reinterpret_cast<SelCand*>(reinterpret_cast<uint8_t*>(ws) + (((size_t)1089 * M * 2 + 255) & ~(size_t)255));
    cudaError_t e = cudaMemcpyAsync(dc, hc.data(), sizeof(SelCand) * J, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    ProfScope ps("select", s);
    patch_integral_em<<<(M + 127) / 128, 128, 0, s>>>(patches, M, II);
    const int smem = (int)(((M + 3) & ~3) * 4 + ((kBins + 3) & ~3) * 4);
    e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int grid = std::min(J, num_sms());
    select_kernel<<<grid, kSelThreads, smem, s>>>(II, M, trip, N, sap, san, tau, dc, J, loss, bucket);
    return cudaGetLastError();
}

size_t select_workspace_bytes(int M, int J) {
    return (((size_t)1089 * M * 2 + 255) & ~(size_t)255) + sizeof(SelCand) * (size_t)J + 256;
}

}  // namespace bd
