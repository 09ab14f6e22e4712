// bad_patch_lab.cu — standalone variant lab for the BAD patch kernel (not part of the product).
// Builds the same packed-pair integral tile as csrc/bad_patch.cu and times test-phase variants:
//   MODE 0: test records from the kernel-parameter constant bank (uniform LDCU loads)
//   MODE 1: test records staged once per CTA in shared memory (LDS.128 broadcast loads)
//   UNIT  : tests per work unit (32 = a whole output word, 16 = a half word)
// All variants must produce identical bits (checked against variant 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/bpl tools/lab/bad_patch_lab.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

struct __align__(16) PT {
    uint32_t off[8];
    int32_t nthr1, na1, a2, pad;
};
struct Tab {
    PT t[512];
};

constexpr int kWarps = 16, kBuildWarps = 8, kEW = 33;
constexpr int kIIBytesA = ((1025 * kEW * 4) + 127) / 128 * 128;
constexpr int kStgPitch = 2080, kStgHalf = 16 * kStgPitch;
constexpr int kTabBytes = 512 * 48;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_tx(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     su32(b)),
                 "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(d)),
                 "l"(s), "r"(n), "r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void issue_half(const uint8_t* P, int64_t n, int64_t t, int h, uint8_t* stg, uint64_t* b) {
    const int64_t first = t * 64 + 32 * h;
    const int64_t cnt = max((int64_t)0, min((int64_t)32, n - first));
    mbar_tx(b, (uint32_t)(cnt * 1024));
    for (int q = 0; 2 * q < cnt; ++q) bulk(stg + q * kStgPitch, P + (first + 2 * q) * 1024, (2 * q + 1 < cnt) ? 2048u : 1024u, b);
}
__device__ __forceinline__ void unpack4(uint32_t wa, uint32_t wb, uint32_t (&v)[4]) {
    const uint32_t lo = __byte_perm(wa, wb, 0x5410), hi = __byte_perm(wa, wb, 0x7632);
    v[0] = __byte_perm(lo, 0u, 0x4240);
    v[1] = __byte_perm(lo, 0u, 0x4341);
    v[2] = __byte_perm(hi, 0u, 0x4240);
    v[3] = __byte_perm(hi, 0u, 0x4341);
}

template <int MODE, int UNIT>
__global__ void __launch_bounds__(kWarps * 32, 1)
    lab_kernel(const uint8_t* __restrict__ P, int64_t n, uint16_t* __restrict__ out, int K, const __grid_constant__ Tab tab,
               int skip_tests, unsigned long long* prof) {
    unsigned long long c_wait = 0, c_build = 0, c_sync1 = 0, c_test = 0, c_sync2 = 0, t0, t1;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* II = reinterpret_cast<uint32_t*>(smem);
    uint8_t* stg0 = smem + kIIBytesA;
    PT* stab = reinterpret_cast<PT*>(stg0 + 2 * kStgHalf);
    uint64_t* bars = reinterpret_cast<uint64_t*>(stg0 + 2 * kStgHalf + ((MODE == 1 || MODE == 4) ? kTabBytes : 0));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_tiles = (n + 63) / 64;
    const int units = K / UNIT, hw = K >> 4;  // output in u16 half-words
    if (threadIdx.x < kEW) II[1024 * kEW + threadIdx.x] = 0u;
    uint32_t* stab16 = reinterpret_cast<uint32_t*>(stab);            // MODE 4: K x 16 B
    uint32_t* stab16c = stab16 + 4 * 512;                             // MODE 4: K x 8 B
    if (MODE == 1)
        for (int i = threadIdx.x; i < K * 12; i += blockDim.x) reinterpret_cast<uint32_t*>(stab)[i] = reinterpret_cast<const uint32_t*>(&tab)[i];
    if (MODE == 4)
        for (int k = threadIdx.x; k < K; k += blockDim.x) {
            const PT& T = tab.t[k];
            for (int c = 0; c < 4; ++c) stab16[4 * k + c] = (T.off[2 * c] >> 2) | ((T.off[2 * c + 1] >> 2) << 16);
            stab16c[2 * k] = (uint32_t)(T.a2 & 0xffff) | ((uint32_t)T.na1 << 16);
            stab16c[2 * k + 1] = (uint32_t)T.nthr1;
        }
    // MODE 2/3: this warp's records in registers (lane = test within the warp's units)
    uint32_t rec[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    {
        const int upw = (units + kWarps - 1) / kWarps;
        const int ui = lane / UNIT, u = warp * upw + ui;
        if (ui < upw && u < units) {
            const PT& T = tab.t[u * UNIT + (lane % UNIT)];
            if (MODE == 2) {
                for (int c = 0; c < 4; ++c) rec[c] = (T.off[2 * c] >> 2) | ((T.off[2 * c + 1] >> 2) << 16);
                rec[4] = (uint32_t)(T.a2 & 0xffff) | ((uint32_t)T.na1 << 16);
                rec[5] = (uint32_t)T.nthr1;
            } else if (MODE == 3) {
                for (int c = 0; c < 8; ++c) rec[c] = T.off[c];
                rec[8] = (uint32_t)(T.a2 & 0xffff) | ((uint32_t)T.na1 << 16);
                rec[9] = (uint32_t)T.nthr1;
            }
        }
    }
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && (int64_t)blockIdx.x < n_tiles) {
        issue_half(P, n, blockIdx.x, 0, stg0, &bars[0]);
        issue_half(P, n, blockIdx.x, 1, stg0 + kStgHalf, &bars[1]);
    }
    const int h = (warp >> 2) & 1, ql = 4 * (warp & 3) + (lane >> 3), cg = lane & 7;
    uint8_t* stg_h = stg0 + h * kStgHalf;
    const uint8_t* src = stg_h + ql * kStgPitch + cg * 4;
    uint32_t* dst = II + (4 * cg) * kEW + (16 * h + ql);
    uint32_t parity = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, parity ^= 1u) {
        t0 = clock64();
        if (warp < kBuildWarps) {
            mbar_wait(&bars[h], parity);
            t1 = clock64(); c_wait += t1 - t0; t0 = t1;
            uint32_t col[4] = {0u, 0u, 0u, 0u};
#pragma unroll 2
            for (int y0 = 0; y0 < 32; y0 += 4) {
                uint32_t wa[4], wb[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    wa[r] = *reinterpret_cast<const uint32_t*>(src + 32 * (y0 + r));
                    wb[r] = *reinterpret_cast<const uint32_t*>(src + 1024 + 32 * (y0 + r));
                }
                uint32_t c[4][4], s[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    unpack4(wa[r], wb[r], c[r]);
                    c[r][1] += c[r][0];
                    c[r][2] += c[r][1];
                    c[r][3] += c[r][2];
                    s[r] = c[r][3];
                }
#pragma unroll
                for (int d = 1; d < 8; d <<= 1)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const uint32_t u = __shfl_up_sync(0xffffffffu, s[r], d, 8);
                        if (cg >= d) s[r] += u;
                    }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint32_t ex = s[r] - c[r][3];
                    uint32_t* d0 = dst + ((y0 + r) * 32) * kEW;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        col[k] += ex + c[r][k];
                        d0[k * kEW] = col[k];
                    }
                }
            }
            t1 = clock64(); c_build += t1 - t0; t0 = t1;
            asm volatile("bar.sync %0, 128;" ::"r"(1 + h) : "memory");
            if ((warp & 3) == 0 && lane == 0 && t + gridDim.x < n_tiles) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_half(P, n, t + gridDim.x, h, stg_h, &bars[h]);
            }
        }
        __syncthreads();
        t1 = clock64(); c_sync1 += t1 - t0; t0 = t1;
        if (!skip_tests) {
            const uint32_t IIs = (uint32_t)__cvta_generic_to_shared(II + lane);
            const int64_t pA = t * 64 + 2 * lane;
            const int upw = (units + kWarps - 1) / kWarps;
            for (int ui = upw - 1; ui >= 0; --ui) {
                const int u = warp * upw + ui;
                uint32_t wA = 0, wB = 0;
#pragma unroll
                for (int j = UNIT - 1; j >= 0; --j) {
                    uint32_t ad[8];
                    int nthr1, na1, a2;
                    const int tix = (u < units ? u : 0) * UNIT + j;
                    if (MODE == 1) {
                        const uint4* T = reinterpret_cast<const uint4*>(stab + tix);
                        const uint4 q0 = T[0], q1 = T[1], q2 = T[2];
                        ad[0] = IIs + q0.x; ad[1] = IIs + q0.y; ad[2] = IIs + q0.z; ad[3] = IIs + q0.w;
                        ad[4] = IIs + q1.x; ad[5] = IIs + q1.y; ad[6] = IIs + q1.z; ad[7] = IIs + q1.w;
                        nthr1 = (int)q2.x; na1 = (int)q2.y; a2 = (int)q2.z;
                    } else if (MODE == 2 || MODE == 3) {
                        const int src = (ui * UNIT + j) & 31;
                        uint32_t r[10];
                        if (MODE == 2) {
#pragma unroll
                            for (int c = 0; c < 6; ++c) r[c] = __shfl_sync(0xffffffffu, rec[c], src);
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                ad[2 * c] = IIs + ((r[c] & 0xffffu) << 2);
                                ad[2 * c + 1] = IIs + ((r[c] >> 16) << 2);
                            }
                            a2 = (int)(r[4] & 0xffffu); na1 = (int)r[4] >> 16; nthr1 = (int)r[5];
                        } else {
#pragma unroll
                            for (int c = 0; c < 10; ++c) r[c] = __shfl_sync(0xffffffffu, rec[c], src);
#pragma unroll
                            for (int c = 0; c < 8; ++c) ad[c] = IIs + r[c];
                            a2 = (int)(r[8] & 0xffffu); na1 = (int)r[8] >> 16; nthr1 = (int)r[9];
                        }
                    } else {  // MODE 4: smem packed16 records (LDS.128 offsets + LDS.64 consts)
                        const uint4 q0 = reinterpret_cast<const uint4*>(stab16)[tix];
                        const uint2 q1 = reinterpret_cast<const uint2*>(stab16c)[tix];
                        const uint32_t r4[4] = {q0.x, q0.y, q0.z, q0.w};
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            ad[2 * c] = IIs + ((r4[c] & 0xffffu) << 2);
                            ad[2 * c + 1] = IIs + ((r4[c] >> 16) << 2);
                        }
                        a2 = (int)(q1.x & 0xffffu); na1 = (int)q1.x >> 16; nthr1 = (int)q1.y;
                    }
                    uint32_t cv[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cv[c]) : "r"(ad[c]));
                    const uint32_t S1 = cv[0] - cv[1] - cv[2] + cv[3];
                    const uint32_t S2 = cv[4] - cv[5] - cv[6] + cv[7];
                    const int eA = (int)(S1 & 0xffffu) * a2 + ((int)(S2 & 0xffffu) * na1 + nthr1);
                    const int eB = (int)(S1 >> 16) * a2 + ((int)(S2 >> 16) * na1 + nthr1);
                    wA = __funnelshift_l((uint32_t)eA, wA, 1);
                    wB = __funnelshift_l((uint32_t)eB, wB, 1);
                }
                if (u < units) {
                    if (UNIT == 32) {
                        if (pA < n) reinterpret_cast<uint32_t*>(out)[(pA * hw) / 2 + u] = wA;
                        if (pA + 1 < n) reinterpret_cast<uint32_t*>(out)[((pA + 1) * hw) / 2 + u] = wB;
                    } else {
                        if (pA < n) out[pA * hw + u] = (uint16_t)wA;
                        if (pA + 1 < n) out[(pA + 1) * hw + u] = (uint16_t)wB;
                    }
                }
            }
        }
        t1 = clock64(); c_test += t1 - t0; t0 = t1;
        __syncthreads();
        t1 = clock64(); c_sync2 += t1 - t0; t0 = t1;
    }
    if (lane == 0) {
        const int r = warp < kBuildWarps ? 0 : 5;
        atomicAdd(prof + r + 0, c_wait); atomicAdd(prof + r + 1, c_build); atomicAdd(prof + r + 2, c_sync1);
        atomicAdd(prof + r + 3, c_test); atomicAdd(prof + r + 4, c_sync2);
    }
}

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

static unsigned long long* g_prof;
template <int MODE, int UNIT>
float run(const uint8_t* dP, int64_t n, uint16_t* dout, int K, const Tab& tab, int skip, int reps) {
    auto k = lab_kernel<MODE, UNIT>;
    const int smem = kIIBytesA + 2 * kStgHalf + ((MODE == 1 || MODE == 4) ? kTabBytes : 0) + 64;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int64_t tiles = (n + 63) / 64;
    const int grid = (int)(tiles < sms ? tiles : sms);
    for (int i = 0; i < 2; ++i) k<<<grid, kWarps * 32, smem>>>(dP, n, dout, K, tab, skip, g_prof);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    CK(cudaMemset(g_prof, 0, 80));
    for (int i = 0; i < reps; ++i) k<<<grid, kWarps * 32, smem>>>(dP, n, dout, K, tab, skip, g_prof);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long hp[10];
    CK(cudaMemcpy(hp, g_prof, 80, cudaMemcpyDeviceToHost));
    const double tiles_per_sm = (double)tiles / grid, norm = (double)reps * grid * tiles_per_sm;
    printf("   [MODE %d UNIT %d K %d skip %d] cycles/tile per warp: builders wait %.0f build %.0f sync1 %.0f test %.0f sync2 %.0f | testers sync1 %.0f test %.0f sync2 %.0f\n",
           MODE, UNIT, K, skip, hp[0] / norm / 8, hp[1] / norm / 8, hp[2] / norm / 8, hp[3] / norm / 8, hp[4] / norm / 8,
           hp[7] / norm / 8, hp[8] / norm / 8, hp[9] / norm / 8);
    return ms / reps;
}

int main() {
    const int64_t n = 4000000;
    std::vector<uint8_t> hP(n * 1024);
    uint64_t s = 12345;
    for (auto& v : hP) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        v = (uint8_t)(s >> 56);
    }
    uint8_t* dP;
    CK(cudaMalloc(&dP, n * 1024));
    CK(cudaMemcpy(dP, hP.data(), n * 1024, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&g_prof, 80));
    uint16_t *d0, *d1;
    CK(cudaMalloc(&d0, n * 64));
    CK(cudaMalloc(&d1, n * 64));
    for (int K : {256, 512}) {
        static Tab tab;
        memset(&tab, 0, sizeof tab);
        for (int k = 0; k < K; ++k) {
            int area[2], p[4], r;
            s = s * 6364136223846793005ull + 1442695040888963407ull;
            r = 1 + (int)((s >> 40) % 5);
            for (int j = 0; j < 4; ++j) {
                s = s * 6364136223846793005ull + 1442695040888963407ull;
                p[j] = (int)((s >> 40) % 32) - 16;
            }
            for (int j = 0; j < 2; ++j) {
                const int px = 16 + p[2 * j], py = 16 + p[2 * j + 1];
                const int x0 = px - r < 0 ? 0 : px - r, x1 = (px + r > 31 ? 31 : px + r) + 1;
                const int y0 = py - r < 0 ? 0 : py - r, y1 = (py + r > 31 ? 31 : py + r) + 1;
                area[j] = (x1 - x0) * (y1 - y0);
                auto off = [](int y, int x) -> uint32_t { return (uint32_t)(((y == 0 || x == 0) ? 1024 : (y - 1) * 32 + (x - 1)) * 33 * 4); };
                tab.t[k].off[4 * j + 0] = off(y1, x1);
                tab.t[k].off[4 * j + 1] = off(y0, x1);
                tab.t[k].off[4 * j + 2] = off(y1, x0);
                tab.t[k].off[4 * j + 3] = off(y0, x0);
            }
            tab.t[k].na1 = -area[0];
            tab.t[k].a2 = area[1];
            tab.t[k].nthr1 = -(int)((s >> 50) % 41) * area[0] * area[1] / 2;
        }
        const int reps = 10;
        auto cmp = [&](uint16_t* a, uint16_t* b) {
            std::vector<uint16_t> x(n * K / 16), y(n * K / 16);
            CK(cudaMemcpy(x.data(), a, x.size() * 2, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(y.data(), b, y.size() * 2, cudaMemcpyDeviceToHost));
            return memcmp(x.data(), y.data(), x.size() * 2) == 0;
        };
        float tb = run<1, 32>(dP, n, d0, K, tab, 1, reps);
        float t1 = run<1, 32>(dP, n, d0, K, tab, 0, reps);
        float t1h = run<1, 16>(dP, n, d1, K, tab, 0, reps);
        int s1h = cmp(d0, d1);
        float t2 = run<2, 16>(dP, n, d1, K, tab, 0, reps);
        int s2 = cmp(d0, d1);
        float t3 = run<3, 16>(dP, n, d1, K, tab, 0, reps);
        int s3 = cmp(d0, d1);
        float t4 = run<4, 16>(dP, n, d1, K, tab, 0, reps);
        int s4 = cmp(d0, d1);
        float t4w = run<4, 32>(dP, n, d1, K, tab, 0, reps);
        int s4w = cmp(d0, d1);
        printf("K=%3d build-only %.3f | lds128x3/32 %.3f | lds128x3/16 %.3f (%d) | shfl16/16 %.3f (%d) | shfl32/16 %.3f (%d) | smem16/16 %.3f (%d) | smem16/32 %.3f (%d)\n",
               K, tb, t1, t1h, s1h, t2, s2, t3, s3, t4, s4, t4w, s4w);
    }
    return 0;
}
