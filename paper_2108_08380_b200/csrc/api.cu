// api.cu — the C ABI of include/bindesc.h: host-side validation, model tables, workspace
// and launch sequencing.  Every compute call enqueues on the caller's stream and returns;
// no host synchronisation, no CPU fallback (a missing device is BD_EUNSUPPORTED/BD_ECUDA).
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <set>
#include <tuple>
#include <new>
#include <functional>
#include <vector>

#include "internal.cuh"

struct bad_model {
    int K;
    int flags;
    int device;
    bd::ImgTest* d_tests;   // device, K records (image path)
    bd::PatchTable tab;     // host copy, passed by value to the patch kernel
};

struct hashsift_model {
    int N;
    int flags;
    int device;
    float* d_wt;    // [N][128] = W (K-major rows: the tcgen05 B operand)
    float* d_bias;  // [N]
};

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

int ok() {
    g_err[0] = 0;
    return BD_OK;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(e == cudaErrorMemoryAllocation ? BD_ENOMEM : BD_ECUDA, "%s: %s (%s)", what,
                cudaGetErrorName(e), cudaGetErrorString(e));
}

#define BD_CUDA(call, what)                         \
    do {                                            \
        cudaError_t e_ = (call);                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

int check_device(int device) {
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (cur != device) return fail(BD_EINVAL, "model was created on device %d, current device is %d", device, cur);
    return BD_OK;
}

int check_images(const uint8_t* images, int n_images, int H, int W, int64_t pitch) {
    if (!images) return fail(BD_EINVAL, "images is NULL");
    if (n_images < 1 || n_images > 65535) return fail(BD_EINVAL, "n_images=%d out of [1, 65535]", n_images);
    if (H < 1 || W < 1 || H > 32768 || W > 32768) return fail(BD_EINVAL, "H=%d W=%d out of [1, 32768]", H, W);
    if (pitch < W) return fail(BD_EINVAL, "pitch %lld < W %d", (long long)pitch, W);
    return BD_OK;
}

int check_kps(const bd_keypoint* kps, int64_t n_kp) {
    if (n_kp < 0) return fail(BD_EINVAL, "n_kp < 0");
    if (n_kp > 0 && !kps) return fail(BD_EINVAL, "kps is NULL");
    if (n_kp > 0 && !aligned(kps, 16)) return fail(BD_EINVAL, "kps must be 16-byte aligned");
    return BD_OK;
}

struct Workspace {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~Workspace() {
        if (p) cudaFreeAsync(p, s);
    }
};

int ws_alloc(Workspace& w, size_t bytes, cudaStream_t s) {
    // keep the current device's pool memory between calls (release threshold: never)
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        std::lock_guard<std::mutex> g(mu);
        if (done.insert(dev).second) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        }
    }
    w.s = s;
    BD_CUDA(cudaMallocAsync(&w.p, bytes ? bytes : 16, s), "cudaMallocAsync(workspace)");
    return BD_OK;
}

// Keypoints per internal chunk of the warped path (bounds workspace: 1 KB patch + 512 B
// SIFT + 1 B status per keypoint).
constexpr int64_t kChunkDefault = 1 << 20;
// BINDESC_CHUNK (keypoints, read once) overrides the chunk of the warped path (experiments)
int64_t chunk_keypoints() {
    static const int64_t c = [] {
        const char* e = getenv("BINDESC_CHUNK");
        const long long v = e ? atoll(e) : 0;
        return v >= 1024 ? (int64_t)v : kChunkDefault;
    }();
    return c;
}
constexpr int kMaxPipeDevices = 64;

}  // namespace

namespace bd {
int num_sms() {
    static std::atomic<int> cache[kMaxPipeDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxPipeDevices) dev = 0;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n <= 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

cudaError_t ensure_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::set<std::tuple<int, const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    if (done.count({dev, fn, bytes})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({dev, fn, bytes});
    return e;
}
}  // namespace bd

extern "C" {

const char* bd_last_error(void) { return g_err; }

int bd_version(void) { return 100; }

int bad_num_bits(const bad_model* m) { return m ? m->K : 0; }
int hashsift_num_bits(const hashsift_model* m) { return m ? m->N : 0; }

int bad_create(const int8_t* pairs, const uint8_t* radii, const float* thresholds, int K, bad_model** out) {
    return bad_create_ex(pairs, radii, thresholds, K, 0, out);
}

int bad_create_ex(const int8_t* pairs, const uint8_t* radii, const float* thresholds, int K, int flags,
                  bad_model** out) {
    if (!out) return fail(BD_EINVAL, "out is NULL");
    if (flags & ~BD_BAD_SCALE_RADIUS) return fail(BD_EINVAL, "unknown bad_create flags 0x%x", flags);
    *out = nullptr;
    if (!pairs || !radii || !thresholds) return fail(BD_EINVAL, "pairs/radii/thresholds is NULL");
    if (K < 32 || K > bd::kMaxBits || K % 32) return fail(BD_EINVAL, "K=%d: need 32 <= K <= 512, K %% 32 == 0", K);
    for (int k = 0; k < K; ++k) {
        for (int j = 0; j < 4; ++j)
            if (pairs[4 * k + j] < -16 || pairs[4 * k + j] > 15)
                return fail(BD_EINVAL, "test %d: offset %d outside [-16, 15]", k, pairs[4 * k + j]);
        if (radii[k] > 7) return fail(BD_EINVAL, "test %d: radius %d > 7", k, radii[k]);
        if (!isfinite(thresholds[k])) return fail(BD_EINVAL, "test %d: non-finite threshold", k);
    }
    int dev = 0;
    BD_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    bad_model* m = new (std::nothrow) bad_model();
    if (!m) return fail(BD_ENOMEM, "host allocation");
    m->K = K;
    m->flags = flags;
    m->device = dev;
    auto clampi = [](double v) -> int32_t {
        const double lim = 1073741824.0;  // 2^30 > any |S1*A2 - S2*A1| (< 225*255*225 < 2^24)
        return (int32_t)(v < -lim ? -lim : (v > lim ? lim : v));
    };
    std::vector<bd::ImgTest> it(K);
    memset(&m->tab, 0, sizeof m->tab);
    for (int k = 0; k < K; ++k) {
        const int r = radii[k];
        const double th = (double)thresholds[k];
        it[k].dx1 = pairs[4 * k + 0];
        it[k].dy1 = pairs[4 * k + 1];
        it[k].dx2 = pairs[4 * k + 2];
        it[k].dy2 = pairs[4 * k + 3];
        it[k].r = r;
        it[k].theta = thresholds[k];
        it[k].t_full = clampi(floor(th * (double)((2 * r + 1) * (2 * r + 1))));  // exact (R4)
        // patch path: centre (16,16), boxes clamped to [0,31]^2 (R5, R7); integral corners
        // (y, x) in 0..32; entry (y-1)*32 + (x-1), zero entry 1024 when y == 0 or x == 0.
        bd::PatchTest& T = m->tab.t[k];
        int area[2];
        for (int j = 0; j < 2; ++j) {
            const int px = 16 + pairs[4 * k + 2 * j], py = 16 + pairs[4 * k + 2 * j + 1];
            const int x0 = std::max(px - r, 0), x1 = std::min(px + r, 31) + 1;
            const int y0 = std::max(py - r, 0), y1 = std::min(py + r, 31) + 1;
            area[j] = (x1 - x0) * (y1 - y0);
            auto off = [](int y, int x) -> uint32_t {
                const int e = (y == 0 || x == 0) ? 1024 : (y - 1) * 32 + (x - 1);
                return (uint32_t)e * 33u * 4u;
            };
            T.off[4 * j + 0] = off(y1, x1);  // + II(y1, x1)
            T.off[4 * j + 1] = off(y0, x1);  // - II(y0, x1)
            T.off[4 * j + 2] = off(y1, x0);  // - II(y1, x0)
            T.off[4 * j + 3] = off(y0, x0);  // + II(y0, x0)
        }
        T.m1 = -area[0];  // integer form; converted to the DP2A byte form below if it fits
        T.m2 = area[1];
        T.nthr1 = -(clampi(floor(th * (double)area[0] * (double)area[1])) + 1);
    }
    m->tab.dp2a = 1;
    for (int k = 0; k < K; ++k)
        if (-m->tab.t[k].m1 > 127 || m->tab.t[k].m2 > 127) m->tab.dp2a = 0;
    if (m->tab.dp2a)
        for (int k = 0; k < K; ++k) {
            bd::PatchTest& T = m->tab.t[k];
            const uint32_t a2 = (uint32_t)T.m2 & 0xffu, na1 = (uint32_t)T.m1 & 0xffu;
            T.m1 = (int32_t)(a2 | (na1 << 16));         // bytes (A2, 0, -A1, 0)
            T.m2 = (int32_t)((a2 << 8) | (na1 << 24));  // bytes (0, A2, 0, -A1)
        }
    // box-clustered order for the image path (bd::ImgBox): box j of test k is item 2k + j; a
    // recursive median split of the box centres (alternating dx / dy) orders them so that every
    // run of 32 consecutive boxes is compact in offset space -> one gather instruction of the
    // kernel touches few cache lines whatever the keypoint's rotation and scale
    std::vector<int> order(2 * K);
    for (int i = 0; i < 2 * K; ++i) order[i] = i;
    auto cx = [&](int i) { return (int)pairs[4 * (i >> 1) + 2 * (i & 1)]; };
    auto cy = [&](int i) { return (int)pairs[4 * (i >> 1) + 2 * (i & 1) + 1]; };
    std::function<void(int, int, int)> kd = [&](int lo, int hi, int depth) {
        if (hi - lo <= 32) return;
        const int mid = lo + (hi - lo) / 2;
        std::stable_sort(order.begin() + lo, order.begin() + hi, [&](int a, int b) {
            return depth % 2 == 0 ? (cx(a) < cx(b) || (cx(a) == cx(b) && cy(a) < cy(b)))
                                  : (cy(a) < cy(b) || (cy(a) == cy(b) && cx(a) < cx(b)));
        });
        kd(lo, mid, depth + 1);
        kd(mid, hi, depth + 1);
    };
    kd(0, 2 * K, 0);
    std::vector<bd::ImgBox> boxes(2 * K);
    std::vector<uint32_t> bpos(K, 0u);
    for (int p = 0; p < 2 * K; ++p) {
        const int i = order[p], k = i >> 1, j = i & 1;
        boxes[p] = bd::ImgBox{pairs[4 * k + 2 * j], pairs[4 * k + 2 * j + 1], radii[k], 0};
        bpos[k] |= (uint32_t)p << (16 * j);
    }
    const int kmax = K <= 256 ? 256 : 512, kR = 2 * kmax / 32;
    std::vector<bd::ImgBox> lane_major((size_t)32 * kR, bd::ImgBox{0, 0, 0, 0});
    for (int p = 0; p < 2 * K; ++p) lane_major[(size_t)(p & 31) * kR + (p >> 5)] = boxes[p];
    const size_t tb = sizeof(bd::ImgTest) * K, bb = sizeof(bd::ImgBox) * 2 * K, pb = sizeof(uint32_t) * K,
                 lb = sizeof(bd::ImgBox) * lane_major.size();
    cudaError_t e = cudaMalloc(&m->d_tests, tb + bb + pb + lb);
    if (e == cudaSuccess) e = cudaMemcpy(m->d_tests, it.data(), tb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy((uint8_t*)m->d_tests + tb, boxes.data(), bb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy((uint8_t*)m->d_tests + tb + bb, bpos.data(), pb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy((uint8_t*)m->d_tests + tb + bb + pb, lane_major.data(), lb, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (m->d_tests) cudaFree(m->d_tests);
        delete m;
        return cuda_fail(e, "bad_create upload");
    }
    *out = m;
    return ok();
}

void bad_destroy(bad_model* m) {
    if (!m) return;
    if (m->d_tests) cudaFree(m->d_tests);
    delete m;
}

int bad_compute(const bad_model* m, const uint8_t* images, int n_images, int H, int W, int64_t pitch,
                const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp, uint32_t* out_bits,
                uint8_t* kp_status, void* stream) {
    if (!m) return fail(BD_EINVAL, "model is NULL");
    int rc;
    if ((rc = check_kps(kps, n_kp)) != BD_OK) return rc;
    if (n_kp == 0) return ok();
    if ((rc = check_images(images, n_images, H, W, pitch)) != BD_OK) return rc;
    if (!out_bits || !aligned(out_bits, 4)) return fail(BD_EINVAL, "out_bits NULL or misaligned");
    if ((int64_t)H * W > 16843009LL) return fail(BD_EINVAL, "H*W too large for uint32 integral sums");
    if ((rc = check_device(m->device)) != BD_OK) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    // radii <= 7 (bad_create) keep every box sum below 2^16, so the integral is stored mod 2^16
    // (half the HBM traffic of the integral and of the corner gathers); the scaled radius variant
    // (box radius r * scale) needs the exact uint32 integral
    const int eb = (m->flags & BD_BAD_SCALE_RADIUS) ? 4 : 2;
    if (eb == 2 && n_kp <= bd::bad_image_local_max_kp()) {  // latency path: no image integral, one launch
        BD_CUDA(bd::launch_bad_image_local(images, n_images, H, W, pitch, kps, kp_image, n_kp, m->d_tests, m->K,
                                           out_bits, kp_status, s),
                "bad_image kernel");
        return ok();
    }
    // uint16 + aligned rows: the vectorised 3-kernel integral, column c stored at index c + 7 of a
    // row pitch rounded to 8 entries (16-byte aligned stores); else the two-pass kernels
    const bool vec = eb == 2 && bd::integral16_vec_ok(images, n_images, H, W, pitch);
    const int64_t ip = vec ? ((W + 8 + 7) / 8) * 8 : W + 1;
    Workspace ws;
    const size_t ii_bytes = ((size_t)ip * (H + 1) * n_images * eb + 255) & ~(size_t)255;
    const size_t band_bytes =
        ((vec ? bd::integral16_vec_workspace_bytes(n_images, H, W) : bd::integral_workspace_bytes(n_images, H, W)) +
         255) & ~(size_t)255;
    const size_t order_bytes = bd::bad_image_order_bytes(n_images, H, W, n_kp);
    if ((rc = ws_alloc(ws, ii_bytes + band_bytes + order_bytes, s)) != BD_OK) return rc;
    void* band_ws = band_bytes ? (uint8_t*)ws.p + ii_bytes : nullptr;
    void* order_ws = order_bytes ? (uint8_t*)ws.p + ii_bytes + band_bytes : nullptr;
    const void* ii = ws.p;  // element (y, c) of the integral at ii[y * ip + c]
    if (vec) {
        BD_CUDA(bd::launch_integral16_vec(images, n_images, H, W, pitch, (uint16_t*)ws.p, ip, s, band_ws),
                "integral kernel");
        ii = (const uint16_t*)ws.p + 7;
    } else if (eb == 2) {
        BD_CUDA(bd::launch_integral16(images, n_images, H, W, pitch, (uint16_t*)ws.p, ip, s, band_ws),
                "integral kernel");
    } else {
        BD_CUDA(bd::launch_integral(images, n_images, H, W, pitch, (uint32_t*)ws.p, ip, s, band_ws),
                "integral kernel");
    }
    BD_CUDA(bd::launch_bad_image(images, n_images, H, W, pitch, ii, eb, ip, kps, kp_image, n_kp, m->d_tests, m->K,
                                 (m->flags & BD_BAD_SCALE_RADIUS) ? 1 : 0, out_bits, kp_status, order_ws, s),
            "bad_image kernel");
    return ok();
}

int bad_compute_patches(const bad_model* m, const uint8_t* patches, int64_t n, uint32_t* out_bits, void* stream) {
    if (!m) return fail(BD_EINVAL, "model is NULL");
    if (n < 0) return fail(BD_EINVAL, "n < 0");
    if (n == 0) return ok();
    if (!patches || !aligned(patches, 16)) return fail(BD_EINVAL, "patches NULL or not 16-byte aligned");
    if (!out_bits || !aligned(out_bits, 4)) return fail(BD_EINVAL, "out_bits NULL or misaligned");
    int rc;
    if ((rc = check_device(m->device)) != BD_OK) return rc;
    BD_CUDA(bd::launch_bad_patches(patches, n, m->tab, m->K, out_bits, nullptr, (cudaStream_t)stream),
            "bad_patch kernel");
    return ok();
}

int hashsift_create(const float* B, int N, hashsift_model** out) { return hashsift_create_ex(B, N, 0, out); }

int hashsift_create_ex(const float* B, int N, int flags, hashsift_model** out) {
    if (!out) return fail(BD_EINVAL, "out is NULL");
    if (flags & ~BD_HS_ROOTSIFT) return fail(BD_EINVAL, "unknown hashsift_create flags 0x%x", flags);
    *out = nullptr;
    if (!B) return fail(BD_EINVAL, "B is NULL");
    if (N < 32 || N > bd::kMaxBits || N % 32) return fail(BD_EINVAL, "N=%d: need 32 <= N <= 512, N %% 32 == 0", N);
    for (int64_t i = 0; i < (int64_t)N * 129; ++i)
        if (!isfinite(B[i])) return fail(BD_EINVAL, "B has a non-finite entry at %lld", (long long)i);
    int dev = 0;
    BD_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    hashsift_model* m = new (std::nothrow) hashsift_model();
    if (!m) return fail(BD_ENOMEM, "host allocation");
    m->N = N;
    m->flags = flags;
    m->device = dev;
    std::vector<float> wt((size_t)128 * N), bias(N);
    for (int k = 0; k < N; ++k) {
        for (int i = 0; i < 128; ++i) wt[(size_t)k * 128 + i] = B[(size_t)k * 129 + i];
        bias[k] = B[(size_t)k * 129 + 128];
    }
    cudaError_t e = cudaMalloc(&m->d_wt, wt.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc(&m->d_bias, bias.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(m->d_wt, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(m->d_bias, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (m->d_wt) cudaFree(m->d_wt);
        if (m->d_bias) cudaFree(m->d_bias);
        delete m;
        return cuda_fail(e, "hashsift_create upload");
    }
    *out = m;
    return ok();
}

void hashsift_destroy(hashsift_model* m) {
    if (!m) return;
    if (m->d_wt) cudaFree(m->d_wt);
    if (m->d_bias) cudaFree(m->d_bias);
    delete m;
}

int hashsift_compute_patches(const hashsift_model* m, const uint8_t* patches, int64_t n, uint32_t* out_bits,
                             float* out_sift, void* stream) {
    if (!m) return fail(BD_EINVAL, "model is NULL");
    if (n < 0) return fail(BD_EINVAL, "n < 0");
    if (n == 0) return ok();
    if (!patches || !aligned(patches, 16)) return fail(BD_EINVAL, "patches NULL or not 16-byte aligned");
    if (!out_bits || !aligned(out_bits, 4)) return fail(BD_EINVAL, "out_bits NULL or misaligned");
    if (out_sift && !aligned(out_sift, 16)) return fail(BD_EINVAL, "out_sift not 16-byte aligned");
    int rc;
    if ((rc = check_device(m->device)) != BD_OK) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    Workspace ws;
    if (!out_sift && (rc = ws_alloc(ws, (size_t)std::min(n, chunk_keypoints()) * 512, s)) != BD_OK) return rc;
    for (int64_t c0 = 0; c0 < n; c0 += (out_sift ? n : chunk_keypoints())) {
        const int64_t cn = out_sift ? n : std::min(chunk_keypoints(), n - c0);
        float* sv = out_sift ? out_sift : (float*)ws.p;
        BD_CUDA(bd::launch_sift(patches + c0 * 1024, cn, sv, m->flags & BD_HS_ROOTSIFT, s), "sift kernel");
        BD_CUDA(bd::launch_project(sv, cn, m->d_wt, m->d_bias, m->N, out_bits + c0 * (m->N / 32), nullptr, s),
                "project kernel");
    }
    return ok();
}

int bd_warp_patches(const uint8_t* images, int n_images, int H, int W, int64_t pitch, const bd_keypoint* kps,
                    const int32_t* kp_image, int64_t n_kp, uint8_t* out_patches, uint8_t* kp_status,
                    void* stream) {
    return bd_warp_patches_ex(images, n_images, H, W, pitch, kps, kp_image, n_kp, BD_WARP_NN, out_patches,
                              kp_status, stream);
}

int bd_warp_patches_ex(const uint8_t* images, int n_images, int H, int W, int64_t pitch, const bd_keypoint* kps,
                       const int32_t* kp_image, int64_t n_kp, int mode, uint8_t* out_patches, uint8_t* kp_status,
                       void* stream) {
    if (mode != BD_WARP_NN && mode != BD_WARP_BILINEAR) return fail(BD_EINVAL, "unknown warp mode %d", mode);
    int rc;
    if ((rc = check_kps(kps, n_kp)) != BD_OK) return rc;
    if (n_kp == 0) return ok();
    if ((rc = check_images(images, n_images, H, W, pitch)) != BD_OK) return rc;
    if (!out_patches || !aligned(out_patches, 16)) return fail(BD_EINVAL, "out_patches NULL or misaligned");
    BD_CUDA(bd::launch_warp_nn(images, n_images, H, W, pitch, mode, kps, kp_image, n_kp, out_patches, kp_status,
                               (cudaStream_t)stream),
            "warp kernel");
    return ok();
}

int bd_describe_warped(const bad_model* bad, const hashsift_model* hs, const uint8_t* images, int n_images, int H,
                       int W, int64_t pitch, const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp,
                       uint32_t* out_bad, uint32_t* out_hs, uint8_t* kp_status, void* stream) {
    return bd_describe_warped_ex(bad, hs, images, n_images, H, W, pitch, kps, kp_image, n_kp, BD_WARP_NN, out_bad,
                                 out_hs, kp_status, stream);
}

int bd_describe_warped_ex(const bad_model* bad, const hashsift_model* hs, const uint8_t* images, int n_images, int H,
                          int W, int64_t pitch, const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp,
                          int mode, uint32_t* out_bad, uint32_t* out_hs, uint8_t* kp_status, void* stream) {
    int rc;
    if (mode != BD_WARP_NN && mode != BD_WARP_BILINEAR) return fail(BD_EINVAL, "unknown warp mode %d", mode);
    if (!bad && !hs) return fail(BD_EINVAL, "both models are NULL");
    if (bad && (!out_bad || !aligned(out_bad, 4))) return fail(BD_EINVAL, "out_bad NULL or misaligned");
    if (hs && (!out_hs || !aligned(out_hs, 4))) return fail(BD_EINVAL, "out_hs NULL or misaligned");
    if ((rc = check_kps(kps, n_kp)) != BD_OK) return rc;
    if (n_kp == 0) return ok();
    if ((rc = check_images(images, n_images, H, W, pitch)) != BD_OK) return rc;
    if (bad && (rc = check_device(bad->device)) != BD_OK) return rc;
    if (hs && (rc = check_device(hs->device)) != BD_OK) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t chunk = std::min(n_kp, chunk_keypoints());
    const size_t patch_bytes = (size_t)chunk * 1024, sift_bytes = hs ? (size_t)chunk * 512 : 0;
    const size_t status_bytes = kp_status ? 0 : (size_t)(chunk + 15) / 16 * 16;
    Workspace ws;
    if ((rc = ws_alloc(ws, patch_bytes + sift_bytes + status_bytes, s)) != BD_OK) return rc;
    uint8_t* patches = (uint8_t*)ws.p;
    float* sv = (float*)(patches + patch_bytes);
    uint8_t* st_ws = patches + patch_bytes + sift_bytes;
    for (int64_t c0 = 0; c0 < n_kp; c0 += chunk) {
        const int64_t cn = std::min(chunk, n_kp - c0);
        uint8_t* st = kp_status ? kp_status + c0 : st_ws;
        BD_CUDA(bd::launch_warp_nn(images, n_images, H, W, pitch, mode, kps + c0, kp_image ? kp_image + c0 : nullptr,
                                   cn, patches, st, s),
                "warp kernel");
        if (bad) {
            uint32_t* ob = out_bad + c0 * (bad->K / 32);
            BD_CUDA(bd::launch_bad_patches(patches, cn, bad->tab, bad->K, ob, st, s), "bad_patch kernel");
        }
        if (hs) {
            uint32_t* oh = out_hs + c0 * (hs->N / 32);
            BD_CUDA(bd::launch_sift(patches, cn, sv, hs->flags & BD_HS_ROOTSIFT, s), "sift kernel");
            BD_CUDA(bd::launch_project(sv, cn, hs->d_wt, hs->d_bias, hs->N, oh, st, s), "project kernel");
        }
    }
    return ok();
}

int hashsift_compute(const hashsift_model* m, const uint8_t* images, int n_images, int H, int W, int64_t pitch,
                     const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp, uint32_t* out_bits,
                     float* out_sift, uint8_t* kp_status, void* stream) {
    if (!m) return fail(BD_EINVAL, "model is NULL");
    if (!out_sift)
        return bd_describe_warped(nullptr, m, images, n_images, H, W, pitch, kps, kp_image, n_kp, nullptr, out_bits,
                                  kp_status, stream);
    int rc;
    if ((rc = check_kps(kps, n_kp)) != BD_OK) return rc;
    if (n_kp == 0) return ok();
    if ((rc = check_images(images, n_images, H, W, pitch)) != BD_OK) return rc;
    if (!out_bits || !aligned(out_bits, 4) || !aligned(out_sift, 16))
        return fail(BD_EINVAL, "out_bits / out_sift NULL or misaligned");
    if ((rc = check_device(m->device)) != BD_OK) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t chunk = std::min(n_kp, chunk_keypoints());
    Workspace ws;
    if ((rc = ws_alloc(ws, (size_t)chunk * 1024 + (kp_status ? 0 : (size_t)chunk + 16), s)) != BD_OK) return rc;
    uint8_t* patches = (uint8_t*)ws.p;
    for (int64_t c0 = 0; c0 < n_kp; c0 += chunk) {
        const int64_t cn = std::min(chunk, n_kp - c0);
        uint8_t* st = kp_status ? kp_status + c0 : patches + (size_t)chunk * 1024;
        BD_CUDA(bd::launch_warp_nn(images, n_images, H, W, pitch, BD_WARP_NN, kps + c0,
                                   kp_image ? kp_image + c0 : nullptr, cn, patches, st, s),
                "warp kernel");
        BD_CUDA(bd::launch_sift(patches, cn, out_sift + c0 * 128, m->flags & BD_HS_ROOTSIFT, s), "sift kernel");
        BD_CUDA(bd::launch_project(out_sift + c0 * 128, cn, m->d_wt, m->d_bias, m->N, out_bits + c0 * (m->N / 32), st,
                                   s),
                "project kernel");
    }
    return ok();
}

int bd_match_hamming(const uint32_t* a, const int64_t* a_off, const uint32_t* b, const int64_t* b_off, int n_pairs,
                     int K, int32_t* nn_ab, int32_t* dist_ab, int32_t* nn_ba, int32_t* dist_ba, uint8_t* mutual,
                     void* stream) {
    if (!a || !b || !a_off || !b_off || !nn_ab) return fail(BD_EINVAL, "a/b/a_off/b_off/nn_ab is NULL");
    if (n_pairs < 1) return fail(BD_EINVAL, "n_pairs=%d < 1", n_pairs);
    if (K < 32 || K > bd::kMaxBits || K % 32) return fail(BD_EINVAL, "K=%d: need 32 <= K <= 512, K %% 32 == 0", K);
    if (mutual && !nn_ba) return fail(BD_EINVAL, "mutual needs nn_ba");
    if (a_off[0] != 0 || b_off[0] != 0) return fail(BD_EINVAL, "offsets must start at 0");
    for (int p = 0; p < n_pairs; ++p)
        if (a_off[p + 1] <= a_off[p] || b_off[p + 1] <= b_off[p])
            return fail(BD_EINVAL, "pair %d: empty or decreasing row range", p);
    if (a_off[n_pairs] > 0x7fffffffLL || b_off[n_pairs] > 0x7fffffffLL) return fail(BD_EINVAL, "too many rows");
    if (!aligned(a, 16) || !aligned(b, 16)) return fail(BD_EINVAL, "a/b must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    Workspace ws;
    int rc;
    if ((rc = ws_alloc(ws, bd::match_workspace_bytes(a_off[n_pairs], b_off[n_pairs], K, n_pairs), s)) != BD_OK)
        return rc;
    BD_CUDA(bd::launch_match(a, b, a_off, b_off, n_pairs, K, nn_ab, dist_ab, nn_ba, dist_ba, mutual, ws.p, s),
            "match kernels");
    return ok();
}

int bd_select_features(const uint8_t* patches, int M, const int32_t* triplets, int N, const int32_t* s_ap,
                       const int32_t* s_an, int tau, const int8_t* cand_pairs, const uint8_t* cand_radii, int J,
                       int64_t* loss, int32_t* bucket, void* stream) {
    if (!patches || !triplets || !s_ap || !s_an || !cand_pairs || !cand_radii || !loss || !bucket)
        return fail(BD_EINVAL, "NULL argument");
    if (M < 1 || M > bd::select_max_patches())
        return fail(BD_EINVAL, "M=%d out of [1, %d]", M, bd::select_max_patches());
    if (N < 1 || J < 1) return fail(BD_EINVAL, "N=%d, J=%d: need >= 1", N, J);
    if (!aligned(patches, 16)) return fail(BD_EINVAL, "patches must be 16-byte aligned");
    for (int j = 0; j < J; ++j) {
        for (int k = 0; k < 4; ++k)
            if (cand_pairs[4 * j + k] < -16 || cand_pairs[4 * j + k] > 15)
                return fail(BD_EINVAL, "candidate %d: offset outside [-16, 15]", j);
        if (cand_radii[j] > 7) return fail(BD_EINVAL, "candidate %d: radius > 7", j);
    }
    cudaStream_t s = (cudaStream_t)stream;
    Workspace ws;
    int rc;
    if ((rc = ws_alloc(ws, bd::select_workspace_bytes(M, J), s)) != BD_OK) return rc;
    BD_CUDA(bd::launch_select(patches, M, triplets, N, s_ap, s_an, tau, cand_pairs, cand_radii, J,
                              reinterpret_cast<long long*>(loss), bucket, ws.p, s),
            "select kernels");
    return ok();
}

int bd_integral_image(const uint8_t* images, int n_images, int H, int W, int64_t pitch, uint32_t* out,
                      void* stream) {
    int rc;
    if ((rc = check_images(images, n_images, H, W, pitch)) != BD_OK) return rc;
    if (!out || !aligned(out, 4)) return fail(BD_EINVAL, "out NULL or misaligned");
    if ((int64_t)H * W > 16843009LL) return fail(BD_EINVAL, "H*W too large for uint32 sums");
    cudaStream_t s = (cudaStream_t)stream;
    Workspace ws;
    const size_t band_bytes = bd::integral_workspace_bytes(n_images, H, W);
    if (band_bytes && (rc = ws_alloc(ws, band_bytes, s)) != BD_OK) return rc;
    BD_CUDA(bd::launch_integral(images, n_images, H, W, pitch, out, W + 1, s, band_bytes ? ws.p : nullptr),
            "integral kernel");
    return ok();
}

// bd_describe_warped_host: the describe_warped step from HOST buffers, host->device traffic
// overlapped with the kernels (DESIGN.md §6 "e2e").  Images are split into chunks; two
// device buffer sets alternate: chunk c's copies run on an H2D stream while chunk c-1 is
// described on the compute stream (the same bd_describe_warped_ex sequence as the device
// API) and chunk c-2's results return on a D2H stream.
int bd_describe_warped_host(const bad_model* bad, const hashsift_model* hs, const uint8_t* images, int n_images,
                            int H, int W, int64_t pitch, const bd_keypoint* kps, const int32_t* kp_image,
                            int64_t n_kp, int mode, uint32_t* out_bad, uint32_t* out_hs, uint8_t* kp_status,
                            int chunk_images) {
    if (mode != BD_WARP_NN && mode != BD_WARP_BILINEAR) return fail(BD_EINVAL, "unknown warp mode %d", mode);
    if (!bad && !hs) return fail(BD_EINVAL, "both models are NULL");
    if (n_kp < 0) return fail(BD_EINVAL, "n_kp < 0");
    if (n_kp == 0) return ok();
    if (bad && !out_bad) return fail(BD_EINVAL, "out_bad is NULL");
    if (hs && !out_hs) return fail(BD_EINVAL, "out_hs is NULL");
    if (!kps || !kp_image) return fail(BD_EINVAL, "kps / kp_image is NULL");
    if (!images || n_images < 1 || H < 1 || W < 1 || pitch < W)
        return fail(BD_EINVAL, "bad images (n_images=%d, H=%d, W=%d, pitch=%lld)", n_images, H, W, (long long)pitch);
    for (int64_t i = 1; i < n_kp; ++i)
        if (kp_image[i] < kp_image[i - 1]) return fail(BD_EINVAL, "kp_image must be non-decreasing (index %lld)", (long long)i);
    int rc;
    if (bad && (rc = check_device(bad->device)) != BD_OK) return rc;
    if (hs && (rc = check_device(hs->device)) != BD_OK) return rc;
    if (chunk_images < 1) chunk_images = std::max(1, (n_images + 7) / 8);
    chunk_images = std::min(chunk_images, n_images);
    const int K = bad ? bad->K : 0, N = hs ? hs->N : 0;
    const int64_t img_bytes = pitch * (int64_t)H;
    const int n_chunks = (n_images + chunk_images - 1) / chunk_images;
    // keypoint range [k0[c], k0[c+1]) of image chunk c; keypoints with an image index
    // outside [0, n_images) fall in no chunk and are reported invalid below
    std::vector<int64_t> k0(n_chunks + 1);
    for (int c = 0; c <= n_chunks; ++c)
        k0[c] = std::lower_bound(kp_image, kp_image + n_kp, std::min(c * chunk_images, n_images)) - kp_image;
    int64_t max_kp = 1;
    for (int c = 0; c < n_chunks; ++c) max_kp = std::max(max_kp, k0[c + 1] - k0[c]);
    // streams, events and the pinned staging of chunk-relative image indices are cached per
    // thread and device (creating them costs more than a chunk's kernels)
    struct Pipe {
        cudaStream_t cs = nullptr, xs = nullptr, ds = nullptr;  // compute, H2D, D2H
        cudaEvent_t h2d[2] = {}, cmp[2] = {}, done[2] = {};
        int32_t* stage = nullptr;  // pinned, 2 x max_kp
        int64_t stage_n = 0;
        bool init = false;
        int dev = 0;
        ~Pipe() {  // thread exit: release this thread's streams, events and staging
            if (!init && !stage) return;
            int cur = 0;
            if (cudaGetDevice(&cur) != cudaSuccess) return;  // runtime already shut down
            cudaSetDevice(dev);
            for (cudaStream_t t : {cs, xs, ds})
                if (t) cudaStreamDestroy(t);
            for (int b = 0; b < 2; ++b)
                for (cudaEvent_t e : {h2d[b], cmp[b], done[b]})
                    if (e) cudaEventDestroy(e);
            if (stage) cudaFreeHost(stage);
            cudaSetDevice(cur);
        }
    };
    static thread_local Pipe pipes[kMaxPipeDevices];
    int dev = 0;
    BD_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= kMaxPipeDevices) return fail(BD_EUNSUPPORTED, "device %d >= %d", dev, kMaxPipeDevices);
    Pipe& r = pipes[dev];
    r.dev = dev;
    if (!r.init) {
        BD_CUDA(cudaStreamCreateWithFlags(&r.cs, cudaStreamNonBlocking), "pipeline stream");
        BD_CUDA(cudaStreamCreateWithFlags(&r.xs, cudaStreamNonBlocking), "pipeline stream");
        BD_CUDA(cudaStreamCreateWithFlags(&r.ds, cudaStreamNonBlocking), "pipeline stream");
        for (int b = 0; b < 2; ++b) {
            BD_CUDA(cudaEventCreateWithFlags(&r.h2d[b], cudaEventDisableTiming), "pipeline event");
            BD_CUDA(cudaEventCreateWithFlags(&r.cmp[b], cudaEventDisableTiming), "pipeline event");
            BD_CUDA(cudaEventCreateWithFlags(&r.done[b], cudaEventDisableTiming), "pipeline event");
        }
        r.init = true;
    }
    if (r.stage_n < 2 * max_kp) {
        if (r.stage) cudaFreeHost(r.stage);
        r.stage = nullptr;
        r.stage_n = 0;
        BD_CUDA(cudaMallocHost(&r.stage, sizeof(int32_t) * 2 * max_kp), "pipeline pinned staging");
        r.stage_n = 2 * max_kp;
    }
    // device buffer sets: one stream-ordered pool allocation on the H2D stream (their first
    // user; the compute and D2H streams are ordered after it through the h2d / cmp events)
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t sz_img = up((size_t)img_bytes * chunk_images), sz_kp = up(sizeof(bd_keypoint) * max_kp),
                 sz_kpi = up(sizeof(int32_t) * max_kp), sz_ob = up((size_t)max_kp * K / 8),
                 sz_oh = up((size_t)max_kp * N / 8), sz_st = up((size_t)max_kp);
    const size_t per_set = sz_img + sz_kp + sz_kpi + sz_ob + sz_oh + sz_st;
    Workspace ws;
    if ((rc = ws_alloc(ws, 2 * per_set, r.xs)) != BD_OK) return rc;
    // on every return: the compute and D2H streams drain before ws is freed on the H2D stream
    struct Drain {
        Pipe& p;
        ~Drain() {
            cudaStreamSynchronize(p.cs);
            cudaStreamSynchronize(p.ds);
        }
    } drain{r};
    uint8_t* img[2];
    bd_keypoint* kpd[2];
    int32_t* kpi[2];
    uint32_t *ob[2], *oh[2];
    uint8_t* st[2];
    for (int b = 0; b < 2; ++b) {
        uint8_t* q = (uint8_t*)ws.p + b * per_set;
        img[b] = q;
        kpd[b] = (bd_keypoint*)(q += sz_img);
        kpi[b] = (int32_t*)(q += sz_kp);
        ob[b] = (uint32_t*)(q += sz_kpi);
        oh[b] = (uint32_t*)(q += sz_ob);
        st[b] = q + sz_oh;
    }
    for (int c = 0; c < n_chunks; ++c) {
        const int b = c & 1;
        const int i0 = c * chunk_images, ni = std::min(chunk_images, n_images - i0);
        const int64_t a = k0[c], m = k0[c + 1] - k0[c];
        int32_t* rel = r.stage + b * max_kp;
        if (c >= 2) {
            // buffer set b (and its pinned staging) is free once chunk c-2's results have left
            BD_CUDA(cudaEventSynchronize(r.done[b]), "pipeline wait");
        }
        for (int64_t i = 0; i < m; ++i) rel[i] = kp_image[a + i] - i0;
        BD_CUDA(cudaMemcpyAsync(img[b], images + img_bytes * i0, (size_t)img_bytes * ni, cudaMemcpyHostToDevice,
                                r.xs),
                "pipeline H2D");
        if (m) {
            BD_CUDA(cudaMemcpyAsync(kpd[b], kps + a, sizeof(bd_keypoint) * m, cudaMemcpyHostToDevice, r.xs),
                    "pipeline H2D");
            BD_CUDA(cudaMemcpyAsync(kpi[b], rel, sizeof(int32_t) * m, cudaMemcpyHostToDevice, r.xs), "pipeline H2D");
        }
        BD_CUDA(cudaEventRecord(r.h2d[b], r.xs), "pipeline event");
        BD_CUDA(cudaStreamWaitEvent(r.cs, r.h2d[b], 0), "pipeline event");
        if (m) {
            if ((rc = bd_describe_warped_ex(bad, hs, img[b], ni, H, W, pitch, kpd[b], kpi[b], m, mode, ob[b],
                                            oh[b], st[b], r.cs)) != BD_OK)
                return rc;
        }
        BD_CUDA(cudaEventRecord(r.cmp[b], r.cs), "pipeline event");
        BD_CUDA(cudaStreamWaitEvent(r.ds, r.cmp[b], 0), "pipeline event");
        if (m && bad)
            BD_CUDA(cudaMemcpyAsync(out_bad + a * (K / 32), ob[b], (size_t)m * K / 8, cudaMemcpyDeviceToHost, r.ds),
                    "pipeline D2H");
        if (m && hs)
            BD_CUDA(cudaMemcpyAsync(out_hs + a * (N / 32), oh[b], (size_t)m * N / 8, cudaMemcpyDeviceToHost, r.ds),
                    "pipeline D2H");
        if (m && kp_status)
            BD_CUDA(cudaMemcpyAsync(kp_status + a, st[b], (size_t)m, cudaMemcpyDeviceToHost, r.ds), "pipeline D2H");
        BD_CUDA(cudaEventRecord(r.done[b], r.ds), "pipeline event");
    }
    BD_CUDA(cudaStreamSynchronize(r.ds), "pipeline sync");
    BD_CUDA(cudaStreamSynchronize(r.cs), "pipeline sync");
    // keypoints whose image index is outside [0, n_images): zero rows, status 1 (as the
    // device API reports them)
    for (int64_t i = 0; i < n_kp; ++i)
        if (kp_image[i] < 0 || kp_image[i] >= n_images) {
            if (bad) std::fill(out_bad + i * (K / 32), out_bad + (i + 1) * (K / 32), 0u);
            if (hs) std::fill(out_hs + i * (N / 32), out_hs + (i + 1) * (N / 32), 0u);
            if (kp_status) kp_status[i] = 1;
        }
    return ok();
}

}  // extern "C"
