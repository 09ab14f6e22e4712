// internal.cuh — shared declarations of the sm_100a kernels behind include/bindesc.h.
// Nothing here is visible across the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/bindesc.h"

// Debug build (libbindesc_debug.so, -DBD_DEBUG_CHECKS; tests run against it with
// BINDESC_DEBUG=1): device-side bounds checks on every computed global / shared index that
// the kernels' own arithmetic produces, shared memory poisoned before use, and mbarrier
// watchdogs (tc.cuh) — this pool's replacement for compute-sanitizer (closed here).  A
// failed check prints the site and traps (the call then returns BD_ECUDA).
#ifdef BD_DEBUG_CHECKS
#define BD_CHECK(cond)                                                                              \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("bindesc debug check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, \
                   __LINE__, blockIdx.x, threadIdx.x);                                              \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#define BD_DEBUG 1
#else
#define BD_CHECK(cond) \
    do {               \
    } while (0)
#define BD_DEBUG 0
#endif

namespace bd {

// debug build: fill the whole dynamic shared memory of the launch with a poison pattern so
// a read of a never-written word yields garbage that the parity tests catch (no-op in release)
__device__ __forceinline__ void debug_poison_smem(void* smem) {
#ifdef BD_DEBUG_CHECKS
    uint32_t bytes;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(bytes));
    for (uint32_t i = threadIdx.x; i < bytes / 4; i += blockDim.x) static_cast<uint32_t*>(smem)[i] = 0xA5A5A5A5u;
    __syncthreads();
#else
    (void)smem;
#endif
}

constexpr int kMaxBits = 512;  // K, N upper bound (param-space tables)

// ---------------------------------------------------------------- BAD model --
// Image path (runtime geometry): one record per test.
struct ImgTest {
    int8_t dx1, dy1, dx2, dy2;
    int32_t r;
    float theta;
    int32_t t_full;  // floor(theta * (2r+1)^2), clamped to +-2^30 (R4, equal full areas)
};

// Image path, box-clustered evaluation (bad_image.cu): the 2K boxes (box 1 and box 2 of every
// test: offset + radius) sorted so that each run of 32 boxes is compact in offset space (a
// recursive median split), and per test the positions of its two boxes in that order.  Device
// table layout of the image path: [K ImgTest][2K ImgBox][K uint32 bpos (box1 | box2 << 16)]
// [32 lanes][kR = 2*KMAX/32 rounds] ImgBox: item 32 rho + lane at [lane][rho] (KMAX = 256 for
// K <= 256, else 512; zero-padded), so a lane loads its records as 16-byte vectors.
struct ImgBox {
    int8_t dx, dy;
    uint8_t r, pad;
};

// Patch path (fixed geometry, centre (16,16)): corner byte offsets into the packed
// integral and nthr1 = -(floor(theta*A1*A2) + 1), so that
// bit = [S1*A2 + S2*(-A1) + nthr1 < 0] (R4).  The areas come in one of two forms, chosen per
// model (PatchTable::dp2a):
//  * dp2a = 1 (every clamped area <= 127, i.e. radii <= 5): m1 = bytes (A2, 0, -A1, 0) and
//    m2 = bytes (0, A2, 0, -A1) as signed bytes, so with the packed box sums
//    S = S_A + 65536 S_B: dp2a.lo(S1, m1) + dp2a.hi(S2, m1) = S1_A*A2 - S2_A*A1 (patch A) and
//    the same with m2 gives patch B — the 16-bit halves are never unpacked;
//  * dp2a = 0: m1 = -A1, m2 = A2 as integers (the halves are unpacked and multiplied).
struct __align__(16) PatchTest {
    uint32_t off[8];  // c0 - c1 - c2 + c3 = S1 ; c4 - c5 - c6 + c7 = S2
    int32_t nthr1;    // -(floor(theta * A1 * A2) + 1), theta*A1*A2 clamped to +-2^30
    int32_t m1, m2;   // areas, see above
    int32_t pad;
};
struct PatchTable {
    PatchTest t[kMaxBits];
    int dp2a;  // area form of the records (see PatchTest)
};

// ----------------------------------------------------------- launchers --------
// All return cudaGetLastError() of their launches.
// ws: integral_workspace_bytes(n, H, W) bytes (small images use a banded column pass), or
// NULL for the single-pass kernels
cudaError_t launch_integral(const uint8_t* img, int n, int H, int W, int64_t pitch, uint32_t* out,
                            int64_t out_pitch, cudaStream_t s, void* ws);
size_t integral_workspace_bytes(int n, int H, int W);
cudaError_t launch_integral16(const uint8_t* img, int n, int H, int W, int64_t pitch, uint16_t* out,
                              int64_t out_pitch, cudaStream_t s, void* ws);
// vectorised uint16 integral (W, pitch multiples of 8, W <= 2048): column c of row y at
// out[y * out_pitch + c + 7] (out_pitch % 8 == 0, out 16-byte aligned)
bool integral16_vec_ok(const uint8_t* img, int n, int H, int W, int64_t pitch);
size_t integral16_vec_workspace_bytes(int n, int H, int W);
cudaError_t launch_integral16_vec(const uint8_t* img, int n, int H, int W, int64_t pitch, uint16_t* out,
                                  int64_t out_pitch, cudaStream_t s, void* ws);
// integral: ii_bytes = 4 (uint32, exact) or 2 (uint16, mod 2^16: box radius <= 7 only)
// small batches (n_kp <= bad_image_local_max_kp(), unscaled radii): one launch, a CTA per
// keypoint with the integral of its window built in shared memory (bad_image.cu)
int bad_image_local_max_kp();
cudaError_t launch_bad_image_local(const uint8_t* images, int n_img, int H, int W, int64_t pitch,
                                   const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp, const ImgTest* tests,
                                   int K, uint32_t* out, uint8_t* status, cudaStream_t s);
cudaError_t launch_bad_image(const uint8_t* images, int n_img, int H, int W, int64_t pitch,
                             const void* integral, int ii_bytes, int64_t ipitch, const bd_keypoint* kps,
                             const int32_t* kp_image, int64_t n_kp, const ImgTest* tests, int K,
                             int scale_radius, uint32_t* out, uint8_t* status, void* order_ws, cudaStream_t s);
// workspace for serving keypoints in spatial order (0 = input order; order_ws = NULL then)
size_t bad_image_order_bytes(int n_img, int H, int W, int64_t n_kp);
// status (nullable): rows whose status byte is nonzero are written as zero (invalid keypoints)
cudaError_t launch_bad_patches(const uint8_t* patches, int64_t n, const PatchTable& tab, int K,
                               uint32_t* out, const uint8_t* status, cudaStream_t s);
// tensor-core build of the same kernel (bad_patch_tc.cu), K <= 256
cudaError_t launch_bad_patches_tc(const uint8_t* patches, int64_t n, const PatchTable& tab, int K,
                                  uint32_t* out, const uint8_t* status, cudaStream_t s);
// mode: BD_WARP_NN or BD_WARP_BILINEAR
cudaError_t launch_warp_nn(const uint8_t* images, int n_img, int H, int W, int64_t pitch, int mode,
                           const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp,
                           uint8_t* patches, uint8_t* status, cudaStream_t s);
// root: apply the RootSIFT transform (BD_HS_ROOTSIFT) after normalisation
cudaError_t launch_sift(const uint8_t* patches, int64_t n, float* sift, int root, cudaStream_t s);
cudaError_t launch_project(const float* sift, int64_t n, const float* w /*[N][128]*/, const float* bias, int N,
                           uint32_t* out, const uint8_t* status, cudaStream_t s);
cudaError_t launch_zero_invalid(const uint8_t* status, int64_t n, uint32_t* out, int words,
                                cudaStream_t s);

// NEXT-1 matcher (match.cu); ws = match_workspace_bytes(...) bytes of device memory
cudaError_t launch_match(const uint32_t* a, const uint32_t* b, const int64_t* a_off, const int64_t* b_off,
                         int n_pairs, int K, int32_t* nn_ab, int32_t* dist_ab, int32_t* nn_ba, int32_t* dist_ba,
                         uint8_t* mutual, void* ws, cudaStream_t s);
size_t match_workspace_bytes(int64_t n_a, int64_t n_b, int K, int n_pairs);

// NEXT-4 feature-selection hot loop (select.cu); ws = select_workspace_bytes(M, J)
cudaError_t launch_select(const uint8_t* patches, int M, const int32_t* trip, int N, const int32_t* sap,
                          const int32_t* san, int tau, const int8_t* cand_pairs, const uint8_t* cand_radii, int J,
                          long long* loss, int32_t* bucket, void* ws, cudaStream_t s);
size_t select_workspace_bytes(int M, int J);
int select_max_patches();

int num_sms();  // of the current device
// cudaFuncSetAttribute(fn, MaxDynamicSharedMemorySize, bytes) once per (device, kernel)
// (the attribute is per device: a process-wide flag would break a second GPU)
cudaError_t ensure_smem_attr(const void* fn, int bytes);

// RAII trace scope (profile.cu): records a CUDA event pair around the launches made in its
// lifetime when bd_profile_start() is active.
class ProfScope {
   public:
    ProfScope(const char* name, cudaStream_t s);
    ~ProfScope();
    ProfScope(const ProfScope&) = delete;
    ProfScope& operator=(const ProfScope&) = delete;

   private:
    cudaStream_t s_;
    int idx_;
};

}  // namespace bd
