/*
 * bindesc.h — C ABI of the B200 (sm_100a) batched BAD / HashSIFT descriptor extractor.
 *
 * Method: arXiv 2108.08380, "Revisiting Binary Local Image Description for Resource
 * Limited Devices".  Citations:  P:n = /root/reference/PAPER.md line n,
 * S:n = /root/reference/SPEC.md line n, R# = reading
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All data pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless the
 *    argument is marked [host].  The caller owns every buffer; the library owns only the
 *    opaque model handles (freed by *_destroy) and transient stream-ordered workspace.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every
 *    compute call only ENQUEUES work on `stream` and returns; it never synchronises.
 *  - Return value: BD_OK (0) or a negative bd_status.  Argument errors are detected on
 *    the host before anything is enqueued; bd_last_error() gives a thread-local message.
 *    No C++ exception crosses this boundary.
 *  - Images: n_images x H rows of `pitch` bytes, uint8 grey levels, row-major, x = column,
 *    y = row, origin top-left.  pitch >= W.
 *  - Patches: n x 32 x 32 uint8, contiguous, 1024 bytes each ("re-scaled to the same
 *    size, 32x32 pixels"); the base pointer must be 16-byte aligned.
 *  - Descriptors: n x (K/32) uint32 words; bit k of a descriptor is bit (k % 32) of word
 *    k / 32, i.e. LSB-first little-endian bytes (R16).
 *  - Keypoints (bd_keypoint): centre (x, y) in pixels (sub-pixel allowed), orientation
 *    `angle` in radians, `scale` > 0 (1 = the 32x32 test frame in image pixels; a detector
 *    diameter d maps to scale = 6.75 d / 32 on the caller side).  A keypoint is
 *    invalid if a field is non-finite, scale <= 0, the centre lies outside
 *    [0, W-1] x [0, H-1] or its image index is outside [0, n_images): it yields an all-zero
 *    row and kp_status = 1 (never undefined behaviour).
 *  - Model handles are immutable after create, so concurrent compute calls on different
 *    streams are safe.
 */
#ifndef BINDESC_H
#define BINDESC_H

#include <stdint.h>

#if defined(__GNUC__)
#define BD_API __attribute__((visibility("default")))
#else
#define BD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BD_OK = 0,
    BD_EINVAL = -1,        /* bad argument (null pointer, K % 32 != 0, offset out of range ...) */
    BD_ENOMEM = -2,        /* device or host allocation failed */
    BD_ECUDA = -3,         /* a CUDA launch / runtime call failed (message in bd_last_error) */
    BD_EUNSUPPORTED = -4   /* no sm_100 device or feature unavailable */
} bd_status;

typedef struct bd_keypoint {
    float x, y;      /* centre, pixels */
    float angle;     /* radians; the offsets of the 32x32 frame are rotated by it (R9) */
    float scale;     /* > 0; the offsets are multiplied by it (R8: box radii are not) */
} bd_keypoint;

typedef struct bad_model bad_model;
typedef struct hashsift_model hashsift_model;

/* ---------------------------------------------------------------- BAD -- */

/* Build a BAD-K model from K box-pair tests (weak descriptor
 * h(x; f, theta) = +1 iff f(x) <= theta, f = mean of the (2r+1)^2 box at u1 minus the mean
 * of the box at u2; h(x) = [h_1 ... h_K]).
 *   pairs       [host] K x 4 int8 {dx1, dy1, dx2, dy2}: offsets of u1, u2 from the keypoint
 *               in the 32x32 frame, each in [-16, 15] (R7: the patch centre is pixel 16)
 *   radii       [host] K uint8 box radii r in [0, 7] (box side 2r+1, R1)
 *   thresholds  [host] K float, finite, grey levels (search space [-255, 255])
 *   K           number of tests, 32 <= K <= 512, K % 32 == 0 (build restriction)
 *   out         receives the handle; destroy with bad_destroy.
 * Errors: BD_EINVAL on null pointers, K out of range, offsets/radii out of range,
 * non-finite thresholds; BD_ENOMEM. */
BD_API int bad_create(const int8_t* pairs, const uint8_t* radii, const float* thresholds, int K,
               bad_model** out);
BD_API void bad_destroy(bad_model* m);
BD_API int bad_num_bits(const bad_model* m);

/* BAD-K on whole images (configs[0], [1]): one integral image per image ("can be
 * efficiently computed using integral images"), then per keypoint K tests whose
 * sample points are p_j = round(kp + R(angle) * scale * (dx_j, dy_j)) with the fixed-order
 * fp32 rule of R6, boxes clamped to the image and averaged over the clamped area (R5), the
 * comparison exact (R4).  Bit k = [f_k <= theta_k] (R2).
 *   images, n_images, H, W, pitch   see conventions; 1 <= H, W <= 32768
 *   kps       n_kp keypoints;  kp_image  n_kp int32 image index per keypoint (nullable:
 *             all keypoints on image 0)
 *   out_bits  n_kp x K/32 uint32
 *   kp_status nullable, n_kp uint8: 0 ok, 1 invalid keypoint (zero row)
 * n_kp == 0 returns BD_OK without work.  Uses stream-ordered workspace: the integral
 * images, (W+1)(H+1) x n_images x 2 bytes (stored mod 2^16, exact for radii <= 7; 4 bytes
 * per entry for models created with BD_BAD_SCALE_RADIUS), plus, for large batches, 4 bytes
 * per keypoint and per 64x64-pixel image cell for serving the keypoints in spatial order
 * (results do not depend on it). */
BD_API int bad_compute(const bad_model* m, const uint8_t* images, int n_images, int H, int W,
                int64_t pitch, const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp,
                uint32_t* out_bits, uint8_t* kp_status, void* stream);

/* BAD-K on pre-extracted 32x32 patches (configs[2]): each patch evaluated at its centre
 * pixel (16, 16) with scale 1 and angle 0 (R7); boxes clamped to the patch (R5). */
BD_API int bad_compute_patches(const bad_model* m, const uint8_t* patches, int64_t n, uint32_t* out_bits,
                        void* stream);

/* ------------------------------------------------------- HashSIFT -- */

/* Build a HashSIFT-N model from B = [W | b] (D(x) = sgn(B [f(x)^T, 1]^T)).
 *   B   [host] N x 129 float, row-major, finite; column 128 is the bias b
 *   N   32 <= N <= 512, N % 32 == 0
 * Errors: BD_EINVAL, BD_ENOMEM. */
BD_API int hashsift_create(const float* B, int N, hashsift_model** out);
BD_API void hashsift_destroy(hashsift_model* m);
BD_API int hashsift_num_bits(const hashsift_model* m);

/* HashSIFT-N on 32x32 patches (configs[3]): SIFT 4x4x8 histogram per patch (R10:
 * replicate-border central differences, Gaussian sigma 16, trilinear binning, L2-normalise,
 * clip 0.2, renormalise, zero stays zero), then p = W v + b and bit k = [p_k >= 0] (R15).
 *   out_bits  n x N/32 uint32
 *   out_sift  nullable, n x 128 float: the SIFT vectors (for parity tests). */
BD_API int hashsift_compute_patches(const hashsift_model* m, const uint8_t* patches, int64_t n,
                             uint32_t* out_bits, float* out_sift, void* stream);

/* HashSIFT-N on keypoints of whole images: nearest-neighbour 32x32 patch warp (below), then
 * as hashsift_compute_patches.  kp_status as in bad_compute. */
BD_API int hashsift_compute(const hashsift_model* m, const uint8_t* images, int n_images, int H, int W,
                     int64_t pitch, const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp,
                     uint32_t* out_bits, float* out_sift, uint8_t* kp_status, void* stream);

/* --------------------------------------------------- warped-patch path (configs[4]) -- */

/* Nearest-neighbour patch warp (S:62-70 with the NN reading, R20): patch pixel (u, v)
 * (u = column) takes the image pixel at the sample point of offset (u-16, v-16) under the
 * R6 rule, clamped into the image (border replicate).
 *   out_patches  n_kp x 32 x 32 uint8 (16-byte aligned); invalid keypoints -> zero patch. */
BD_API int bd_warp_patches(const uint8_t* images, int n_images, int H, int W, int64_t pitch,
                    const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp,
                    uint8_t* out_patches, uint8_t* kp_status, void* stream);

/* configs[4] step: NN-warp every keypoint's patch once, then BAD-K (on the warped patch,
 * R20) and HashSIFT-N on it.  Either model may be NULL (its output is then skipped).
 *   out_bad  n_kp x K/32 (nullable iff bad == NULL);  out_hs  n_kp x N/32 (nullable iff
 *   hs == NULL).  Invalid keypoints give zero rows in both outputs and kp_status = 1. */
BD_API int bd_describe_warped(const bad_model* bad, const hashsift_model* hs, const uint8_t* images,
                       int n_images, int H, int W, int64_t pitch, const bd_keypoint* kps,
                       const int32_t* kp_image, int64_t n_kp, uint32_t* out_bad, uint32_t* out_hs,
                       uint8_t* kp_status, void* stream);

/* ------------------------------------------------ NEXT-2 / NEXT-3: variants (§8(f)) -- */

/* Model / warp option flags. */
enum {
    BD_BAD_SCALE_RADIUS = 1,  /* bad_create_ex: image-path box radius r' = floor(r*scale + 1/2),
                                 r*scale and + 1/2 in fp32 (reading R27; closer to the normalised
                                 frame of P:127); the patch path (scale 1) is unchanged */
    BD_HS_ROOTSIFT = 1,       /* hashsift_create_ex: RootSIFT pre-hash transform v' = sqrt(v/sum v)
                                 of the SIFT vector (zero stays zero) */
    BD_WARP_NN = 0,           /* warp mode: nearest neighbour, offsets (u-16, v-16), R6 (default) */
    BD_WARP_BILINEAR = 1      /* warp mode: bilinear (reading R28): offsets (u-15.5, v-15.5),
                                 fp32 weights in a fixed order, border replicate, round half up */
};

/* bad_create with flags (0 = bad_create).  Errors as bad_create; unknown flags -> BD_EINVAL. */
BD_API int bad_create_ex(const int8_t* pairs, const uint8_t* radii, const float* thresholds, int K, int flags,
                         bad_model** out);

/* hashsift_create with flags (0 = hashsift_create). */
BD_API int hashsift_create_ex(const float* B, int N, int flags, hashsift_model** out);

/* bd_warp_patches / bd_describe_warped with an explicit warp mode (BD_WARP_NN or
 * BD_WARP_BILINEAR); the mode-less calls use BD_WARP_NN. */
BD_API int bd_warp_patches_ex(const uint8_t* images, int n_images, int H, int W, int64_t pitch,
                              const bd_keypoint* kps, const int32_t* kp_image, int64_t n_kp, int mode,
                              uint8_t* out_patches, uint8_t* kp_status, void* stream);
BD_API int bd_describe_warped_ex(const bad_model* bad, const hashsift_model* hs, const uint8_t* images,
                                 int n_images, int H, int W, int64_t pitch, const bd_keypoint* kps,
                                 const int32_t* kp_image, int64_t n_kp, int mode, uint32_t* out_bad,
                                 uint32_t* out_hs, uint8_t* kp_status, void* stream);

/* bd_describe_warped_ex from HOST memory (the end-to-end call; DESIGN.md §6 "e2e").
 * Same operation and results as bd_describe_warped_ex, but images, kps, kp_image and the
 * outputs are host pointers, and the call is SYNCHRONOUS (returns when every output is in
 * host memory).  The images are split into chunks of chunk_images (<= 0: n_images / 8,
 * rounded up); per chunk its images and keypoints are copied to the device while the
 * previous chunk is described, so with PINNED host buffers (cudaHostAlloc) the copies
 * overlap the kernels; pageable buffers give the same results without the overlap.
 *   kp_image  n_kp int32, required, NON-DECREASING (keypoints grouped by image);
 *             indices outside [0, n_images) give zero rows and kp_status = 1
 * Allocates 2 x (chunk images + chunk keypoints + outputs) of device memory and a pinned
 * staging buffer for the call's duration; uses private streams, and the library's CURRENT
 * device.  Errors: as bd_describe_warped_ex, plus BD_EINVAL for a decreasing kp_image. */
BD_API int bd_describe_warped_host(const bad_model* bad, const hashsift_model* hs, const uint8_t* images,
                                   int n_images, int H, int W, int64_t pitch, const bd_keypoint* kps,
                                   const int32_t* kp_image, int64_t n_kp, int mode, uint32_t* out_bad,
                                   uint32_t* out_hs, uint8_t* kp_status, int chunk_images);

/* ------------------------------------------- NEXT-1: Hamming NN / mutual-NN matching -- */

/* Brute-force Hamming matching of binary descriptor sets (the paper's
 * pipeline step "BFMatcher with Mutual Nearest Neighbors (MNN)", P:559-560, P:566-570;
 * S:514-540).  For every query a_i the train descriptor b_j with minimal Hamming distance,
 * ties -> lowest j.  The similarity of P:123, S(x, y) = h(x)^T h(y) = K - 2 Hamming
 * with h in {-1, +1}^K, is computed EXACTLY as a +-1 block-scaled FP4 tensor-core GEMM
 * (tcgen05 kind::mxf4, e2m1 +-1.0, unit scales, f32 accumulators holding integers
 * |S| <= 512); the NN is the row argmax of S.
 *   a, b         descriptors, K/32 uint32 words per row (R16 packing), device
 *   a_off, b_off [host] n_pairs + 1 row offsets: pair p matches rows [a_off[p], a_off[p+1])
 *                of a against rows [b_off[p], b_off[p+1]) of b; every pair non-empty
 *   K            bits per descriptor, 32 <= K <= 512, K % 32 == 0
 *   nn_ab        n_a int32: index of the nearest b row WITHIN its pair's block
 *   dist_ab      n_a int32: its Hamming distance (nullable)
 *   nn_ba, dist_ba  the same for b against a (nullable; required when mutual != NULL)
 *   mutual       n_a uint8 (nullable): 1 iff nn_ba[nn_ab[i]] == i
 * Uses stream-ordered workspace of about (n_a + n_b) * K / 2 bytes.  Errors: BD_EINVAL on null
 * pointers, bad K, empty or decreasing offsets, misalignment. */
BD_API int bd_match_hamming(const uint32_t* a, const int64_t* a_off, const uint32_t* b, const int64_t* b_off,
                            int n_pairs, int K, int32_t* nn_ab, int32_t* dist_ab, int32_t* nn_ba,
                            int32_t* dist_ba, uint8_t* mutual, void* stream);

/* ------------------------------------------- NEXT-4: feature-selection hot loop (§8(f)) -- */

/* One iteration of BAD's greedy feature selection (Algorithm 1 lines 4-12) with
 * the integer-sort threshold search of Algorithm 2 (m = 5110 buckets of 0.1 over
 * [-255, 255]), for J candidate box pairs over N triplets of 32x32 patches.
 * Readings R29-R31: per triplet L_i(theta) = [tau - S_ap - h_a h_p + S_an +
 * h_a h_n]_+ (Eq. 2) with integer prior similarities S^(t-1) and integer margin tau;
 * h = +1 iff f <= theta with f = mean(box1) - mean(box2) (clamped boxes at (16,16) + offsets);
 * bucket b(f) = floor((f + 255) * 10) exactly; the sweep over bucket upper edges is exact
 * at ties.  Everything is integer arithmetic, so results are deterministic and exact.
 *   patches    M x 1024 uint8 (device), M <= 40000
 *   triplets   N x 3 int32 (device): patch indices (a, p, n), each in [0, M)
 *   s_ap, s_an N int32 (device): S^(t-1)(a_i, p_i), S^(t-1)(a_i, n_i)
 *   cand_pairs [host] J x 4 int8 in [-16, 15]; cand_radii [host] J uint8 in [0, 7]
 *   loss       J int64: L* of each candidate;  bucket  J int32: b* (-1: theta = -inf, all
 *              bits -1); a threshold realising b* is -255 + (b*+1)/10 - 1e-6
 * Uses (1089 * 2 * M + 48 * J) bytes of stream-ordered workspace.  Errors: BD_EINVAL on
 * null pointers, M out of range, N < 1, J < 1, bad candidate geometry. */
BD_API int bd_select_features(const uint8_t* patches, int M, const int32_t* triplets, int N, const int32_t* s_ap,
                              const int32_t* s_an, int tau, const int8_t* cand_pairs, const uint8_t* cand_radii,
                              int J, int64_t* loss, int32_t* bucket, void* stream);

/* ------------------------------------------------------------------- utilities -- */

/* Integral image: out is n_images x (H+1) x (W+1) uint32 with
 * out(r, c) = sum of pixels with row < r and col < c; first row and column zero.
 * H * W * 255 must fit in uint32 (H * W <= 16843009).  Exposed for the a1 parity test. */
BD_API int bd_integral_image(const uint8_t* images, int n_images, int H, int W, int64_t pitch,
                      uint32_t* out, void* stream);

/* Kernel-level tracing (CUDA events around every kernel the library launches).
 * bd_profile_start() clears the counters and starts recording; bd_profile_stop() stops.
 * bd_profile_query(i, ...) waits for the recorded events and returns, for the i-th kernel
 * name seen (i = 0, 1, ...), its total launches and total device milliseconds; it returns
 * BD_EINVAL when i is past the last name.  Recording costs two cudaEventRecord per launch. */
BD_API int bd_profile_start(void);
BD_API int bd_profile_stop(void);
BD_API int bd_profile_query(int i, const char** name, int64_t* launches, double* ms);

/* Thread-local message describing the last non-OK return on this thread ("" if none). */
BD_API const char* bd_last_error(void);

/* ABI version (major * 10000 + minor * 100 + patch). */
BD_API int bd_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BINDESC_H */
