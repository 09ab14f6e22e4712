/*
 * bindesc_oracle.c — the CPU ORACLE for the BAD / HashSIFT extraction path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2108_08380_b200/) never links, imports or calls it, and this file
 * includes nothing from the product path (it even duplicates the keypoint struct).
 *
 * It is deliberately plain and slow: box sums are brute-force double loops (no
 * integral images), SIFT is a direct per-pixel loop in float64, the projection is
 * a float64 dot product.  Each function cites the passage it follows:
 *   P:n  = /root/reference/PAPER.md line n   (arXiv 2108.08380, LaTeX source)
 *   S:n  = /root/reference/SPEC.md line n
 *   R#   = reading # of SURVEY.md §8(c), restated in DESIGN.md §2
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *        (no FMA contraction: the fp32 sample-point rule R6 is evaluated op by op)
 *
 * Parity status per function: every function below is pinned by a
 * `-m "not gpu"` test in tests/test_oracle_*.py; the SIFT conventions (R10) are
 * pinned by closed forms and invariants only — the paper prints no SIFT values.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846

typedef struct { float x, y, angle, scale; } or_keypoint; /* duplicate of bd_keypoint, by design */

/* threads: the caller's count, else BINDESC_ORACLE_THREADS, else OpenMP's default */
static int or_nthreads(int nt) {
#ifdef _OPENMP
    if (nt > 0) return nt;
    const char* e = getenv("BINDESC_ORACLE_THREADS");
    if (e && atoi(e) > 0) return atoi(e);
    return omp_get_max_threads();
#else
    (void)nt;
    return 1;
#endif
}

int or_max_threads(void) { return or_nthreads(0); }

/* ------------------------------------------------------------------------- */
/* Keypoint frame.  R6: a = (float)(scale*cos(angle)), b = (float)(scale*sin(angle)),
 * trig in float64 (glibc).  BJ.ns: "p1 and p2 rotated and scaled by the keypoint's
 * angle and scale".  Returns 1 if either float64 value lies within 4 float64-ulp of
 * an fp32 rounding boundary (a "fragile" keypoint, R6), else 0. */
static int fragile_round(double c) {
    float f = (float)c;
    float lo = nextafterf(f, -INFINITY), hi = nextafterf(f, INFINITY);
    double m1 = 0.5 * ((double)f + (double)lo), m2 = 0.5 * ((double)f + (double)hi);
    double u = fabs(c) > 0 ? ldexp(1.0, ilogb(c) - 52) : ldexp(1.0, -1074);
    return fabs(c - m1) < 4 * u || fabs(c - m2) < 4 * u;
}

/* Test hook (tests/test_oracle_bad.py pins the fragility rule itself): the R6 flag of one
 * float64 coefficient and the (a, b, fragile) frame of one keypoint, exactly as or_bad_image
 * computes them. */
int or_fragile_round(double c) { return fragile_round(c); }

static int kp_frame(const or_keypoint* kp, float* a, float* b);
int or_kp_frame(const float* kp4, float* ab) {
    or_keypoint kp;
    memcpy(&kp, kp4, sizeof kp);
    return kp_frame(&kp, ab, ab + 1);
}

static int kp_frame(const or_keypoint* kp, float* a, float* b) {
    double c = (double)kp->scale * cos((double)kp->angle);
    double s = (double)kp->scale * sin((double)kp->angle);
    *a = (float)c;
    *b = (float)s;
    return fragile_round(c) || fragile_round(s);
}

/* Sample point rule (R6; "boxes ... centered in pixels
 * u_i of patch x"): offsets (dx,dy) in the 32x32 test frame are rotated and scaled,
 *   X = x + (a*dx - b*dy),  Y = y + (b*dx + a*dy)    (fp32, this exact order, no FMA)
 * then rounded half-up: p = floor(X + 0.5) evaluated in float64.
 * *margin receives min distance of X, Y to a rounding boundary n + 1/2. */
static void sample_point(float x, float y, float a, float b, int dx, int dy,
                         long* px, long* py, double* margin) {
    float fdx = (float)dx, fdy = (float)dy;
    float t1 = a * fdx;
    float t2 = b * fdy;
    float X = x + (t1 - t2);
    float t3 = b * fdx;
    float t4 = a * fdy;
    float Y = y + (t3 + t4);
    double Xd = (double)X + 0.5, Yd = (double)Y + 0.5;
    *px = (long)floor(Xd);
    *py = (long)floor(Yd);
    if (margin) {
        double mx = fabs(Xd - floor(Xd + 0.5)), my = fabs(Yd - floor(Yd + 0.5));
        *margin = mx < my ? mx : my;
    }
}

static long clampl(long v, long lo, long hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Box sum by brute force (BJ.ns: "computes box sums by brute-force summation, not
 * integral images").  P:118: "average gray values of two boxes of size s centered in
 * pixels u_i"; R1: box side = 2r+1; R5 / S:56: centre clamped into the image, the
 * box clamped to the image, average over the clamped area (A >= 1). */
static void box_sum(const uint8_t* img, long H, long W, long pitch, long cx, long cy, int r,
                    int64_t* S, int64_t* A) {
    cx = clampl(cx, 0, W - 1);
    cy = clampl(cy, 0, H - 1);
    long x0 = clampl(cx - r, 0, W - 1), x1 = clampl(cx + r, 0, W - 1);
    long y0 = clampl(cy - r, 0, H - 1), y1 = clampl(cy + r, 0, H - 1);
    int64_t s = 0;
    for (long yy = y0; yy <= y1; ++yy)
        for (long xx = x0; xx <= x1; ++xx) s += img[yy * pitch + xx];
    *S = s;
    *A = (int64_t)(x1 - x0 + 1) * (int64_t)(y1 - y0 + 1);
}

/* One BAD weak descriptor (h(x; f, theta) = +1 if f(x) <= theta, else -1;
 * f = mean(box at u1) - mean(box at u2), R3) as the bit [h = +1] (R2).
 * f <= theta  <=>  S1*A2 - S2*A1 <= theta*A1*A2  (A1*A2 > 0), evaluated exactly: the
 * left side is an integer < 2^53 and theta (fp32, 24-bit mantissa) times A1*A2 (< 2^14)
 * is exact in float64 (R4). */
static int bad_bit(int64_t S1, int64_t A1, int64_t S2, int64_t A2, float theta, int* tie) {
    double lhs = (double)(S1 * A2 - S2 * A1);
    double rhs = (double)theta * (double)(A1 * A2);
    if (tie) *tie = (lhs == rhs);
    return lhs <= rhs;
}

/* BAD-K descriptor of one keypoint on one image.  P:122: h(x) = [h_1..h_K]; packing
 * LSB-first (R16): bit k -> byte k/8, bit k%8.  out: ceil(K/8) bytes. */
static void bad_one(const uint8_t* img, long H, long W, long pitch, const or_keypoint* kp,
                    const int8_t* pairs, const uint8_t* radii, const float* thr, int K,
                    uint8_t* out, double* margin_out, int* ties_out) {
    float a, b;
    kp_frame(kp, &a, &b);
    double mmin = 1.0;
    int ties = 0;
    memset(out, 0, (size_t)(K + 7) / 8);
    for (int k = 0; k < K; ++k) {
        long p1x, p1y, p2x, p2y;
        double m1, m2;
        sample_point(kp->x, kp->y, a, b, pairs[4 * k + 0], pairs[4 * k + 1], &p1x, &p1y, &m1);
        sample_point(kp->x, kp->y, a, b, pairs[4 * k + 2], pairs[4 * k + 3], &p2x, &p2y, &m2);
        if (m1 < mmin) mmin = m1;
        if (m2 < mmin) mmin = m2;
        int64_t S1, A1, S2, A2;
        box_sum(img, H, W, pitch, p1x, p1y, radii[k], &S1, &A1);
        box_sum(img, H, W, pitch, p2x, p2y, radii[k], &S2, &A2);
        int tie = 0;
        int bit = bad_bit(S1, A1, S2, A2, thr[k], &tie);
        ties += tie;
        if (bit) out[k >> 3] |= (uint8_t)(1u << (k & 7));
    }
    if (margin_out) *margin_out = mmin;
    if (ties_out) *ties_out = ties;
}

/* Keypoint validity: finite fields, scale > 0, centre inside
 * [0, W-1] x [0, H-1], image index in range. */
static int kp_valid(const or_keypoint* kp, int32_t img_idx, long n_img, long H, long W) {
    if (!(isfinite(kp->x) && isfinite(kp->y) && isfinite(kp->angle) && isfinite(kp->scale))) return 0;
    if (!(kp->scale > 0.0f)) return 0;
    if (kp->x < 0.0f || kp->y < 0.0f || kp->x > (float)(W - 1) || kp->y > (float)(H - 1)) return 0;
    if (img_idx < 0 || img_idx >= n_img) return 0;
    return 1;
}

/* BAD on images (configs[0], [1]).  images: n_img x H rows of `pitch` bytes.
 * kp_image[i]: image of keypoint i (NULL -> all on image 0).  out: n_kp x ceil(K/8).
 * status (nullable): 0 ok, 1 invalid keypoint (zero row).  fragile (nullable): 1 when the
 * keypoint's trig coefficients or any sample lies within 1e-4 of a rounding boundary (R6).
 * ties (nullable): number of exact f == theta ties per keypoint. */
void or_bad_image(const uint8_t* images, long n_img, long H, long W, long pitch,
                  const float* kps4, const int32_t* kp_image, long n_kp,
                  const int8_t* pairs, const uint8_t* radii, const float* thr, int K,
                  uint8_t* out, uint8_t* status, uint8_t* fragile, int32_t* ties, int nthreads) {
    const long row = (K + 7) / 8;
#pragma omp parallel for schedule(dynamic, 8) num_threads(or_nthreads(nthreads))
    for (long i = 0; i < n_kp; ++i) {
        or_keypoint kp;
        memcpy(&kp, kps4 + 4 * i, sizeof kp);
        int32_t ii = kp_image ? kp_image[i] : 0;
        if (!kp_valid(&kp, ii, n_img, H, W)) {
            memset(out + i * row, 0, (size_t)row);
            if (status) status[i] = 1;
            if (fragile) fragile[i] = 0;
            if (ties) ties[i] = 0;
            continue;
        }
        double m;
        int t;
        bad_one(images + (size_t)ii * (size_t)H * (size_t)pitch, H, W, pitch, &kp, pairs, radii,
                thr, K, out + i * row, &m, &t);
        if (status) status[i] = 0;
        if (fragile) {
            float a, b;
            fragile[i] = (uint8_t)(kp_frame(&kp, &a, &b) || m < 1e-4);
        }
        if (ties) ties[i] = t;
    }
}

/* BAD on pre-extracted 32x32 patches (configs[2]), each evaluated at the patch centre
 * pixel (16,16) with scale 1 and angle 0 (R7): the same rule with a = 1, b = 0. */
void or_bad_patches(const uint8_t* patches, long n, const int8_t* pairs, const uint8_t* radii,
                    const float* thr, int K, uint8_t* out, int32_t* ties, int nthreads) {
    const long row = (K + 7) / 8;
#pragma omp parallel for schedule(dynamic, 64) num_threads(or_nthreads(nthreads))
    for (long i = 0; i < n; ++i) {
        or_keypoint kp = {16.0f, 16.0f, 0.0f, 1.0f};
        int t;
        bad_one(patches + (size_t)i * 1024, 32, 32, 32, &kp, pairs, radii, thr, K, out + i * row,
                NULL, &t);
        if (ties) ties[i] = t;
    }
}

/* Nearest-neighbour patch warp (configs[4], R20; S:62-70 with the NN reading of
 * SURVEY §8(a) a5): patch pixel (u = col, v = row), u, v in 0..31, takes the image
 * pixel at the sample point of offset (u-16, v-16) (same rule as BAD, R6), clamped
 * into the image (border replicate).  Invalid keypoints give a zero patch. */
void or_warp_nn(const uint8_t* images, long n_img, long H, long W, long pitch, const float* kps4,
                const int32_t* kp_image, long n_kp, uint8_t* out, uint8_t* status, int nthreads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(or_nthreads(nthreads))
    for (long i = 0; i < n_kp; ++i) {
        or_keypoint kp;
        memcpy(&kp, kps4 + 4 * i, sizeof kp);
        int32_t ii = kp_image ? kp_image[i] : 0;
        uint8_t* o = out + (size_t)i * 1024;
        if (!kp_valid(&kp, ii, n_img, H, W)) {
            memset(o, 0, 1024);
            if (status) status[i] = 1;
            continue;
        }
        if (status) status[i] = 0;
        const uint8_t* img = images + (size_t)ii * (size_t)H * (size_t)pitch;
        float a, b;
        kp_frame(&kp, &a, &b);
        for (int v = 0; v < 32; ++v)
            for (int u = 0; u < 32; ++u) {
                long px, py;
                sample_point(kp.x, kp.y, a, b, u - 16, v - 16, &px, &py, NULL);
                px = clampl(px, 0, W - 1);
                py = clampl(py, 0, H - 1);
                o[v * 32 + u] = img[py * pitch + px];
            }
    }
}

/* SIFT descriptor of one normalised 32x32 patch ("the vector of real valued
 * features provided by SIFT"; "only describes a normalized 32x32 px image patch";
 * conventions R10 / S:373), float64:
 *  1. gx = P[y][min(x+1,31)] - P[y][max(x-1,0)], gy likewise with y pointing down
 *  2. m = sqrt(gx^2 + gy^2); theta = atan2(gy, gx) in [0, 2pi)
 *  3. w = exp(-((x-15.5)^2 + (y-15.5)^2) / (2*16^2))      (sigma = half the patch width)
 *  4. trilinear: cx = (x-3.5)/8, cy = (y-3.5)/8, co = theta/(pi/4); bin o centred at o*45deg
 *     hist[(j*4+i)*8 + (o mod 8)] += m*w*(1-|cx-i|)(1-|cy-j|)(1-|co-o|) for the 8 corners
 *     whose cell (j,i) lies in [0,4)^2
 *  5. v = h/|h|; v_i = min(v_i, clip); v = v/|v|; the zero histogram stays zero
 * `raw` (nullable) receives the un-normalised histogram. */
static void sift_one(const uint8_t* P, double clip, double* v, double* raw) {
    double h[128];
    memset(h, 0, sizeof h);
    for (int y = 0; y < 32; ++y)
        for (int x = 0; x < 32; ++x) {
            int xp = x + 1 > 31 ? 31 : x + 1, xm = x - 1 < 0 ? 0 : x - 1;
            int yp = y + 1 > 31 ? 31 : y + 1, ym = y - 1 < 0 ? 0 : y - 1;
            double gx = (double)P[y * 32 + xp] - (double)P[y * 32 + xm];
            double gy = (double)P[yp * 32 + x] - (double)P[ym * 32 + x];
            double m = sqrt(gx * gx + gy * gy);
            if (m == 0.0) continue;
            double th = atan2(gy, gx);
            if (th < 0.0) th += 2.0 * OR_PI;
            double w = exp(-(((double)x - 15.5) * ((double)x - 15.5) +
                             ((double)y - 15.5) * ((double)y - 15.5)) / (2.0 * 16.0 * 16.0));
            double cx = ((double)x - 3.5) / 8.0, cy = ((double)y - 3.5) / 8.0;
            double co = th / (OR_PI / 4.0);
            double i0 = floor(cx), j0 = floor(cy), o0 = floor(co);
            double fx = cx - i0, fy = cy - j0, fo = co - o0;
            for (int dj = 0; dj < 2; ++dj)
                for (int di = 0; di < 2; ++di)
                    for (int dor = 0; dor < 2; ++dor) {
                        int j = (int)j0 + dj, i = (int)i0 + di;
                        if (j < 0 || j > 3 || i < 0 || i > 3) continue;
                        int o = (((int)o0 + dor) % 8 + 8) % 8;
                        double wt = (dj ? fy : 1.0 - fy) * (di ? fx : 1.0 - fx) * (dor ? fo : 1.0 - fo);
                        h[(j * 4 + i) * 8 + o] += m * w * wt;
                    }
        }
    if (raw) memcpy(raw, h, sizeof h);
    double n2 = 0.0;
    for (int k = 0; k < 128; ++k) n2 += h[k] * h[k];
    if (n2 == 0.0) {
        memset(v, 0, 128 * sizeof(double));
        return;
    }
    double n = sqrt(n2);
    for (int k = 0; k < 128; ++k) {
        double t = h[k] / n;
        v[k] = t < clip ? t : clip;
    }
    n2 = 0.0;
    for (int k = 0; k < 128; ++k) n2 += v[k] * v[k];
    n = sqrt(n2);
    for (int k = 0; k < 128; ++k) v[k] /= n;
}

void or_sift(const uint8_t* patches, long n, double clip, double* out, double* raw, int nthreads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(or_nthreads(nthreads))
    for (long i = 0; i < n; ++i)
        sift_one(patches + (size_t)i * 1024, clip, out + (size_t)i * 128, raw ? raw + (size_t)i * 128 : NULL);
}

/* HashSIFT binarisation (D(x) = sgn(B [f(x)^T, 1]^T), B is N x 129 = [W | b],
 * S:411): p_k = sum_i W[k][i] v_i + b[k] in float64; bit_k = [p_k >= 0] (sgn(0) := +1,
 * R15 / S:436); packed LSB-first like BAD.  proj (nullable): the float64 p_k. */
void or_project(const double* sift, long n, const float* B, int N, uint8_t* out, double* proj,
                int nthreads) {
    const long row = (N + 7) / 8;
#pragma omp parallel for schedule(dynamic, 64) num_threads(or_nthreads(nthreads))
    for (long i = 0; i < n; ++i) {
        const double* v = sift + (size_t)i * 128;
        uint8_t* o = out + i * row;
        memset(o, 0, (size_t)row);
        for (int k = 0; k < N; ++k) {
            const float* Wk = B + (size_t)k * 129;
            double p = 0.0;
            for (int d = 0; d < 128; ++d) p += (double)Wk[d] * v[d];
            p += (double)Wk[128];
            if (proj) proj[(size_t)i * N + k] = p;
            if (p >= 0.0) o[k >> 3] |= (uint8_t)(1u << (k & 7));
        }
    }
}

/* Full HashSIFT on patches (configs[3]) = or_sift (clip 0.2) + or_project, fused per patch
 * so the CPU baseline does not materialise the 128-d vectors. */
void or_hashsift_patches(const uint8_t* patches, long n, const float* B, int N, uint8_t* out,
                         int nthreads) {
    const long row = (N + 7) / 8;
#pragma omp parallel for schedule(dynamic, 16) num_threads(or_nthreads(nthreads))
    for (long i = 0; i < n; ++i) {
        double v[128];
        sift_one(patches + (size_t)i * 1024, 0.2, v, NULL);
        or_project(v, 1, B, N, out + i * row, NULL, 1);
    }
}

/* ------------------------------------------------------------------------- */
/* NEXT-1 matcher oracle.  Hamming distance = number of differing
 * bits, counted bit by bit over the K bits ("number of differing bits"); pad bits
 * are zero by construction.  Brute force: for each query the train row with minimal distance,
 * ties -> lowest train index.  Pair p matches a rows [a_off[p], a_off[p+1]) against
 * b rows [b_off[p], b_off[p+1]); nn indices are relative to the pair's b block. */
static int hamming_bits(const uint32_t* x, const uint32_t* y, int K) {
    int d = 0;
    for (int k = 0; k < K; ++k) d += (int)(((x[k >> 5] ^ y[k >> 5]) >> (k & 31)) & 1u);
    return d;
}

void or_match(const uint32_t* a, const int64_t* a_off, const uint32_t* b, const int64_t* b_off, int n_pairs,
              int K, int32_t* nn, int32_t* dist, int nthreads) {
    const int words = K / 32;
    for (int p = 0; p < n_pairs; ++p) {
        const long a0 = (long)a_off[p], a1 = (long)a_off[p + 1], b0 = (long)b_off[p], b1 = (long)b_off[p + 1];
#pragma omp parallel for schedule(dynamic, 16) num_threads(or_nthreads(nthreads))
        for (long i = a0; i < a1; ++i) {
            int best = K + 1, bj = -1;
            for (long j = b0; j < b1; ++j) {
                int d = hamming_bits(a + (size_t)i * words, b + (size_t)j * words, K);
                if (d < best) { best = d; bj = (int)(j - b0); }   /* strict: lowest index on ties */
            }
            nn[i] = bj;
            if (dist) dist[i] = best;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* NEXT-3 variants.
 * (a) RootSIFT ("Hellinger distance ... RootSIFT"): v' = sqrt(v / sum v),
 *     the zero vector maps to zero.  Applied to a SIFT descriptor before the projection. */
void or_root_sift(const double* in, long n, double* out) {
    for (long i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = 0; k < 128; ++k) s += in[i * 128 + k];
        for (int k = 0; k < 128; ++k) out[i * 128 + k] = s > 0.0 ? sqrt(in[i * 128 + k] / s) : 0.0;
    }
}

/* (b) BAD with the box radius scaled by the keypoint scale (reading R27): r' = floor(r*s + 1/2)
 *     with r*s and the + 1/2 in fp32 (round half up); otherwise identical to or_bad_image
 *     (sample points R6, clamped boxes R5, exact compare R4). */
void or_bad_image_scaled(const uint8_t* images, long n_img, long H, long W, long pitch, const float* kps4,
                         const int32_t* kp_image, long n_kp, const int8_t* pairs, const uint8_t* radii,
                         const float* thr, int K, uint8_t* out, uint8_t* status, int nthreads) {
    const long row = (K + 7) / 8;
#pragma omp parallel for schedule(dynamic, 8) num_threads(or_nthreads(nthreads))
    for (long i = 0; i < n_kp; ++i) {
        or_keypoint kp;
        memcpy(&kp, kps4 + 4 * i, sizeof kp);
        int32_t ii = kp_image ? kp_image[i] : 0;
        uint8_t* o = out + i * row;
        memset(o, 0, (size_t)row);
        if (!kp_valid(&kp, ii, n_img, H, W)) {
            if (status) status[i] = 1;
            continue;
        }
        if (status) status[i] = 0;
        const uint8_t* img = images + (size_t)ii * (size_t)H * (size_t)pitch;
        float a, b;
        kp_frame(&kp, &a, &b);
        for (int k = 0; k < K; ++k) {
            long p1x, p1y, p2x, p2y;
            sample_point(kp.x, kp.y, a, b, pairs[4 * k + 0], pairs[4 * k + 1], &p1x, &p1y, NULL);
            sample_point(kp.x, kp.y, a, b, pairs[4 * k + 2], pairs[4 * k + 3], &p2x, &p2y, NULL);
            float rs = (float)radii[k] * kp.scale;
            int r = (int)floorf(rs + 0.5f);
            int64_t S1, A1, S2, A2;
            box_sum(img, H, W, pitch, p1x, p1y, r, &S1, &A1);
            box_sum(img, H, W, pitch, p2x, p2y, r, &S2, &A2);
            if (bad_bit(S1, A1, S2, A2, thr[k], NULL)) o[k >> 3] |= (uint8_t)(1u << (k & 7));
        }
    }
}

/* NEXT-2: bilinear patch normalisation (reading R28).  Patch pixel (u, v) samples the
 * image at X = x + (a*du - b*dv), Y = y + (b*du + a*dv) with du = u - 15.5, dv = v - 15.5 (the
 * crop square centred on the keypoint, side 32*scale, rotated by the angle), evaluated with
 * the R6 fp32 rule; x0 = floor(X), fx = X - x0 (both exact in fp32); the four neighbours are
 * clamped into the image (border replicate); the value
 *     v = (1-fy)*((1-fx)*I00 + fx*I01) + fy*((1-fx)*I10 + fx*I11)
 * is evaluated in fp32 in this order without FMA and rounded half up: p = floor(v + 1/2).
 * The quantised output is decided in fp32 on both sides (same rule as the GPU), so the
 * comparison is exact. */
void or_warp_bilinear(const uint8_t* images, long n_img, long H, long W, long pitch, const float* kps4,
                      const int32_t* kp_image, long n_kp, uint8_t* out, uint8_t* status, int nthreads) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(or_nthreads(nthreads))
    for (long i = 0; i < n_kp; ++i) {
        or_keypoint kp;
        memcpy(&kp, kps4 + 4 * i, sizeof kp);
        int32_t ii = kp_image ? kp_image[i] : 0;
        uint8_t* o = out + (size_t)i * 1024;
        if (!kp_valid(&kp, ii, n_img, H, W)) {
            memset(o, 0, 1024);
            if (status) status[i] = 1;
            continue;
        }
        if (status) status[i] = 0;
        const uint8_t* img = images + (size_t)ii * (size_t)H * (size_t)pitch;
        float a, b;
        kp_frame(&kp, &a, &b);
        for (int v = 0; v < 32; ++v)
            for (int u = 0; u < 32; ++u) {
                float du = (float)u - 15.5f, dv = (float)v - 15.5f;
                float t1 = a * du, t2 = b * dv, t3 = b * du, t4 = a * dv;
                float X = kp.x + (t1 - t2);
                float Y = kp.y + (t3 + t4);
                float fx0 = floorf(X), fy0 = floorf(Y);
                float fx = X - fx0, fy = Y - fy0;
                long x0 = (long)fx0, y0 = (long)fy0;
                long xa = clampl(x0, 0, W - 1), xb = clampl(x0 + 1, 0, W - 1);
                long ya = clampl(y0, 0, H - 1), yb = clampl(y0 + 1, 0, H - 1);
                float I00 = img[ya * pitch + xa], I01 = img[ya * pitch + xb];
                float I10 = img[yb * pitch + xa], I11 = img[yb * pitch + xb];
                float gx = 1.0f - fx, gy = 1.0f - fy;
                float top = gx * I00 + fx * I01;
                float bot = gx * I10 + fx * I11;
                float val = gy * top + fy * bot;
                long p = (long)floorf(val + 0.5f);
                o[v * 32 + u] = (uint8_t)clampl(p, 0, 255);
            }
    }
}

/* ------------------------------------------------------------------------- */
/* NEXT-4: one iteration of the BAD feature-selection hot loop (Algorithm 1 lines 4-12,
 * P:146-183) with Algorithm 2's integer-sort threshold search ("m = 511/0.1 =
 * 5110 possible values for theta").  Readings R29-R31:
 *  R29  Eq. 2 as written: per triplet  L_i(theta) = [tau - S_ap - h_a h_p + S_an + h_a h_n]_+
 *       with the prior similarities S^(t-1) as INTEGERS (sums of t-1 products of +-1 bits)
 *       and an integer margin tau, so every loss and loss change is an integer.
 *  R30  f(x) = mean(box1) - mean(box2) on the 32x32 patch at (16,16) with clamped
 *       boxes (R5); for a fixed candidate the clamped areas A1, A2 are patch-independent, so
 *       f = num/den with num = S1*A2 - S2*A1 and den = A1*A2 exactly.  Bucket
 *       b(f) = floor((f + 255) * 10), in [0, 5110], computed exactly in integers; h = +1 iff
 *       f <= theta, theta scanned over bucket upper edges: theta_b includes every
 *       value with bucket <= b.  theta_{-1} = -inf (all bits -1).
 *  R31  Events per triplet (Algorithm 2 lines 2-9) are taken at the DISTINCT feature values of
 *       the triplet's members, each carrying the exact jump L_i(v) - L_i(v-) (members with
 *       equal f cross together), so the sweep is exact at ties.  L* = min over b in
 *       {-1, 0..5110} of L(theta_b) (first minimum in sweep order, -inf first); a threshold
 *       realising it is theta* = -255 + (b*+1)/10 - 1e-6 (just below the bucket's upper edge;
 *       feature values are rationals with denominators <= 225^2, so the gap is >= 2e-6).
 * out_loss[j] = L*, out_bucket[j] = b* (-1 for theta = -inf). */
static int64_t trip_loss(int tau, int sap, int san, int ha, int hp, int hn) {
    int64_t v = (int64_t)tau - sap - ha * hp + san + ha * hn;
    return v > 0 ? v : 0;
}

void or_select_features(const uint8_t* patches, int M, const int32_t* trip, int N, const int32_t* sap,
                        const int32_t* san, int tau, const int8_t* cand, const uint8_t* radii, int J,
                        int64_t* out_loss, int32_t* out_bucket, int nthreads) {
    enum { NB = 5111 };
#pragma omp parallel for schedule(dynamic, 1) num_threads(or_nthreads(nthreads))
    for (int j = 0; j < J; ++j) {
        int64_t* num = (int64_t*)malloc(sizeof(int64_t) * (size_t)M);
        int32_t* bkt = (int32_t*)malloc(sizeof(int32_t) * (size_t)M);
        int64_t* hist = (int64_t*)calloc(NB, sizeof(int64_t));
        int64_t A1 = 0, A2 = 0;
        for (int m = 0; m < M; ++m) {
            int64_t S1, S2;
            box_sum(patches + (size_t)m * 1024, 32, 32, 32, 16 + cand[4 * j], 16 + cand[4 * j + 1], radii[j], &S1, &A1);
            box_sum(patches + (size_t)m * 1024, 32, 32, 32, 16 + cand[4 * j + 2], 16 + cand[4 * j + 3], radii[j], &S2,
                    &A2);
            num[m] = S1 * A2 - S2 * A1;
            /* b = floor((num/den + 255) * 10) = floor((10 num + 2550 den) / den), den > 0 */
            int64_t den = A1 * A2, q = 10 * num[m] + 2550 * den;
            int64_t b = q >= 0 ? q / den : -((-q + den - 1) / den);
            bkt[m] = (int32_t)b;
        }
        int64_t L0 = 0;
        for (int i = 0; i < N; ++i) {
            const int32_t idx[3] = {trip[3 * i], trip[3 * i + 1], trip[3 * i + 2]};
            L0 += trip_loss(tau, sap[i], san[i], -1, -1, -1);
            /* distinct values in increasing order; at each, the exact jump of L_i */
            for (int m = 0; m < 3; ++m) {
                int64_t v = num[idx[m]];
                int first = 1;  /* process each distinct value once: at its lowest member index */
                for (int q = 0; q < m; ++q)
                    if (num[idx[q]] == v) first = 0;
                if (!first) continue;
                int h_before[3], h_after[3];
                for (int q = 0; q < 3; ++q) {
                    h_before[q] = num[idx[q]] < v ? 1 : -1;   /* theta just below v */
                    h_after[q] = num[idx[q]] <= v ? 1 : -1;   /* theta = v (inclusive) */
                }
                int64_t d = trip_loss(tau, sap[i], san[i], h_after[0], h_after[1], h_after[2]) -
                            trip_loss(tau, sap[i], san[i], h_before[0], h_before[1], h_before[2]);
                hist[bkt[idx[m]]] += d;
            }
        }
        int64_t best = L0, acc = L0;
        int32_t bb = -1;
        for (int b = 0; b < NB; ++b) {
            acc += hist[b];
            if (acc < best) { best = acc; bb = b; }
        }
        out_loss[j] = best;
        out_bucket[j] = bb;
        free(num); free(bkt); free(hist);
    }
}

/* Pin helper: the loss of one candidate at an arbitrary real threshold, by definition
 * (h = +1 iff f <= theta, f = num/den exactly compared as num <= theta*den in long double). */
int64_t or_feature_loss_at(const uint8_t* patches, const int32_t* trip, int N, const int32_t* sap,
                           const int32_t* san, int tau, const int8_t* c4, int r, double theta) {
    int64_t L = 0;
    for (int i = 0; i < N; ++i) {
        int h[3];
        for (int q = 0; q < 3; ++q) {
            int64_t S1, S2, A1, A2;
            const uint8_t* P = patches + (size_t)trip[3 * i + q] * 1024;
            box_sum(P, 32, 32, 32, 16 + c4[0], 16 + c4[1], r, &S1, &A1);
            box_sum(P, 32, 32, 32, 16 + c4[2], 16 + c4[3], r, &S2, &A2);
            long double f = (long double)S1 / A1 - (long double)S2 / A2;
            h[q] = f <= theta ? 1 : -1;
        }
        L += trip_loss(tau, sap[i], san[i], h[0], h[1], h[2]);
    }
    return L;
}
