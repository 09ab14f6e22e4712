"""Seeded synthetic input generators — TEST / BENCH INFRASTRUCTURE.

This module is the ONLY code shared by the CUDA product path's tests and the CPU
oracle (DESIGN.md §3 "input recipe").  It holds none of the method's arithmetic
(no box sums, no gradients, no projections): only counter-based random numbers
and the integer-exact smoothed-noise recipe of BASELINE.json configs[0..4]
("seeded Gaussian-smoothed noise (sigma 2, values 0-255)").

Everything here is integer-exact so that the numpy implementation below and the
CUDA twin in ``synth/synth.cu`` produce bit-identical bytes (checked by a GPU
test).  Reading R18 of SURVEY.md §8(c), made integer:

  z(i, j)   = sum of the 4 low bytes of hash(seed, 1, unit, i, j) - 510
              (Irwin-Hall of 4 uniform bytes: mean 0, variance 21845)
  F(i, j)   = sum_{a,b=-6..6} w_a w_b z(i+a, j+b)      integer Gaussian, sigma 2
              w = round(256 exp(-k^2/8)), k = 0..6  -> 256,226,155,83,35,11,3
  pixel     = clamp(128 + round_half_up(F * G1 * gain_q / 2^42), 0, 255)
              G1 = round(48 * 2^32 / (sqrt(21845) * sum w^2))  (48 grey levels per std)
              gain_q = 1024 for images, U{512..2048} per patch (gain 0.5..2, configs[2])

The noise is defined on all integer (i, j) (negative too), so images and patches
have no border effects.  Keypoints / tests / W / b are host-generated arrays
handed to both sides unchanged.
"""
from __future__ import annotations

import math
import numpy as np

# ----------------------------------------------------------------------------
# counter-based hash (splitmix64 finaliser chained over the counter words)
# ----------------------------------------------------------------------------
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)

STREAM_PIXELS = 1
STREAM_KEYPOINTS = 2
STREAM_TESTS = 3
STREAM_W = 4
STREAM_B = 5
STREAM_GAIN = 6


def _mix64(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint64(30))
    x = x * _M1
    x = x ^ (x >> np.uint64(27))
    x = x * _M2
    x = x ^ (x >> np.uint64(31))
    return x


def hash64(seed: int, stream: int, a, b=0, c=0) -> np.ndarray:
    """hash(seed, stream, a, b, c) -> uint64.  a, b, c: int64-compatible arrays
    (negative values wrap mod 2^64, identically in synth.cu)."""
    with np.errstate(over="ignore"):
        a = np.asarray(a, dtype=np.int64).astype(np.uint64)
        b = np.asarray(b, dtype=np.int64).astype(np.uint64)
        c = np.asarray(c, dtype=np.int64).astype(np.uint64)
        k = np.uint64((seed * 0x100000001B3 + stream * 0x9E37) & 0xFFFFFFFFFFFFFFFF)
        h = _mix64(k + _G)
        h = _mix64(h ^ (a * _G + np.uint64(1)))
        h = _mix64(h ^ (b * _M1 + np.uint64(2)))
        h = _mix64(h ^ (c * _M2 + np.uint64(3)))
    return h


def u24(h: np.ndarray) -> np.ndarray:
    """uniform in [0, 1) with 24-bit resolution, float64."""
    return (h >> np.uint64(40)).astype(np.float64) * (1.0 / 16777216.0)


# ----------------------------------------------------------------------------
# smoothed-noise recipe (integer exact)
# ----------------------------------------------------------------------------
BLUR_RADIUS = 6
BLUR_W = np.array([3, 11, 35, 83, 155, 226, 256, 226, 155, 83, 35, 11, 3], dtype=np.int64)
assert all(BLUR_W[6 + k] == round(256 * math.exp(-k * k / 8.0)) for k in range(7))
SUM_W2 = int((BLUR_W * BLUR_W).sum())          # 232226
NOISE_VAR = 4 * (256 * 256 - 1) // 12          # 21845
G1 = int(round(48.0 * 2.0 ** 32 / (math.sqrt(NOISE_VAR) * SUM_W2)))
SHIFT = 42                                      # 32 (G1) + 10 (gain_q / 1024)
GAIN_ONE = 1024


def _noise(seed: int, units: np.ndarray, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    h = hash64(seed, STREAM_PIXELS, units[:, None, None], rows[None, :, None], cols[None, None, :])
    m = np.uint64(0xFF)
    z = (h & m) + ((h >> np.uint64(8)) & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(24)) & m)
    return z.astype(np.int64) - 510


def _fields(seed: int, units, H: int, W: int) -> np.ndarray:
    """integer smoothed-noise fields (n, H, W) for the given unit indices."""
    R = BLUR_RADIUS
    units = np.asarray(units, dtype=np.int64).reshape(-1)
    rows = np.arange(-R, H + R, dtype=np.int64)
    cols = np.arange(-R, W + R, dtype=np.int64)
    z = _noise(seed, units, rows, cols)                    # (n, H+2R, W+2R)
    t = np.zeros((len(units), H + 2 * R, W), dtype=np.int64)
    for k in range(2 * R + 1):
        t += BLUR_W[k] * z[:, :, k:k + W]
    f = np.zeros((len(units), H, W), dtype=np.int64)
    for k in range(2 * R + 1):
        f += BLUR_W[k] * t[:, k:k + H, :]
    return f


def _quantise(f: np.ndarray, gain_q) -> np.ndarray:
    g = np.asarray(gain_q, dtype=np.int64) * np.int64(G1)
    if g.ndim:
        g = g.reshape((-1,) + (1,) * (f.ndim - 1))
    v = (f * g + np.int64(1 << (SHIFT - 1))) >> np.int64(SHIFT)
    return np.clip(v + 128, 0, 255).astype(np.uint8)


def image(seed: int, index: int, H: int, W: int) -> np.ndarray:
    """uint8 HxW smoothed-noise image number `index` of stream `seed`."""
    return _quantise(_fields(seed, [index], H, W)[0], GAIN_ONE)


def images(seed: int, indices, H: int, W: int) -> np.ndarray:
    idx = list(indices)
    out = np.empty((len(idx), H, W), dtype=np.uint8)
    for n, i in enumerate(idx):
        out[n] = image(seed, i, H, W)
    return out


def patch_gain(seed: int, indices) -> np.ndarray:
    """per-patch contrast gain numerator in {512..2048} (gain = q/1024 in [0.5, 2])."""
    h = hash64(seed, STREAM_GAIN, np.asarray(indices, dtype=np.int64))
    return (512 + (h % np.uint64(1537))).astype(np.int64)


def patches(seed: int, indices, chunk: int = 4096) -> np.ndarray:
    """uint8 (n, 32, 32) patches; patch p is its own noise field (unit = p) with gain q_p/1024."""
    idx = np.asarray(list(indices) if not isinstance(indices, np.ndarray) else indices,
                     dtype=np.int64).reshape(-1)
    out = np.empty((len(idx), 32, 32), dtype=np.uint8)
    for s in range(0, len(idx), chunk):
        u = idx[s:s + chunk]
        out[s:s + chunk] = _quantise(_fields(seed, u, 32, 32), patch_gain(seed, u))
    return out


# ----------------------------------------------------------------------------
# keypoints (BASELINE configs[0], [1], [4])
# ----------------------------------------------------------------------------
KP_DTYPE = np.dtype([("x", np.float32), ("y", np.float32), ("angle", np.float32), ("scale", np.float32)])


def keypoints_grid(seed: int, image_index: int, n: int, H: int, W: int, margin: int = 24) -> np.ndarray:
    """configs[0]: integer positions uniform in [m, W-1-m] x [m, H-1-m], scale 1, angle 0."""
    k = np.arange(n, dtype=np.int64)
    hx = hash64(seed, STREAM_KEYPOINTS, image_index, k, 0)
    hy = hash64(seed, STREAM_KEYPOINTS, image_index, k, 1)
    kp = np.zeros(n, dtype=KP_DTYPE)
    kp["x"] = (margin + (hx % np.uint64(W - 2 * margin))).astype(np.float32)
    kp["y"] = (margin + (hy % np.uint64(H - 2 * margin))).astype(np.float32)
    kp["scale"] = 1.0
    kp["angle"] = 0.0
    return kp


def keypoints_random(seed: int, image_index: int, n: int, H: int, W: int, margin: int,
                     scale_max: float) -> np.ndarray:
    """configs[1]/[4]: float positions uniform in [m, W-1-m] x [m, H-1-m], scale log-uniform
    in [1, scale_max], angle uniform in [0, 2pi)."""
    k = np.arange(n, dtype=np.int64)
    u = [u24(hash64(seed, STREAM_KEYPOINTS, image_index, k, j)) for j in range(4)]
    kp = np.zeros(n, dtype=KP_DTYPE)
    kp["x"] = (margin + u[0] * (W - 1 - 2 * margin)).astype(np.float32)
    kp["y"] = (margin + u[1] * (H - 1 - 2 * margin)).astype(np.float32)
    kp["scale"] = np.exp(u[2] * math.log(scale_max)).astype(np.float32)
    kp["angle"] = (u[3] * (2.0 * math.pi)).astype(np.float32)
    return kp


def keypoints_as_array(kp: np.ndarray) -> np.ndarray:
    """structured -> float32 (n, 4) [x, y, angle, scale] (the bd_keypoint layout)."""
    return np.stack([kp["x"], kp["y"], kp["angle"], kp["scale"]], axis=1).astype(np.float32)


# ----------------------------------------------------------------------------
# BAD test tables (configs[0]: "p1 and p2 uniform in a 32x32 patch centred on the
# keypoint, box radius r uniform in {1..5}, threshold uniform in [-20,20]")
# ----------------------------------------------------------------------------
def bad_tests(seed: int, K: int, rmin: int = 1, rmax: int = 5, tmax: float = 20.0):
    """-> pairs int8 (K,4) [dx1,dy1,dx2,dy2] in [-16,15], radii uint8 (K,), thresholds f32 (K,)."""
    pairs = np.zeros((K, 4), dtype=np.int8)
    radii = np.zeros(K, dtype=np.uint8)
    thr = np.zeros(K, dtype=np.float32)
    for k in range(K):
        t = 0
        while True:
            h = [int(hash64(seed, STREAM_TESTS, k, t, j)) for j in range(4)]
            d = [(hh % 32) - 16 for hh in h]
            if (d[0], d[1]) != (d[2], d[3]):
                break
            t += 1
        pairs[k] = d
        radii[k] = rmin + int(hash64(seed, STREAM_TESTS, k, 1 << 20, 4)) % (rmax - rmin + 1)
        u = float(u24(hash64(seed, STREAM_TESTS, k, 1 << 20, 5)))
        thr[k] = np.float32(-tmax + 2.0 * tmax * u)
    return pairs, radii, thr


def hashsift_matrix(seed: int, N: int, dim: int = 128) -> np.ndarray:
    """configs[3]: W ~ N(0, 1/128) (N x 128), b ~ N(0, 0.01) (variances)
    -> float32 B = [W | b] of shape (N, 129)."""
    rw = np.random.default_rng(np.random.PCG64([seed, STREAM_W]))
    rb = np.random.default_rng(np.random.PCG64([seed, STREAM_B]))
    W = rw.standard_normal((N, dim)) * math.sqrt(1.0 / 128.0)
    b = rb.standard_normal(N) * 0.1
    return np.concatenate([W, b[:, None]], axis=1).astype(np.float32)


# ----------------------------------------------------------------------------
# the five BASELINE.json workloads
# ----------------------------------------------------------------------------
CONFIGS = {
    0: dict(name="c0: BAD-256, 1x640x480 image, 500 kp (scale 1, angle 0)", kind="bad_image",
            n_images=1, H=480, W=640, kp_per_image=500, K=256, kp="grid", margin=24),
    1: dict(name="c1: BAD-512, 64x1920x1080 images, 2000 kp/img (scale logU[1,4], angle U)",
            kind="bad_image", n_images=64, H=1080, W=1920, kp_per_image=2000, K=512, kp="random",
            margin=98, scale_max=4.0),
    2: dict(name="c2: BAD-256, 4M 32x32 patches", kind="bad_patch", n_patches=4_000_000, K=256),
    3: dict(name="c3: HashSIFT-256, 1M 32x32 patches", kind="hashsift_patch", n_patches=1_000_000, N=256),
    4: dict(name="c4: BAD-512 + HashSIFT-256 on NN-warped patches, 8192x3840x2160, 4000 kp/img",
            kind="warped", n_images=8192, H=2160, W=3840, kp_per_image=4000, K=512, N=256,
            kp="random", margin=138, scale_max=6.0),
}


def config_keypoints(cfg_id: int, image_index: int, n: int | None = None) -> np.ndarray:
    c = CONFIGS[cfg_id]
    n = c["kp_per_image"] if n is None else n
    if c["kp"] == "grid":
        return keypoints_grid(cfg_id, image_index, n, c["H"], c["W"], c["margin"])
    return keypoints_random(cfg_id, image_index, n, c["H"], c["W"], c["margin"], c["scale_max"])


def keypoints_random_batch(seed: int, image_indices, n: int, H: int, W: int, margin: int,
                           scale_max: float) -> np.ndarray:
    """keypoints_random for many images at once -> float32 (len(images) * n, 4), image-major.
    Identical values to concatenating keypoints_random(seed, i, ...) over the images."""
    imgs = np.asarray(image_indices, dtype=np.int64).reshape(-1, 1)
    k = np.arange(n, dtype=np.int64).reshape(1, -1)
    out = np.empty((imgs.shape[0] * n, 4), dtype=np.float32)
    u = u24(hash64(seed, STREAM_KEYPOINTS, imgs, k, 0)).reshape(-1)
    out[:, 0] = (margin + u * (W - 1 - 2 * margin)).astype(np.float32)
    u = u24(hash64(seed, STREAM_KEYPOINTS, imgs, k, 1)).reshape(-1)
    out[:, 1] = (margin + u * (H - 1 - 2 * margin)).astype(np.float32)
    u = u24(hash64(seed, STREAM_KEYPOINTS, imgs, k, 3)).reshape(-1)
    out[:, 2] = (u * (2.0 * math.pi)).astype(np.float32)
    u = u24(hash64(seed, STREAM_KEYPOINTS, imgs, k, 2)).reshape(-1)
    out[:, 3] = np.exp(u * math.log(scale_max)).astype(np.float32)
    return out
