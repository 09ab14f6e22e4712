"""CPU oracle for the BAD / HashSIFT extraction path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2108_08380_b200`` never imports it, and this package imports nothing from
the product (the two share only the input generators in ``synth/``).

The arithmetic lives in ``bindesc_oracle.c`` (plain C, float64, brute-force box sums,
direct-loop SIFT); this module only builds it with gcc and marshals numpy arrays.
Parity status: every entry point is pinned by ``tests/test_oracle_*.py``; the SIFT
conventions are pinned by closed forms/invariants only (the paper prints no SIFT
values — DESIGN.md §4).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bindesc_oracle.c")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
          "-Wall", "-Wno-unknown-pragmas"]
# BINDESC_ORACLE_SANITIZE=1: a separate AddressSanitizer + UndefinedBehaviorSanitizer build of the
# same source (SURVEY §5 "host -fsanitize=address,undefined for the oracle"); the Python process
# must preload the runtime: tools/oracle_sanitize.sh
_SAN = os.environ.get("BINDESC_ORACLE_SANITIZE") == "1"
_LIB = os.path.join(_HERE, "liboracle_san.so" if _SAN else "liboracle.so")
if _SAN:
    CFLAGS = CFLAGS + ["-fsanitize=address,undefined", "-fno-sanitize-recover=undefined", "-fno-omit-frame-pointer",
                       "-g"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        L = ctypes.c_long
        I = ctypes.c_int
        D = ctypes.c_double
        _lib.or_bad_image.argtypes = [P, L, L, L, L, P, P, L, P, P, P, I, P, P, P, P, I]
        _lib.or_bad_patches.argtypes = [P, L, P, P, P, I, P, P, I]
        _lib.or_warp_nn.argtypes = [P, L, L, L, L, P, P, L, P, P, I]
        _lib.or_sift.argtypes = [P, L, D, P, P, I]
        _lib.or_project.argtypes = [P, L, P, I, P, P, I]
        _lib.or_hashsift_patches.argtypes = [P, L, P, I, P, I]
        _lib.or_max_threads.restype = I
        _lib.or_match.argtypes = [P, P, P, P, I, I, P, P, I]
        _lib.or_root_sift.argtypes = [P, L, P]
        _lib.or_bad_image_scaled.argtypes = [P, L, L, L, L, P, P, L, P, P, P, I, P, P, I]
        _lib.or_warp_bilinear.argtypes = [P, L, L, L, L, P, P, L, P, P, I]
        _lib.or_select_features.argtypes = [P, I, P, I, P, P, I, P, P, I, P, P, I]
        _lib.or_feature_loss_at.argtypes = [P, P, I, P, P, I, P, I, D]
        _lib.or_feature_loss_at.restype = ctypes.c_int64
        _lib.or_fragile_round.argtypes = [D]
        _lib.or_fragile_round.restype = I
        _lib.or_kp_frame.argtypes = [P, P]
        _lib.or_kp_frame.restype = I
    return _lib


def fragile_round(c: float) -> bool:
    """R6 test hook: is the float64 coefficient c within 4 float64-ulp of an fp32 rounding
    boundary (the midpoint between two adjacent fp32 values)?"""
    return bool(lib().or_fragile_round(float(c)))


def kp_frame(kp):
    """R6 test hook: (a, b, fragile) of one keypoint [x, y, angle, scale] as or_bad_image uses it."""
    k = _c(kp, np.float32).reshape(4)
    ab = np.zeros(2, np.float32)
    fr = lib().or_kp_frame(_p(k), _p(ab))
    return float(ab[0]), float(ab[1]), bool(fr)


def max_threads() -> int:
    return int(lib().or_max_threads())


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def bad_image(images, kps, pairs, radii, thr, kp_image=None, nthreads=0, want_aux=False):
    """images: uint8 (n, H, W); kps: float32 (m, 4) [x, y, angle, scale]; pairs int8 (K,4);
    radii uint8 (K,); thr float32 (K,).  -> uint8 (m, ceil(K/8)) [, status, fragile, ties]."""
    images = _c(images, np.uint8)
    if images.ndim == 2:
        images = images[None]
    n, H, W = images.shape
    kps = _c(kps, np.float32).reshape(-1, 4)
    m = kps.shape[0]
    pairs, radii, thr = _c(pairs, np.int8), _c(radii, np.uint8), _c(thr, np.float32)
    K = len(radii)
    kpi = None if kp_image is None else _c(kp_image, np.int32)
    out = np.zeros((m, (K + 7) // 8), dtype=np.uint8)
    status = np.zeros(m, dtype=np.uint8)
    fragile = np.zeros(m, dtype=np.uint8)
    ties = np.zeros(m, dtype=np.int32)
    lib().or_bad_image(_p(images), n, H, W, W, _p(kps), _p(kpi), m, _p(pairs), _p(radii), _p(thr), K,
                       _p(out), _p(status), _p(fragile), _p(ties), nthreads)
    if want_aux:
        return out, status, fragile, ties
    return out


def bad_patches(patches, pairs, radii, thr, nthreads=0, want_ties=False):
    patches = _c(patches, np.uint8).reshape(-1, 32, 32)
    pairs, radii, thr = _c(pairs, np.int8), _c(radii, np.uint8), _c(thr, np.float32)
    K = len(radii)
    out = np.zeros((patches.shape[0], (K + 7) // 8), dtype=np.uint8)
    ties = np.zeros(patches.shape[0], dtype=np.int32)
    lib().or_bad_patches(_p(patches), patches.shape[0], _p(pairs), _p(radii), _p(thr), K, _p(out),
                         _p(ties), nthreads)
    return (out, ties) if want_ties else out


def warp_nn(images, kps, kp_image=None, nthreads=0, want_status=False):
    images = _c(images, np.uint8)
    if images.ndim == 2:
        images = images[None]
    n, H, W = images.shape
    kps = _c(kps, np.float32).reshape(-1, 4)
    m = kps.shape[0]
    kpi = None if kp_image is None else _c(kp_image, np.int32)
    out = np.zeros((m, 32, 32), dtype=np.uint8)
    status = np.zeros(m, dtype=np.uint8)
    lib().or_warp_nn(_p(images), n, H, W, W, _p(kps), _p(kpi), m, _p(out), _p(status), nthreads)
    return (out, status) if want_status else out


def sift(patches, clip=0.2, nthreads=0, want_raw=False):
    patches = _c(patches, np.uint8).reshape(-1, 32, 32)
    n = patches.shape[0]
    out = np.zeros((n, 128), dtype=np.float64)
    raw = np.zeros((n, 128), dtype=np.float64) if want_raw else None
    lib().or_sift(_p(patches), n, float(clip), _p(out), _p(raw), nthreads)
    return (out, raw) if want_raw else out


def project(sift_vecs, B, nthreads=0, want_proj=False):
    v = _c(sift_vecs, np.float64).reshape(-1, 128)
    B = _c(B, np.float32)
    N = B.shape[0]
    assert B.shape[1] == 129
    out = np.zeros((v.shape[0], (N + 7) // 8), dtype=np.uint8)
    proj = np.zeros((v.shape[0], N), dtype=np.float64) if want_proj else None
    lib().or_project(_p(v), v.shape[0], _p(B), N, _p(out), _p(proj), nthreads)
    return (out, proj) if want_proj else out


def hashsift_patches(patches, B, nthreads=0):
    patches = _c(patches, np.uint8).reshape(-1, 32, 32)
    B = _c(B, np.float32)
    N = B.shape[0]
    out = np.zeros((patches.shape[0], (N + 7) // 8), dtype=np.uint8)
    lib().or_hashsift_patches(_p(patches), patches.shape[0], _p(B), N, _p(out), nthreads)
    return out


def match(a, a_off, b, b_off, K, nthreads=0):
    """NEXT-1 brute-force Hamming NN: a, b uint32 (rows, K/32); a_off, b_off int64
    (n_pairs + 1).  -> (nn int32 (n_a,) pair-relative, dist int32 (n_a,))."""
    a = _c(a, np.uint32)
    b = _c(b, np.uint32)
    a_off = _c(a_off, np.int64)
    b_off = _c(b_off, np.int64)
    n_a = int(a_off[-1])
    nn = np.zeros(n_a, dtype=np.int32)
    dist = np.zeros(n_a, dtype=np.int32)
    lib().or_match(_p(a), _p(a_off), _p(b), _p(b_off), len(a_off) - 1, K, _p(nn), _p(dist), nthreads)
    return nn, dist


def mutual(nn_ab, nn_ba, a_off, b_off):
    """pair (i, j) is mutual iff j = NN(i) and i = NN(j) (pair-relative indices)."""
    out = np.zeros(len(nn_ab), dtype=np.uint8)
    for p in range(len(a_off) - 1):
        for i in range(a_off[p], a_off[p + 1]):
            out[i] = nn_ba[b_off[p] + nn_ab[i]] == i - a_off[p]
    return out


def root_sift(v):
    """NEXT-3 RootSIFT: sqrt(v / sum(v)); zero -> zero."""
    v = _c(v, np.float64).reshape(-1, 128)
    out = np.zeros_like(v)
    lib().or_root_sift(_p(v), v.shape[0], _p(out))
    return out


def bad_image_scaled(images, kps, pairs, radii, thr, kp_image=None, nthreads=0, want_status=False):
    """NEXT-3 BAD on images with box radius floor(r*scale + 1/2) (reading R27)."""
    images = _c(images, np.uint8)
    if images.ndim == 2:
        images = images[None]
    n, H, W = images.shape
    kps = _c(kps, np.float32).reshape(-1, 4)
    m = kps.shape[0]
    pairs, radii, thr = _c(pairs, np.int8), _c(radii, np.uint8), _c(thr, np.float32)
    K = len(radii)
    kpi = None if kp_image is None else _c(kp_image, np.int32)
    out = np.zeros((m, (K + 7) // 8), dtype=np.uint8)
    status = np.zeros(m, dtype=np.uint8)
    lib().or_bad_image_scaled(_p(images), n, H, W, W, _p(kps), _p(kpi), m, _p(pairs), _p(radii), _p(thr), K,
                              _p(out), _p(status), nthreads)
    return (out, status) if want_status else out


def warp_bilinear(images, kps, kp_image=None, nthreads=0, want_status=False):
    """NEXT-2 bilinear 32x32 patch (reading R28), border replicate, round half up."""
    images = _c(images, np.uint8)
    if images.ndim == 2:
        images = images[None]
    n, H, W = images.shape
    kps = _c(kps, np.float32).reshape(-1, 4)
    m = kps.shape[0]
    kpi = None if kp_image is None else _c(kp_image, np.int32)
    out = np.zeros((m, 32, 32), dtype=np.uint8)
    status = np.zeros(m, dtype=np.uint8)
    lib().or_warp_bilinear(_p(images), n, H, W, W, _p(kps), _p(kpi), m, _p(out), _p(status), nthreads)
    return (out, status) if want_status else out


def select_features(patches, triplets, s_ap, s_an, tau, cand_pairs, cand_radii, nthreads=0):
    """NEXT-4 hot loop (Alg. 1 lines 4-12 + Alg. 2 integer-sort, readings R29-R31):
    -> (loss int64 (J,), bucket int32 (J,), -1 = theta -inf)."""
    patches = _c(patches, np.uint8).reshape(-1, 32, 32)
    tr = _c(triplets, np.int32).reshape(-1, 3)
    sap, san = _c(s_ap, np.int32), _c(s_an, np.int32)
    cp, cr = _c(cand_pairs, np.int8).reshape(-1, 4), _c(cand_radii, np.uint8)
    J = len(cr)
    loss = np.zeros(J, np.int64)
    bucket = np.zeros(J, np.int32)
    lib().or_select_features(_p(patches), patches.shape[0], _p(tr), tr.shape[0], _p(sap), _p(san), int(tau),
                             _p(cp), _p(cr), J, _p(loss), _p(bucket), nthreads)
    return loss, bucket


def feature_loss_at(patches, triplets, s_ap, s_an, tau, pair4, r, theta):
    """L(theta) of one candidate by definition (pin helper)."""
    patches = _c(patches, np.uint8).reshape(-1, 32, 32)
    tr = _c(triplets, np.int32).reshape(-1, 3)
    sap, san = _c(s_ap, np.int32), _c(s_an, np.int32)
    c4 = _c(pair4, np.int8).reshape(4)
    return int(lib().or_feature_loss_at(_p(patches), _p(tr), tr.shape[0], _p(sap), _p(san), int(tau), _p(c4),
                                        int(r), float(theta)))


def bucket_theta(b):
    """R31: a threshold realising bucket b's sweep loss: just below the bucket's upper edge
    -255 + (b+1)/10 (every feature value is a rational num/den with den <= 225^2, so the gap
    to the edge is >= 1/(10*50625) = 2e-6 > 1e-6).  b = -1 -> -inf."""
    return -np.inf if b < 0 else -255.0 + (b + 1) / 10.0 - 1e-6
