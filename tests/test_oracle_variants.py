"""Pins for the NEXT-2 / NEXT-3 oracle variants.

* RootSIFT: zero -> zero, one-hot -> one-hot, random -> sqrt(v / sum v)
  computed with numpy, unit L2 norm.
* BAD with scaled box radius (reading R27): scale 1 equals or_bad_image; an integer scale-2
  keypoint at angle 0 equals or_bad_image with the radii doubled and the keypoint scale 2
  (same sample points, box radius 2r); hand example on the ramp image.
* Bilinear warp (reading R28): identity geometry reproduces the crop exactly
  (S:68); a constant image gives a constant patch at any angle; a half-pixel shift
  gives the rounded-half-up mean of neighbours (closed form); rotation by (float)(pi/2) gives
  the rot90 crop; border replicate."""
import math

import numpy as np

import oracle
import synth


def test_root_sift_closed_forms():
    z = np.zeros((1, 128))
    assert (oracle.root_sift(z) == 0).all()
    e = np.zeros((1, 128))
    e[0, 17] = 0.37
    r = oracle.root_sift(e)
    assert r[0, 17] == 1.0 and np.count_nonzero(r) == 1
    rng = np.random.default_rng(0)
    v = rng.random((20, 128))
    r = oracle.root_sift(v)
    np.testing.assert_allclose(r, np.sqrt(v / v.sum(1, keepdims=True)), rtol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(r, axis=1), 1.0, rtol=1e-12)


def test_bad_scaled_radius_reductions():
    img = synth.images(31, range(2), 90, 120)
    kp = synth.keypoints_as_array(synth.keypoints_random(31, 0, 300, 90, 120, 40, 1.0))
    kp[:, 3] = 1.0
    kpi = np.zeros(len(kp), np.int32)
    pairs, radii, thr = synth.bad_tests(31, 64, rmin=1, rmax=3)
    assert (oracle.bad_image_scaled(img, kp, pairs, radii, thr, kp_image=kpi) ==
            oracle.bad_image(img, kp, pairs, radii, thr, kp_image=kpi)).all()
    # integer scale 2, angle 0: r' = 2r
    kp2 = kp.copy()
    kp2[:, :2] = np.round(kp2[:, :2])
    kp2[:, 2] = 0.0
    kp2[:, 3] = 2.0
    r2 = (2 * radii).astype(np.uint8)
    assert (oracle.bad_image_scaled(img, kp2, pairs, radii, thr, kp_image=kpi) ==
            oracle.bad_image(img, kp2, pairs, r2, thr, kp_image=kpi)).all()


def test_bad_scaled_radius_ramp():
    # ramp I(y,x) = 16x + 2y + 10 on 16x16; kp (8,8), scale 2: offsets (+1,0) vs (-1,0) -> points
    # (10,8), (6,8); r = 1 -> r' = 2: unclamped 5x5 boxes, means I(8,10) = 186, I(8,6) = 122 -> f = 64
    y, x = np.mgrid[0:16, 0:16]
    img = (16 * x + 2 * y + 10).astype(np.uint8)
    kp = np.array([[8, 8, 0, 2]], np.float32)
    pairs = np.array([[1, 0, -1, 0]], np.int8)
    for th, bit in ((64.0, 1), (63.9, 0)):
        b = oracle.bad_image_scaled(img, kp, pairs, np.array([1], np.uint8), np.array([th], np.float32))
        assert (b[0, 0] & 1) == bit


def _img(H=40, W=48, seed=5):
    return np.random.default_rng(seed).integers(0, 256, size=(H, W), dtype=np.uint8)


def test_bilinear_identity_and_constant():
    I = _img(32, 32)
    P = oracle.warp_bilinear(I, np.array([[15.5, 15.5, 0.0, 1.0]], np.float32))
    assert (P[0] == I).all()  # S:68 identity resample, exact here
    C = np.full((40, 50), 77, np.uint8)
    kp = np.array([[20, 20, a, s] for a in (0.0, 1.0, math.pi, 4.0) for s in (0.7, 1.0, 2.5)], np.float32)
    assert (oracle.warp_bilinear(C, kp) == 77).all()


def test_bilinear_half_pixel_and_rot90():
    I = _img(32, 33)
    P = oracle.warp_bilinear(I, np.array([[16.0, 15.5, 0.0, 1.0]], np.float32))[0]
    ref = np.floor((I[:, :32].astype(np.float64) + I[:, 1:33]) / 2 + 0.5)  # fx = 1/2
    assert (P == ref).all()
    I = _img(32, 32, 6)
    P = oracle.warp_bilinear(I, np.array([[15.5, 15.5, np.float32(math.pi / 2), 1.0]], np.float32))[0]
    # patch (u, v) samples (x, y) = (15.5 - (v - 15.5), 15.5 + (u - 15.5)) = (31 - v, u)
    assert (P == I[np.arange(32)[None, :], 31 - np.arange(32)[:, None]]).all()


def test_bilinear_border_replicate_and_invalid():
    I = _img(20, 20, 7)
    P, st = oracle.warp_bilinear(I, np.array([[0, 0, 0, 1], [3, 3, 0, -1]], np.float32), want_status=True)
    assert (P[0, :16, :16] == I[0, 0]).all()      # everything up-left of the corner is pixel (0, 0)
    assert st.tolist() == [0, 1] and (P[1] == 0).all()
