"""Pins for the nearest-neighbour warp oracle (or_warp_nn; configs[4], R20).

Closed forms: identity keypoint = crop ("identity geometry"), angle (float)(pi/2) =
90-degree rotated crop, scale 2 = stride-2 subsampled crop, border replication,
invalid keypoints -> zero patch + status 1.
"""
import math

import numpy as np

import oracle
import synth


def test_identity_is_crop():
    img = synth.image(31, 0, 100, 120)
    kp = np.array([[40, 50, 0, 1], [16, 16, 0, 1], [103, 83, 0, 1]], np.float32)
    P = oracle.warp_nn(img, kp)
    for p, (x, y, _, _) in zip(P, kp.astype(int)):
        assert (p == img[y - 16:y + 16, x - 16:x + 16]).all()


def test_rot90_is_rotated_crop():
    img = synth.image(32, 0, 100, 100)
    x, y = 50, 45
    P = oracle.warp_nn(img, np.array([[x, y, np.float32(math.pi / 2), 1]], np.float32))[0]
    # patch pixel (u, v) <- image at (x - (v - 16), y + (u - 16))
    v, u = np.mgrid[0:32, 0:32]
    assert (P == img[y + (u - 16), x - (v - 16)]).all()


def test_scale_two_is_subsampled():
    img = synth.image(33, 0, 120, 120)
    x, y = 60, 61
    P = oracle.warp_nn(img, np.array([[x, y, 0, 2]], np.float32))[0]
    assert (P == img[y - 32:y + 32:2, x - 32:x + 32:2]).all()


def test_half_pixel_rounds_up():
    img = synth.image(34, 0, 80, 80)
    P = oracle.warp_nn(img, np.array([[40.5, 39.5, 0, 1]], np.float32))[0]
    # floor(X + 0.5): 40.5 + d -> 41 + d ; 39.5 + d -> 40 + d
    assert (P == img[40 - 16:40 + 16, 41 - 16:41 + 16]).all()


def test_border_replicate_and_invalid():
    img = synth.image(35, 0, 40, 50)
    kp = np.array([[0, 0, 0, 1], [49, 39, 0, 1], [-1, 3, 0, 1], [3, 3, 0, -1]], np.float32)
    P, st = oracle.warp_nn(img, kp, want_status=True)
    assert list(st) == [0, 0, 1, 1]
    v, u = np.mgrid[0:32, 0:32]
    assert (P[0] == img[np.clip(v - 16, 0, 39), np.clip(u - 16, 0, 49)]).all()
    assert (P[1] == img[np.clip(39 + v - 16, 0, 39), np.clip(49 + u - 16, 0, 49)]).all()
    assert (P[2] == 0).all() and (P[3] == 0).all()
