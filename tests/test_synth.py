"""Host checks of the seeded input generators (synth/): determinism, the recipe's
statistics (BASELINE configs: values 0-255, sigma-2 smoothing), ranges of keypoints,
test tables and hash matrices.  The CUDA twin is compared byte for byte in
tests/test_gpu_synth.py."""
import math

import numpy as np

import synth


def test_image_stats_and_determinism():
    a = synth.image(0, 0, 480, 640)
    assert (a == synth.image(0, 0, 480, 640)).all()
    assert not (a == synth.image(0, 1, 480, 640)).all()
    assert abs(a.mean() - 128) < 3 and abs(a.std() - 48) < 3
    assert a.min() == 0 and a.max() == 255
    # smoothness: neighbouring pixels are strongly correlated (sigma 2 blur)
    c = np.corrcoef(a[:, :-1].ravel().astype(float), a[:, 1:].ravel().astype(float))[0, 1]
    assert c > 0.9


def test_image_crop_consistency():
    # images are windows of one infinite field per unit: generating at a different size
    # gives the same top-left pixels (no border effects)
    a = synth.image(1, 3, 64, 80)
    b = synth.image(1, 3, 40, 50)
    assert (a[:40, :50] == b).all()


def test_patches_and_gains():
    P = synth.patches(2, range(256))
    q = synth.patch_gain(2, range(256))
    assert P.shape == (256, 32, 32)
    assert q.min() >= 512 and q.max() <= 2048
    sd = P.reshape(256, -1).std(1)
    assert np.corrcoef(sd, np.minimum(q, 1400))[0, 1] > 0.5
    assert (synth.patches(2, [5, 7]) == P[[5, 7]]).all()


def test_keypoints():
    kp = synth.config_keypoints(0, 0)
    assert len(kp) == 500 and (kp["x"] >= 24).all() and (kp["x"] <= 640 - 25).all()
    assert (kp["y"] >= 24).all() and (kp["y"] <= 480 - 25).all()
    assert (kp["x"] == np.round(kp["x"])).all() and (kp["scale"] == 1).all() and (kp["angle"] == 0).all()
    kp = synth.config_keypoints(1, 3)
    assert len(kp) == 2000
    assert (kp["x"] >= 98).all() and (kp["x"] <= 1920 - 99).all()
    assert (kp["scale"] >= 1).all() and (kp["scale"] <= 4).all()
    assert (kp["angle"] >= 0).all() and (kp["angle"] <= np.float32(2 * math.pi)).all()
    kp4 = synth.config_keypoints(4, 0, 100)
    assert (kp4["scale"] <= 6).all() and (kp4["x"] >= 138).all()


def test_bad_tests_table():
    pairs, radii, thr = synth.bad_tests(0, 512)
    assert pairs.min() >= -16 and pairs.max() <= 15
    assert ((pairs[:, 0] != pairs[:, 2]) | (pairs[:, 1] != pairs[:, 3])).all()
    assert set(radii.tolist()) == {1, 2, 3, 4, 5}
    assert thr.min() >= -20 and thr.max() <= 20
    p2, r2, t2 = synth.bad_tests(0, 256)
    assert (p2 == pairs[:256]).all() and (t2 == thr[:256]).all()


def test_hashsift_matrix():
    B = synth.hashsift_matrix(3, 256)
    assert B.shape == (256, 129) and B.dtype == np.float32
    assert abs(B[:, :128].std() - math.sqrt(1 / 128)) < 0.003
    assert abs(B[:, 128].std() - 0.1) < 0.02


def test_keypoint_batch_matches_per_image():
    c = synth.CONFIGS[4]
    b = synth.keypoints_random_batch(4, [3, 9], 50, c["H"], c["W"], c["margin"], c["scale_max"])
    ref = np.concatenate([synth.keypoints_as_array(
        synth.keypoints_random(4, i, 50, c["H"], c["W"], c["margin"], c["scale_max"])) for i in (3, 9)])
    assert (b == ref).all()
