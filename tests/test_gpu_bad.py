"""GPU parity of the BAD path (configs[0], [1], [2]) against the CPU oracle — bit-exact.

All calls go through the C ABI (paper_2108_08380_b200 ctypes binding).  Inputs are the
seeded synthetic workloads of BASELINE.json; the oracle computes its side from the numpy
generator (never from anything the CUDA path produced)."""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import assert_bad_exact, to_bytes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def bd():
    import paper_2108_08380_b200 as bd
    return bd


def _kp_tensor(torch, kp):
    return torch.from_numpy(synth.keypoints_as_array(kp) if kp.dtype.names else kp).cuda()


# ------------------------------------------------------------------ a1 integral --
def test_integral_spec_examples(torch, bd):
    # 1x1 [5] -> [[0,0],[0,5]];  2x2 [[1,2],[3,4]] -> [[0,0,0],[0,1,3],[0,4,10]]
    ii = bd.integral_image(torch.tensor([[5]], dtype=torch.uint8, device="cuda"))
    assert ii.cpu().numpy().tolist() == [[[0, 0], [0, 5]]]
    ii = bd.integral_image(torch.tensor([[1, 2], [3, 4]], dtype=torch.uint8, device="cuda"))
    assert ii.cpu().numpy().tolist() == [[[0, 0, 0], [0, 1, 3], [0, 4, 10]]]


@pytest.mark.parametrize("H,W", [(8, 8), (33, 33), (480, 640), (1080, 1920), (7, 1000), (600, 3)])
def test_integral_brute_force(torch, bd, H, W):
    rng = np.random.default_rng(H * W)
    img = rng.integers(0, 256, size=(2, H, W), dtype=np.uint8)
    ii = bd.integral_image(torch.from_numpy(img).cuda()).cpu().numpy().view(np.uint32)
    ref = np.zeros((2, H + 1, W + 1), np.int64)
    ref[:, 1:, 1:] = img.astype(np.int64).cumsum(1).cumsum(2)
    assert (ii == ref).all()
    if H * W <= 1200:  # every box = brute-force sum
        for y0 in range(H + 1):
            for y1 in range(y0, H + 1):
                x0, x1 = 0, W
                s = int(ii[0, y1, x1]) - int(ii[0, y0, x1]) - int(ii[0, y1, x0]) + int(ii[0, y0, x0])
                assert s == int(img[0, y0:y1, x0:x1].sum())


# ------------------------------------------------------------- configs[0] ---------
def test_c0_full_parity(torch, bd):
    c = synth.CONFIGS[0]
    img = synth.image(0, 0, c["H"], c["W"])
    kp = synth.keypoints_as_array(synth.config_keypoints(0, 0))
    pairs, radii, thr = synth.bad_tests(0, 256)
    ref = oracle.bad_image(img, kp, pairs, radii, thr)
    m = bd.BadModel(pairs, radii, thr)
    out = bd.bad_compute(m, torch.from_numpy(img).cuda(), torch.from_numpy(kp).cuda())
    torch.cuda.synchronize()
    assert out.shape == (500, 8)
    assert_bad_exact(out, ref, 256, what="c0")


def test_ramp_golden_through_gpu(torch, bd):
    # the hand-derived ramp cases (tests/golden/bad_ramp_8x8.txt) through the C ABI; K = 32
    # copies of each case padded with a harmless test
    import os
    y, x = np.mgrid[0:8, 0:8]
    img = torch.from_numpy((16 * x + 2 * y + 10).astype(np.uint8)).cuda()
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "bad_ramp_8x8.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        kx, ky, ang, sc, dx1, dy1, dx2, dy2, r, th, exp = [float(t) for t in line.split()]
        pairs = np.tile(np.array([[dx1, dy1, dx2, dy2]], np.int8), (32, 1))
        m = bd.BadModel(pairs, np.full(32, r, np.uint8), np.full(32, th, np.float32))
        kp = torch.tensor([[kx, ky, np.float32(ang), sc]], dtype=torch.float32, device="cuda")
        out = to_bytes(bd.bad_compute(m, img, kp))
        assert (np.unpackbits(out, bitorder="little") == int(exp)).all(), line


# ------------------------------------------------------------- configs[1] ---------
def test_c1_full_launch_sampled_parity(torch, bd):
    """all 64 1920x1080 images and 128,000 keypoints on the GPU (the bench launch); the
    oracle checks every keypoint of 3 sampled images (first, middle, last)."""
    import synth.gpu as sg
    c = synth.CONFIGS[1]
    n, H, W, per = c["n_images"], c["H"], c["W"], c["kp_per_image"]
    imgs = sg.images(1, 0, n, H, W)
    kp = np.concatenate([synth.keypoints_as_array(synth.config_keypoints(1, i)) for i in range(n)])
    kpi = np.repeat(np.arange(n, dtype=np.int32), per)
    pairs, radii, thr = synth.bad_tests(1, 512)
    m = bd.BadModel(pairs, radii, thr)
    status = torch.empty(n * per, dtype=torch.uint8, device="cuda")
    out = bd.bad_compute(m, imgs, torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda(), status=status)
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == 0).all()
    g = out.cpu().numpy()
    n_fragile = 0
    for i in (0, 31, 63):
        img = synth.image(1, i, H, W)
        sl = slice(i * per, (i + 1) * per)
        ref, st, fragile, _ = oracle.bad_image(img, kp[sl], pairs, radii, thr, want_aux=True)
        n_fragile += assert_bad_exact(g[sl], ref, 512, fragile=fragile, what=f"c1 image {i}")
    assert n_fragile > 0  # the hard R6 rows are among the rows checked (and matched exactly)


def test_rotated_scaled_random_with_borders(torch, bd):
    """keypoints anywhere (incl. the border rows/columns) on small images: clamped boxes,
    unequal areas, invalid keypoints, several images via kp_image."""
    rng = np.random.default_rng(7)
    H, W, n = 70, 90, 3
    imgs = synth.images(21, range(n), H, W)
    m_kp = 3000
    kp = np.zeros((m_kp, 4), np.float32)
    kp[:, 0] = rng.uniform(0, W - 1, m_kp)
    kp[:, 1] = rng.uniform(0, H - 1, m_kp)
    kp[:, 2] = rng.uniform(-7, 7, m_kp)
    kp[:, 3] = np.exp(rng.uniform(-1, 1.5, m_kp))
    kp[:20, 0] = np.arange(20) % 2 * (W - 1)   # exact borders
    kp[20:25] = [[np.nan, 3, 0, 1], [3, 3, 0, 0], [W, 3, 0, 1], [3, -1, 0, 1], [3, 3, np.inf, 1]]
    kpi = rng.integers(0, n, m_kp).astype(np.int32)
    kpi[30] = n  # invalid image index
    pairs, radii, thr = synth.bad_tests(21, 256, rmin=0, rmax=7)
    ref, st, fragile, _ = oracle.bad_image(imgs, kp, pairs, radii, thr, kp_image=kpi, want_aux=True)
    m = bd.BadModel(pairs, radii, thr)
    status = torch.empty(m_kp, dtype=torch.uint8, device="cuda")
    out = bd.bad_compute(m, torch.from_numpy(imgs).cuda(), torch.from_numpy(kp).cuda(),
                         torch.from_numpy(kpi).cuda(), status=status)
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == st).all()
    assert st[20:25].all() and st[30] == 1
    valid = st == 0
    assert valid.mean() > 0.9
    n_frag = assert_bad_exact(out, ref, 256, fragile=fragile, what="random/borders")
    assert n_frag > 0  # fragile rows are checked bit-exactly too (no exemption)


def test_bad_compute_empty(torch, bd):
    pairs, radii, thr = synth.bad_tests(0, 32)
    m = bd.BadModel(pairs, radii, thr)
    img = torch.zeros((10, 10), dtype=torch.uint8, device="cuda")
    out = bd.bad_compute(m, img, torch.zeros((0, 4), dtype=torch.float32, device="cuda"))
    assert out.shape == (0, 1)


# ------------------------------------------------------------- configs[2] ---------
@pytest.mark.parametrize("n,K", [(1, 256), (2, 32), (63, 256), (64, 512), (65, 256), (1000, 512), (4097, 256)])
def test_patches_ragged(torch, bd, n, K):
    P = synth.patches(2, range(n))
    pairs, radii, thr = synth.bad_tests(2 + K, K, rmin=0, rmax=7)
    ref = oracle.bad_patches(P, pairs, radii, thr)
    m = bd.BadModel(pairs, radii, thr)
    out = bd.bad_compute_patches(m, torch.from_numpy(P).cuda())
    torch.cuda.synchronize()
    assert_bad_exact(out, ref, K, what=f"patches n={n} K={K}")


def test_patches_extremes(torch, bd):
    # constant 0 / 255 patches, checkerboards, ties (integer thresholds on flat regions)
    P = np.zeros((8, 32, 32), np.uint8)
    P[1] = 255
    P[2] = (np.indices((32, 32)).sum(0) % 2 * 255).astype(np.uint8)
    P[3, :, 16:] = 255
    P[4] = np.arange(32, dtype=np.uint8)[None, :] * 8
    P[5] = 128
    P[6, 10:20, 10:20] = 255
    P[7] = np.random.default_rng(3).integers(0, 256, (32, 32))
    pairs, radii, thr = synth.bad_tests(5, 256, rmin=0, rmax=7)
    thr = np.round(thr / 4).astype(np.float32)
    ref, ties = oracle.bad_patches(P, pairs, radii, thr, want_ties=True)
    m = bd.BadModel(pairs, radii, thr)
    out = bd.bad_compute_patches(m, torch.from_numpy(P).cuda())
    assert ties.sum() > 0
    assert_bad_exact(out, ref, 256, what="extremes")


def test_c2_full_launch_sampled_parity(torch, bd):
    """all 4,000,000 configs[2] patches on the GPU (the bench launch); the oracle checks
    65,536 sampled patches (random + head + ragged tail)."""
    import synth.gpu as sg
    n = synth.CONFIGS[2]["n_patches"]
    P = sg.patches(2, 0, n)
    pairs, radii, thr = synth.bad_tests(2, 256)
    m = bd.BadModel(pairs, radii, thr)
    out = bd.bad_compute_patches(m, P)
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    idx = np.unique(np.concatenate([np.arange(512), n - 1 - np.arange(512), rng.integers(0, n, 64512)]))
    ref = oracle.bad_patches(synth.patches(2, idx), pairs, radii, thr)
    assert_bad_exact(out[torch.from_numpy(idx).cuda()], ref, 256, what="c2 sample")


def test_r6_fragile_keypoints_exact(torch, bd):
    """Hand-built R6-fragile keypoints (tests/test_oracle_bad.py pins the flag): a float64
    coefficient exactly on an fp32 rounding midpoint (scale 1 + 2^-23, angle 1.5 * 2^-30) and
    samples at n + 1/2 exactly and +-5e-5 from it, next to non-fragile controls.  The GPU
    evaluates the same fp32 rule, so every row must match bit-exactly."""
    img = synth.image(18, 0, 200, 200)
    pairs, radii, thr = synth.bad_tests(18, 512)
    base = [[100.0, 100.0, 1.5 * 2.0 ** -30, 1 + 2.0 ** -23],      # coefficient on a midpoint
            [100.0, 100.0, 1.25 * 2.0 ** -30, 1 + 2.0 ** -23],     # a quarter ulp away (control)
            [100.5, 100.0, 0.0, 1.0], [100.50005, 99.5, 0.0, 1.0], [99.49995, 100.5, 0.0, 1.0],
            [100.5002, 100.0, 0.0, 1.0]]
    rng = np.random.default_rng(18)
    extra = np.zeros((500, 4), np.float32)  # random keypoints with half-integer centres
    extra[:, 0] = rng.integers(60, 140, 500) + 0.5
    extra[:, 1] = rng.integers(60, 140, 500) + rng.choice([0.0, 0.5], 500)
    extra[:, 2] = rng.choice([0.0, np.float32(math.pi / 2), np.float32(math.pi), 1.5 * 2.0 ** -30], 500)
    extra[:, 3] = rng.choice([1.0, 2.0, 1 + 2.0 ** -23], 500)
    kp = np.concatenate([np.array(base, np.float32), extra])
    ref, st, fragile, _ = oracle.bad_image(img, kp, pairs, radii, thr, want_aux=True)
    assert (st == 0).all()
    assert list(fragile[:6]) == [1, 0, 1, 1, 1, 0]
    assert fragile.mean() > 0.5
    out = bd.bad_compute(bd.BadModel(pairs, radii, thr), torch.from_numpy(img).cuda(), torch.from_numpy(kp).cuda())
    torch.cuda.synchronize()
    assert_bad_exact(out, ref, 512, fragile=fragile, what="R6-fragile keypoints")


def test_local_path_large_windows(torch, bd):
    """Small batches take the one-launch local-integral kernel; keypoints whose window exceeds
    its shared-memory budget (scales 2.5-6 here) sum their boxes from the image bytes instead.
    Both must be bit-exact."""
    rng = np.random.default_rng(31)
    H, W, n, m_kp = 300, 320, 2, 400
    imgs = synth.images(31, range(n), H, W)
    kp = np.zeros((m_kp, 4), np.float32)
    kp[:, 0] = rng.uniform(0, W - 1, m_kp)
    kp[:, 1] = rng.uniform(0, H - 1, m_kp)
    kp[:, 2] = rng.uniform(0, 2 * np.pi, m_kp)
    kp[:, 3] = rng.uniform(2.5, 6.0, m_kp)
    kp[:40, 3] = rng.uniform(0.5, 1.5, 40)  # and some that fit
    kpi = rng.integers(0, n, m_kp).astype(np.int32)
    pairs, radii, thr = synth.bad_tests(31, 512, rmin=0, rmax=7)
    ref, st, fragile, _ = oracle.bad_image(imgs, kp, pairs, radii, thr, kp_image=kpi, want_aux=True)
    m = bd.BadModel(pairs, radii, thr)
    out = bd.bad_compute(m, torch.from_numpy(imgs).cuda(), torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda())
    torch.cuda.synchronize()
    assert (st == 0).all()
    assert_bad_exact(out, ref, 512, fragile=fragile, what="local path, large windows")


def test_regular_image_path_parity():
    """The image-integral path (vec uint16 integral, spatial order, box-clustered kernel) that
    large batches take: the image-path parity tests again with the local path switched off
    (BINDESC_LOCAL_MAX_KP=0), in a subprocess."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, BINDESC_LOCAL_MAX_KP="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_bad.py", "tests/test_gpu_fuzz.py",
                        "-k", "(c0_full or ramp_golden or rotated_scaled or fragile or large_windows or bad_image_fuzz)"
                              " and not regular_image_path"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
