"""GPU parity of the NEXT-2 / NEXT-3 variants against the oracle (C ABI):
bilinear warp byte-exact (the fp32 quantisation rule R28 is shared), BAD with scaled radius
bit-exact (R27), RootSIFT within the R14 SIFT tolerance and HashSIFT bits under R13, HashSIFT-512
 under R13, and the ORB-equivalent table (r = 2, theta = 0) bit-exact."""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import assert_bad_exact, assert_sift_close, hashsift_compare

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


def _kps(seed, n, H, W, margin, smax, n_img):
    rng = np.random.default_rng(seed)
    kp = np.zeros((n, 4), np.float32)
    kp[:, 0] = rng.uniform(0, W - 1, n)
    kp[:, 1] = rng.uniform(0, H - 1, n)
    kp[:, 2] = rng.uniform(0, 2 * math.pi, n)
    kp[:, 3] = np.exp(rng.uniform(0, math.log(smax), n))
    kp[: n // 2, 0] = rng.uniform(margin, W - 1 - margin, n // 2)   # half inside, half near borders
    kp[: n // 2, 1] = rng.uniform(margin, H - 1 - margin, n // 2)
    kpi = rng.integers(0, n_img, n).astype(np.int32)
    return kp, kpi


def test_bilinear_warp_parity(torch, bd):
    imgs = synth.images(41, range(3), 300, 400)
    kp, kpi = _kps(41, 4000, 300, 400, 100, 3.0, 3)
    kp[:3] = [[0, 0, 0.3, 2.0], [np.nan, 1, 0, 1], [15.5, 15.5, 0, 1]]
    ref, st = oracle.warp_bilinear(imgs, kp, kp_image=kpi, want_status=True)
    status = torch.empty(len(kp), dtype=torch.uint8, device="cuda")
    out = bd.warp_patches(torch.from_numpy(imgs).cuda(), torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda(),
                          status=status, mode="bilinear")
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == st).all()
    g = out.cpu().numpy()
    bad = np.nonzero((g != ref).reshape(len(kp), -1).any(1))[0]
    assert len(bad) == 0, bad[:10]


def test_describe_warped_bilinear(torch, bd):
    imgs = synth.images(42, range(2), 400, 500)
    kp, kpi = _kps(42, 3000, 400, 500, 120, 3.0, 2)
    pairs, radii, thr = synth.bad_tests(42, 256)
    B = synth.hashsift_matrix(42, 256)
    P, st = oracle.warp_bilinear(imgs, kp, kp_image=kpi, want_status=True)
    ref_bad = oracle.bad_patches(P, pairs, radii, thr)
    ref_hs, proj = oracle.project(oracle.sift(P), B, want_proj=True)
    ref_bad[st == 1] = 0
    ref_hs[st == 1] = 0
    proj[st == 1] = 1.0
    ob, oh = bd.describe_warped(bd.BadModel(pairs, radii, thr), bd.HashSiftModel(B), torch.from_numpy(imgs).cuda(),
                                torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda(), mode="bilinear")
    torch.cuda.synchronize()
    assert_bad_exact(ob, ref_bad, 256, what="BAD on bilinear patches")
    hashsift_compare(oh, ref_hs, proj, 256)


def test_bad_scaled_radius_parity(torch, bd):
    imgs = synth.images(43, range(2), 260, 330)
    kp, kpi = _kps(43, 3000, 260, 330, 80, 4.0, 2)
    pairs, radii, thr = synth.bad_tests(43, 512, rmin=0, rmax=7)
    ref, st = oracle.bad_image_scaled(imgs, kp, pairs, radii, thr, kp_image=kpi, want_status=True)
    status = torch.empty(len(kp), dtype=torch.uint8, device="cuda")
    out = bd.bad_compute(bd.BadModel(pairs, radii, thr, scale_radius=True), torch.from_numpy(imgs).cuda(),
                         torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda(), status=status)
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == st).all()
    # every row bit-exact, R6-fragile sample points included (no exemption)
    _, _, fragile, _ = oracle.bad_image(imgs, kp, pairs, radii, thr, kp_image=kpi, want_aux=True)
    assert_bad_exact(out, ref, 512, fragile=fragile, what="scaled radius")


def test_rootsift_parity(torch, bd):
    import synth.gpu as sg
    n = 20000
    P = sg.patches(3, 0, n)
    B = synth.hashsift_matrix(44, 256)
    m = bd.HashSiftModel(B, rootsift=True)
    out, sift = bd.hashsift_compute_patches(m, P, want_sift=True)
    torch.cuda.synchronize()
    Ph = synth.patches(3, range(n))
    v = oracle.root_sift(oracle.sift(Ph))
    assert_sift_close(sift, v)
    ref, proj = oracle.project(v, B, want_proj=True)
    hashsift_compare(out, ref, proj, 256)


def test_hashsift_512_parity(torch, bd):
    import synth.gpu as sg
    n = 20000
    P = sg.patches(3, 0, n)
    B = synth.hashsift_matrix(45, 512)
    out = bd.hashsift_compute_patches(bd.HashSiftModel(B), P)
    torch.cuda.synchronize()
    ref, proj = oracle.project(oracle.sift(synth.patches(3, range(n))), B, want_proj=True)
    hashsift_compare(out, ref, proj, 512)


def test_orb_equivalent_table(torch, bd):
    # ORB = "BAD features with s = 5 and theta = 0" -> radius 2, all thresholds 0
    import synth.gpu as sg
    pairs, _, _ = synth.bad_tests(46, 256)
    radii = np.full(256, 2, np.uint8)
    thr = np.zeros(256, np.float32)
    n = 50000
    P = sg.patches(2, 0, n)
    out = bd.bad_compute_patches(bd.BadModel(pairs, radii, thr), P)
    torch.cuda.synchronize()
    ref = oracle.bad_patches(synth.patches(2, range(n)), pairs, radii, thr)
    assert_bad_exact(out, ref, 256, what="ORB-equivalent table")


def test_bad_scaled_radius_large_scales(torch, bd):
    """scales of 20..400 on a 300x300 image with radii up to 7 — scaled radii
    beyond the image extent and clamped areas up to 300*300, whose product needs int64."""
    imgs = synth.images(45, range(1), 300, 300)
    rng = np.random.default_rng(45)
    m = 100  # every box is large: the oracle sums up to 90,000 pixels per box by brute force
    kp = np.stack([rng.uniform(0, 299, m), rng.uniform(0, 299, m), rng.uniform(0, 6.3, m),
                   np.exp(rng.uniform(np.log(20), np.log(400), m))], 1).astype(np.float32)
    kp[:4, 3] = [20.0, 1e3, 1e4, 5e4]  # r' = r * scale far beyond the image: clamped boxes
    pairs, radii, thr = synth.bad_tests(45, 256, rmin=0, rmax=7)
    ref, st = oracle.bad_image_scaled(imgs, kp, pairs, radii, thr, want_status=True)
    out = bd.bad_compute(bd.BadModel(pairs, radii, thr, scale_radius=True), torch.from_numpy(imgs).cuda(),
                         torch.from_numpy(kp).cuda())
    torch.cuda.synchronize()
    assert (st == 0).all()
    assert_bad_exact(out, ref, 256, what="scaled radius, large scales")
