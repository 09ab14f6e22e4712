"""GPU parity of the HashSIFT path (configs[3]) and the warped path (configs[4]) against the
CPU oracle: SIFT within 1e-4 relative (R14); hash bits equal except where the oracle's
|projection| < 1e-3, with those at most 0.1% of all bits (R13); warp and BAD-on-warped
bit-exact."""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import assert_bad_exact, assert_sift_close, hashsift_compare, to_bytes

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


def special_patches():
    P = np.zeros((10, 32, 32), np.uint8)
    P[1] = 93                                   # constant -> zero SIFT, bits = [b >= 0]
    P[2, :, 16:] = 255                          # vertical step edge
    P[3, :, :16] = 255                          # mirrored
    P[4, 16:, :] = 255                          # horizontal
    P[5, 11, 10] = 255                          # single pixel
    y, x = np.mgrid[0:32, 0:32]
    P[6] = (3 * x + 3 * y + 20).astype(np.uint8)  # 45-degree ramp
    P[7] = (np.indices((32, 32)).sum(0) % 2 * 255).astype(np.uint8)
    P[8] = np.random.default_rng(1).integers(0, 256, (32, 32))
    P[9] = 255
    return P


@pytest.mark.parametrize("n,N", [(10, 256), (1, 32), (33, 512), (1000, 256), (4099, 256)])
def test_hashsift_patches_small(torch, bd, n, N):
    P = np.concatenate([special_patches(), synth.patches(3, range(max(0, n - 10)))])[:n]
    B = synth.hashsift_matrix(3 + N, N)
    v = oracle.sift(P)
    ref, proj = oracle.project(v, B, want_proj=True)
    m = bd.HashSiftModel(B)
    out, sift = bd.hashsift_compute_patches(m, torch.from_numpy(P).cuda(), want_sift=True)
    torch.cuda.synchronize()
    assert_sift_close(sift, v)
    hashsift_compare(out, ref, proj, N)


def test_hashsift_constant_patch_bits_are_bias_signs(torch, bd):
    B = synth.hashsift_matrix(3, 256)
    m = bd.HashSiftModel(B)
    out = bd.hashsift_compute_patches(m, torch.full((4, 32, 32), 50, dtype=torch.uint8, device="cuda"))
    b = np.unpackbits(to_bytes(out), axis=1, bitorder="little")
    assert (b == (B[:, 128] >= 0)[None]).all()


def test_c3_full_launch_sampled_parity(torch, bd):
    """all 1,000,000 configs[3] patches on the GPU; the oracle checks 16,384 sampled."""
    import synth.gpu as sg
    n = synth.CONFIGS[3]["n_patches"]
    P = sg.patches(3, 0, n)
    B = synth.hashsift_matrix(3, 256)
    m = bd.HashSiftModel(B)
    out, sift = bd.hashsift_compute_patches(m, P, want_sift=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(12)
    idx = np.unique(np.concatenate([np.arange(256), n - 1 - np.arange(256), rng.integers(0, n, 15872)]))
    Ph = synth.patches(3, idx)
    v = oracle.sift(Ph)
    ref, proj = oracle.project(v, B, want_proj=True)
    ti = torch.from_numpy(idx).cuda()
    assert_sift_close(sift[ti], v)
    stats = hashsift_compare(out[ti], ref, proj, 256)
    print("c3 hash parity:", stats)


# ------------------------------------------------------------ configs[4] -------------
def _c4_inputs(n_img, per, H=None, W=None):
    c = synth.CONFIGS[4]
    H = H or c["H"]
    W = W or c["W"]
    imgs = synth.images(4, range(n_img), H, W)
    kp = np.concatenate([synth.keypoints_as_array(
        synth.keypoints_random(4, i, per, H, W, c["margin"], c["scale_max"])) for i in range(n_img)])
    kpi = np.repeat(np.arange(n_img, dtype=np.int32), per)
    return imgs, kp, kpi


def test_warp_parity(torch, bd):
    imgs, kp, kpi = _c4_inputs(2, 3000, 600, 800)
    kp[:5] = [[0, 0, 1.0, 6.0], [799, 599, 2.0, 6.0], [np.nan, 0, 0, 1], [3, 3, 0, -2], [400.5, 300.5, 0, 1]]
    ref, st = oracle.warp_nn(imgs, kp, kp_image=kpi, want_status=True)
    status = torch.empty(len(kp), dtype=torch.uint8, device="cuda")
    out = bd.warp_patches(torch.from_numpy(imgs).cuda(), torch.from_numpy(kp).cuda(),
                          torch.from_numpy(kpi).cuda(), status=status)
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == st).all()
    g = out.cpu().numpy()
    bad = np.nonzero((g != ref).reshape(len(kp), -1).any(1))[0]
    assert len(bad) == 0, bad[:10]


def test_describe_warped_parity(torch, bd):
    """configs[4] on 2 full-size 3840x2160 images x 4000 keypoints: BAD-512 on the warped
    patch bit-exact, HashSIFT-256 under the band rule, invalid keypoints zeroed."""
    imgs, kp, kpi = _c4_inputs(2, 4000)
    kp[7] = [np.nan, 1, 0, 1]
    pairs, radii, thr = synth.bad_tests(4, 512)
    B = synth.hashsift_matrix(4, 256)
    P, st = oracle.warp_nn(imgs, kp, kp_image=kpi, want_status=True)
    ref_bad = oracle.bad_patches(P, pairs, radii, thr)
    v = oracle.sift(P)
    ref_hs, proj = oracle.project(v, B, want_proj=True)
    ref_bad[st == 1] = 0
    ref_hs[st == 1] = 0
    proj[st == 1] = 1.0
    mb, mh = bd.BadModel(pairs, radii, thr), bd.HashSiftModel(B)
    status = torch.empty(len(kp), dtype=torch.uint8, device="cuda")
    ob, oh = bd.describe_warped(mb, mh, torch.from_numpy(imgs).cuda(), torch.from_numpy(kp).cuda(),
                                torch.from_numpy(kpi).cuda(), status=status)
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == st).all() and st[7] == 1
    assert_bad_exact(ob, ref_bad, 512, what="c4 BAD-512 on warped patches")
    hashsift_compare(oh, ref_hs, proj, 256)
    # hashsift_compute (images) = the HashSIFT half of the same step
    sift = torch.empty((len(kp), 128), dtype=torch.float32, device="cuda")
    oh2 = bd.hashsift_compute(mh, torch.from_numpy(imgs).cuda(), torch.from_numpy(kp).cuda(),
                              torch.from_numpy(kpi).cuda(), sift=sift)
    torch.cuda.synchronize()
    assert (oh2.cpu().numpy() == oh.cpu().numpy()).all()
    assert_sift_close(sift[torch.from_numpy(st == 0).cuda()], v[st == 0])


def test_c4_multichunk_sampled_parity(torch, bd):
    """configs[4] geometry at the size where bd_describe_warped runs two internal chunks
    (264 images x 4000 keypoints = 1,056,000 > 2^20) with the bench's launch configuration:
    inputs generated on the device by synth.gpu (byte-identical to the numpy generator), every
    keypoint of images 0, 262 (straddles the chunk boundary at keypoint 1,048,576) and 263
    checked against the oracle — BAD-512 bit-exact, HashSIFT-256 under the band rule."""
    import synth.gpu as sg
    c = synth.CONFIGS[4]
    H, W, per, n = c["H"], c["W"], c["kp_per_image"], 264
    imgs = sg.images(4, 0, n, H, W)
    kp = synth.keypoints_random_batch(4, range(n), per, H, W, c["margin"], c["scale_max"])
    kpi = np.repeat(np.arange(n, dtype=np.int32), per)
    pairs, radii, thr = synth.bad_tests(4, 512)
    B = synth.hashsift_matrix(4, 256)
    mb, mh = bd.BadModel(pairs, radii, thr), bd.HashSiftModel(B)
    status = torch.empty(len(kp), dtype=torch.uint8, device="cuda")
    ob, oh = bd.describe_warped(mb, mh, imgs, torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda(),
                                status=status)
    torch.cuda.synchronize()
    assert int(status.sum().item()) == 0
    gb, gh = ob.cpu().numpy(), oh.cpu().numpy()
    for i in (0, 262, 263):
        sl = slice(i * per, (i + 1) * per)
        P = oracle.warp_nn(synth.image(4, i, H, W), kp[sl])
        ref_bad = oracle.bad_patches(P, pairs, radii, thr)
        ref_hs, proj = oracle.project(oracle.sift(P), B, want_proj=True)
        assert_bad_exact(gb[sl], ref_bad, 512, what=f"c4 image {i}")
        hashsift_compare(gh[sl], ref_hs, proj, 256)


def test_c4_full_bench_config_sampled_parity(torch, bd):
    """configs[4] at its FULL size in bench.py's launch configuration (N = 1): all 8192
    3840x2160 images generated on the device (67.9 GB), all 32.768 M keypoints through one
    bd_describe_warped call (32 internal chunks of 2^20); every keypoint of images 0, 4095 and
    8191 (the first, a middle and the last chunk) checked against the oracle — BAD-512
    bit-exact, HashSIFT-256 under the band rule — and no keypoint flagged invalid."""
    import synth.gpu as sg
    c = synth.CONFIGS[4]
    H, W, per, n = c["H"], c["W"], c["kp_per_image"], c["n_images"]
    free, _ = torch.cuda.mem_get_info()
    if free < 80 * 2**30:
        pytest.skip("needs ~75 GB of free device memory")
    imgs = sg.images(4, 0, n, H, W)
    kp = torch.from_numpy(synth.keypoints_random_batch(4, range(n), per, H, W, c["margin"], c["scale_max"])).cuda()
    kpi = torch.from_numpy(np.repeat(np.arange(n, dtype=np.int32), per)).cuda()
    pairs, radii, thr = synth.bad_tests(4, 512)
    B = synth.hashsift_matrix(4, 256)
    mb, mh = bd.BadModel(pairs, radii, thr), bd.HashSiftModel(B)
    status = torch.empty(n * per, dtype=torch.uint8, device="cuda")
    ob, oh = bd.describe_warped(mb, mh, imgs, kp, kpi, status=status)
    torch.cuda.synchronize()
    assert int(status.sum().item()) == 0
    kp_np = kp.cpu().numpy()
    for i in (0, n // 2 - 1, n - 1):
        sl = slice(i * per, (i + 1) * per)
        P = oracle.warp_nn(synth.image(4, i, H, W), kp_np[sl])
        assert_bad_exact(ob[sl].cpu().numpy(), oracle.bad_patches(P, pairs, radii, thr), 512, what=f"c4 image {i}")
        ref_hs, proj = oracle.project(oracle.sift(P), B, want_proj=True)
        hashsift_compare(oh[sl].cpu().numpy(), ref_hs, proj, 256)


def octant_patches():
    """Linear ramps in 64 directions (every octant, both sides of each octant boundary, the axes
    and the diagonals exactly: |gx| == |gy|, gx == 0, gy == 0) and their mirrored / transposed
    variants — every pixel's gradient falls in a known octant, the cases the octant-indexed
    histogram entries (sift.cu) map to their two bins."""
    y, x = np.mgrid[0:32, 0:32].astype(np.float64)
    out = []
    for k in range(64):
        a = 2 * math.pi * k / 64
        out.append(np.clip(128 + 3.5 * (math.cos(a) * (x - 15.5) + math.sin(a) * (y - 15.5)), 0, 255))
    for dx, dy in [(1, 1), (-1, 1), (1, -1), (-1, -1), (0, 1), (1, 0), (0, -1), (-1, 0), (2, 1), (1, 2), (-2, 1)]:
        out.append(np.clip(128 + 3 * (dx * x + dy * y) - 3 * (dx + dy) * 15.5, 0, 255))
    return np.round(np.stack(out)).astype(np.uint8)


def test_sift_every_octant(torch, bd):
    P = octant_patches()
    B = synth.hashsift_matrix(77, 256)
    v = oracle.sift(P)
    ref, proj = oracle.project(v, B, want_proj=True)
    out, sift = bd.hashsift_compute_patches(bd.HashSiftModel(B), torch.from_numpy(P).cuda(), want_sift=True)
    torch.cuda.synchronize()
    assert_sift_close(sift, v)
    hashsift_compare(out, ref, proj, 256)
