"""Seeded fuzz of the C ABI against the oracle over the parameter space the header allows:
pitch > W, tiny and odd image sizes, every K in 32..512 (step 32) on both BAD paths, radii 0..7,
HashSIFT N in 32..512, patch counts around tile boundaries, and keypoints anywhere (borders,
outside, non-finite).  BAD bit-exact on every row (R6-fragile rows included; their count is reported), HashSIFT under
R13, warps byte-exact."""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import assert_bad_exact, hashsift_compare, to_bytes

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


def _pitched(torch, imgs, extra):
    """device images with row pitch W + extra (the C ABI's pitch argument) -> (tensor view, base)"""
    n, H, W = imgs.shape
    buf = torch.zeros((n, H, W + extra), dtype=torch.uint8, device="cuda")
    buf[:, :, :W] = torch.from_numpy(imgs).cuda()
    return buf


@pytest.mark.parametrize("case", range(8))
def test_bad_image_fuzz(torch, bd, case):
    rng = np.random.default_rng(1000 + case)
    H, W = int(rng.integers(1, 200)), int(rng.integers(1, 260))
    n_img = int(rng.integers(1, 4))
    K = int(rng.integers(1, 17)) * 32
    imgs = synth.images(60 + case, range(n_img), H, W)
    m = int(rng.integers(1, 700))
    kp = np.zeros((m, 4), np.float32)
    # most keypoints valid (centre inside the image, image index in range) so the clamped-box /
    # unequal-area compare branch is exercised on real rows; ~10% invalid of each kind
    kp[:, 0] = rng.uniform(0, W - 1, m)
    kp[:, 1] = rng.uniform(0, H - 1, m)
    out_x = rng.random(m) < 0.05
    kp[out_x, 0] = rng.choice([-2.0, -0.01, W - 0.99, W + 1.0], out_x.sum())
    out_y = rng.random(m) < 0.05
    kp[out_y, 1] = rng.choice([-2.0, -0.01, H - 0.99, H + 1.0], out_y.sum())
    border = rng.random(m) < 0.1  # exact border rows / columns
    kp[border, 0] = rng.choice([0.0, W - 1.0], border.sum())
    kp[:, 2] = rng.uniform(-10, 10, m)
    kp[:, 3] = np.exp(rng.uniform(-1.5, 1.8, m))
    kp[rng.random(m) < 0.02, 3] = np.nan
    kpi = rng.integers(0, n_img, m).astype(np.int32)
    bad_i = rng.random(m) < 0.05
    kpi[bad_i] = rng.choice([-1, n_img], bad_i.sum())
    pairs, radii, thr = synth.bad_tests(70 + case, K, rmin=0, rmax=7)
    ref, st, fragile, _ = oracle.bad_image(imgs, kp, pairs, radii, thr, kp_image=kpi, want_aux=True)
    assert (st == 0).mean() >= 0.5, f"case {case}: only {(st == 0).mean():.0%} valid keypoints"
    extra = int(rng.integers(0, 40))
    buf = _pitched(torch, imgs, extra)
    # the binding derives the pitch from the tensor stride: pass the padded buffer's [:, :, :W] view
    view = buf[:, :, :W]
    L = bd.lib()
    import ctypes
    model = bd.BadModel(pairs, radii, thr)
    out = torch.empty((m, K // 32), dtype=torch.int32, device="cuda")
    status = torch.empty(m, dtype=torch.uint8, device="cuda")
    tk, ti = torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda()
    if case % 2:  # the binding accepts the row-strided view (pitch from stride(1))
        bd.bad_compute(model, view, tk, ti, out=out, status=status)
    else:         # the raw C ABI with an explicit pitch
        rc = L.bad_compute(model.handle, view.data_ptr(), n_img, H, W, W + extra, tk.data_ptr(), ti.data_ptr(), m,
                           out.data_ptr(), status.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert rc == 0, L.bd_last_error()
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == st).all()
    assert_bad_exact(out, ref, K, fragile=fragile, what=f"fuzz {case}: {n_img}x{H}x{W} pitch {W + extra} K {K}")


# rmax 5: every clamped area <= 121 -> the DP2A record form; rmax 7: areas up to 225 -> the
# integer form (PatchTest, internal.cuh)
@pytest.mark.parametrize("rmax", [5, 7])
@pytest.mark.parametrize("K", list(range(32, 513, 32)))
def test_bad_patches_every_K(torch, bd, K, rmax):
    rng = np.random.default_rng(K + rmax)
    n = int(rng.integers(1, 300))
    P = synth.patches(80 + K, range(n))
    pairs, radii, thr = synth.bad_tests(90 + K + rmax, K, rmin=0, rmax=rmax)
    out = bd.bad_compute_patches(bd.BadModel(pairs, radii, thr), torch.from_numpy(P).cuda())
    torch.cuda.synchronize()
    assert_bad_exact(out, oracle.bad_patches(P, pairs, radii, thr), K, what=f"patches K={K}")


@pytest.mark.parametrize("N", [32, 64, 96, 160, 224, 256, 288, 384, 480, 512])
def test_hashsift_every_N(torch, bd, N):
    n = 300 + N
    P = synth.patches(5, range(n))
    B = synth.hashsift_matrix(100 + N, N)
    out = bd.hashsift_compute_patches(bd.HashSiftModel(B), torch.from_numpy(P).cuda())
    torch.cuda.synchronize()
    ref, proj = oracle.project(oracle.sift(P), B, want_proj=True)
    hashsift_compare(out, ref, proj, N)


@pytest.mark.parametrize("pad", [19, 17])  # pitch 152 (4-aligned rows: bilinear pair loads) / 150
@pytest.mark.parametrize("mode", ["nn", "bilinear"])
def test_warp_pitched_fuzz(torch, bd, mode, pad):
    rng = np.random.default_rng(7 if mode == "nn" else 8)
    H, W, n_img, m = 77, 133, 2, 900
    imgs = synth.images(9, range(n_img), H, W)
    kp = np.zeros((m, 4), np.float32)
    kp[:, 0] = rng.uniform(0, W - 1, m)
    kp[:, 1] = rng.uniform(0, H - 1, m)
    kp[:, 2] = rng.uniform(0, 2 * math.pi, m)
    kp[:, 3] = np.exp(rng.uniform(-1, 1.5, m))
    kpi = rng.integers(0, n_img, m).astype(np.int32)
    f = oracle.warp_nn if mode == "nn" else oracle.warp_bilinear
    ref = f(imgs, kp, kp_image=kpi)
    buf = _pitched(torch, imgs, pad)
    L = bd.lib()
    out = torch.empty((m, 32, 32), dtype=torch.uint8, device="cuda")
    tk, ti = torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda()
    rc = L.bd_warp_patches_ex(buf.data_ptr(), n_img, H, W, W + pad, tk.data_ptr(), ti.data_ptr(), m,
                              bd.WARP_MODES[mode], out.data_ptr(), None, torch.cuda.current_stream().cuda_stream)
    assert rc == 0, L.bd_last_error()
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == ref).all()


def test_cuda_core_patch_build_parity():
    """The CUDA-core patch kernel (bad_patch.cu), which the tensor-core build (bad_patch_tc.cu)
    replaced as the default: its own parity run, in a subprocess with BINDESC_PATCH_TC=0."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, BINDESC_PATCH_TC="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_fuzz.py", "tests/test_gpu_bad.py",
                        "-k", "bad_patches_every_K or patches_ragged or patches_extremes"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
