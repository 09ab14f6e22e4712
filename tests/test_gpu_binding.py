"""The Python binding's argument checks: the C ABI cannot see the size of a
device buffer, so the binding rejects wrong shapes / dtypes / devices before any launch —
and accepts row-strided image views (a pitched buffer) with the pitch taken from stride(1)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import assert_bad_exact

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


def test_rejects_wrong_buffers(torch, bd):
    img = torch.zeros((2, 64, 64), dtype=torch.uint8, device="cuda")
    m = bd.BadModel(*synth.bad_tests(0, 64))
    kp = torch.full((10, 4), 30.0, device="cuda")
    kp[:, 2] = 0
    kp[:, 3] = 1
    with pytest.raises(ValueError):  # short output buffer
        bd.bad_compute(m, img, kp, out=torch.empty((9, 2), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):  # too few words per row
        bd.bad_compute(m, img, kp, out=torch.empty((10, 1), dtype=torch.int32, device="cuda"))
    with pytest.raises(TypeError):
        bd.bad_compute(m, img, kp, out=torch.empty((10, 2), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):  # short kp_image
        bd.bad_compute(m, img, kp, torch.zeros(9, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):  # kps not (m, 4)
        bd.bad_compute(m, img, kp[:, :3].contiguous())
    with pytest.raises(ValueError):  # short status
        bd.bad_compute(m, img, kp, status=torch.empty(3, dtype=torch.uint8, device="cuda"))
    with pytest.raises(TypeError):   # CPU tensor: no fallback
        bd.bad_compute(m, img.cpu(), kp)
    hs = bd.HashSiftModel(synth.hashsift_matrix(0, 64))
    P = torch.zeros((5, 32, 32), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        bd.hashsift_compute_patches(hs, P, out=torch.empty((5, 3), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        bd.hashsift_compute_patches(hs, P, sift=torch.empty((4, 128), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        bd.describe_warped(m, hs, img, kp, out_hs=torch.empty((10, 1), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        bd.warp_patches(img, kp, out=torch.empty((10, 32, 31), dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):  # rows not contiguous
        bd.bad_compute(m, img[:, :, ::2], kp)


def test_pitched_view_matches_oracle(torch, bd):
    n, H, W, pad = 2, 90, 110, 13
    imgs = synth.images(33, range(n), H, W)
    buf = torch.zeros((n, H, W + pad), dtype=torch.uint8, device="cuda")
    buf[:, :, :W] = torch.from_numpy(imgs).cuda()
    rng = np.random.default_rng(33)
    kp = np.stack([rng.uniform(0, W - 1, 400), rng.uniform(0, H - 1, 400), rng.uniform(0, 6.3, 400),
                   np.exp(rng.uniform(-0.5, 1, 400))], 1).astype(np.float32)
    kpi = rng.integers(0, n, 400).astype(np.int32)
    pairs, radii, thr = synth.bad_tests(33, 256)
    ref = oracle.bad_image(imgs, kp, pairs, radii, thr, kp_image=kpi)
    out = bd.bad_compute(bd.BadModel(pairs, radii, thr), buf[:, :, :W], torch.from_numpy(kp).cuda(),
                         torch.from_numpy(kpi).cuda())
    torch.cuda.synchronize()
    assert_bad_exact(out, ref, 256, what="pitched view")
    P = bd.warp_patches(buf[:, :, :W], torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda())
    assert (P.cpu().numpy() == oracle.warp_nn(imgs, kp, kp_image=kpi)).all()
