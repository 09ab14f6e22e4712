"""GPU tests of bd_describe_warped_host (the end-to-end call from host buffers):
results bit-identical to the device call bd_describe_warped_ex for every chunking, BAD-512
bit-exact and HashSIFT-256 under the band rule (R13) against the oracle, keypoints whose
image index is out of range zeroed with status 1, pinned and pageable buffers alike."""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import assert_bad_exact, hashsift_compare

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


def _inputs(seed, n_img, per, H, W):
    imgs = synth.images(seed, range(n_img), H, W)
    rng = np.random.default_rng(seed)
    n = n_img * per
    kp = np.zeros((n, 4), np.float32)
    kp[:, 0] = rng.uniform(0, W - 1, n)
    kp[:, 1] = rng.uniform(0, H - 1, n)
    kp[:, 2] = rng.uniform(0, 2 * math.pi, n)
    kp[:, 3] = np.exp(rng.uniform(0, math.log(3.0), n))
    kpi = np.sort(rng.integers(0, n_img, n)).astype(np.int32)
    kpi[:3] = -1          # before image 0: invalid
    kpi[-2:] = n_img      # past the last image: invalid
    kp[10] = [np.nan, 1, 0, 1]
    return imgs, kp, kpi


@pytest.fixture(scope="module")
def case(torch, bd):
    imgs, kp, kpi = _inputs(51, 7, 400, 320, 480)
    pairs, radii, thr = synth.bad_tests(51, 512)
    B = synth.hashsift_matrix(51, 256)
    mb, mh = bd.BadModel(pairs, radii, thr), bd.HashSiftModel(B)
    st_dev = torch.empty(len(kp), dtype=torch.uint8, device="cuda")
    ob, oh = bd.describe_warped(mb, mh, torch.from_numpy(imgs).cuda(), torch.from_numpy(kp).cuda(),
                                torch.from_numpy(kpi).cuda(), status=st_dev)
    torch.cuda.synchronize()
    return dict(imgs=imgs, kp=kp, kpi=kpi, pairs=pairs, radii=radii, thr=thr, B=B, mb=mb, mh=mh,
                dev=(ob.cpu().numpy(), oh.cpu().numpy(), st_dev.cpu().numpy()))


@pytest.mark.parametrize("chunk", [1, 3, 0, 7, 100])
@pytest.mark.parametrize("pinned", [True, False])
def test_host_equals_device(torch, bd, case, chunk, pinned):
    imgs = torch.from_numpy(case["imgs"])
    kp, kpi = torch.from_numpy(case["kp"]), torch.from_numpy(case["kpi"])
    if pinned:
        imgs, kp, kpi = imgs.pin_memory(), kp.pin_memory(), kpi.pin_memory()
    status = torch.full((len(kp),), 7, dtype=torch.uint8)
    ob, oh = bd.describe_warped_host(case["mb"], case["mh"], imgs, kp, kpi, status=status, chunk_images=chunk)
    db, dh, dst = case["dev"]
    assert (status.numpy() == dst).all()
    assert (ob.numpy() == db).all()
    assert (oh.numpy() == dh).all()


def test_host_oracle_parity(torch, bd, case):
    imgs, kp, kpi = case["imgs"], case["kp"], case["kpi"]
    status = torch.empty(len(kp), dtype=torch.uint8)
    ob, oh = bd.describe_warped_host(case["mb"], case["mh"], torch.from_numpy(imgs), torch.from_numpy(kp),
                                     torch.from_numpy(kpi), status=status, chunk_images=2)
    st = status.numpy()
    out_range = (kpi < 0) | (kpi >= len(imgs))
    assert st[out_range].all() and st[10] == 1
    assert (ob.numpy()[out_range] == 0).all() and (oh.numpy()[out_range] == 0).all()
    ok = ~out_range
    P, st_ref = oracle.warp_nn(imgs, kp[ok], kp_image=kpi[ok], want_status=True)
    assert (st[ok] == st_ref).all()
    ref_bad = oracle.bad_patches(P, case["pairs"], case["radii"], case["thr"])
    ref_hs, proj = oracle.project(oracle.sift(P), case["B"], want_proj=True)
    ref_bad[st_ref == 1] = 0
    ref_hs[st_ref == 1] = 0
    proj[st_ref == 1] = 1.0
    assert_bad_exact(ob.numpy()[ok], ref_bad, 512, what="host-path BAD-512")
    hashsift_compare(oh.numpy()[ok], ref_hs, proj, 256)


def test_host_bad_only_and_errors(torch, bd, case):
    imgs, kp, kpi = (torch.from_numpy(case[k]) for k in ("imgs", "kp", "kpi"))
    ob, oh = bd.describe_warped_host(case["mb"], None, imgs, kp, kpi, chunk_images=4)
    assert oh is None and (ob.numpy() == case["dev"][0]).all()
    bad_order = kpi.clone()
    bad_order[5], bad_order[-5] = bad_order[-5].item(), bad_order[5].item()
    with pytest.raises(bd.BindescError, match="non-decreasing"):
        bd.describe_warped_host(case["mb"], None, imgs, kp, bad_order)
    # empty keypoint set: nothing to do
    e = torch.empty((0, 4), dtype=torch.float32)
    ob, _ = bd.describe_warped_host(case["mb"], None, imgs, e, torch.empty(0, dtype=torch.int32))
    assert ob.shape == (0, 16)


def test_host_bilinear_equals_device(torch, bd, case):
    """the host pipeline forwards the warp mode (NEXT-2 bilinear) unchanged"""
    imgs, kp, kpi = (torch.from_numpy(case[k]) for k in ("imgs", "kp", "kpi"))
    db, dh = bd.describe_warped(case["mb"], case["mh"], imgs.cuda(), kp.cuda(), kpi.cuda(), mode="bilinear")
    torch.cuda.synchronize()
    ob, oh = bd.describe_warped_host(case["mb"], case["mh"], imgs, kp, kpi, mode="bilinear", chunk_images=2)
    assert (ob.numpy() == db.cpu().numpy()).all() and (oh.numpy() == dh.cpu().numpy()).all()
