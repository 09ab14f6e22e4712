"""GPU: the C ABI is safe to call from several host threads at once (bindesc.h: model
handles are immutable after create; workspace, kernel attributes and the host-pipeline
streams are per call / per thread / per device).  Four threads run describe_warped (each on
its own stream) and describe_warped_host concurrently on shared models; every result must
equal the single-threaded one bit for bit."""
import threading

import numpy as np
import pytest

import synth

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


def test_threads_share_models(torch, bd):
    H, W, n_img, per = 500, 700, 4, 600
    imgs_np = synth.images(71, range(n_img), H, W)
    kp_np = synth.keypoints_random_batch(71, range(n_img), per, H, W, 60, 2.5)
    kpi_np = np.repeat(np.arange(n_img, dtype=np.int32), per)
    mb, mh = bd.BadModel(*synth.bad_tests(71, 512)), bd.HashSiftModel(synth.hashsift_matrix(71, 256))
    imgs, kp, kpi = (torch.from_numpy(x).cuda() for x in (imgs_np, kp_np, kpi_np))
    ref_b, ref_h = bd.describe_warped(mb, mh, imgs, kp, kpi)
    torch.cuda.synchronize()
    ref_b, ref_h = ref_b.cpu(), ref_h.cpu()
    errors = []

    def device_worker(seed):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    ob, oh = bd.describe_warped(mb, mh, imgs, kp, kpi, stream=s)
                    s.synchronize()
                    if not (torch.equal(ob.cpu(), ref_b) and torch.equal(oh.cpu(), ref_h)):
                        errors.append(f"device worker {seed}: mismatch")
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(f"device worker {seed}: {e!r}")

    def host_worker(seed):
        try:
            h_imgs, h_kp, h_kpi = (torch.from_numpy(x) for x in (imgs_np, kp_np, kpi_np))
            for chunk in (1, 3):
                ob, oh = bd.describe_warped_host(mb, mh, h_imgs, h_kp, h_kpi, chunk_images=chunk)
                if not (torch.equal(ob, ref_b) and torch.equal(oh, ref_h)):
                    errors.append(f"host worker {seed}: mismatch (chunk {chunk})")
        except Exception as e:  # noqa: BLE001
            errors.append(f"host worker {seed}: {e!r}")

    threads = [threading.Thread(target=device_worker, args=(i,)) for i in range(2)]
    threads += [threading.Thread(target=host_worker, args=(i,)) for i in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
