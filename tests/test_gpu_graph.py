"""GPU: the C-ABI calls are stream-ordered and capturable into CUDA graphs (workspace comes
from the stream-ordered pool, no host synchronisation inside a call).  A captured
bd_describe_warped / bad_compute replays bit-identically to direct calls, including after the
captured input buffers are overwritten with new data (the graph reads them at replay)."""
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


def _capture(torch, fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    return g


def test_describe_warped_graph_replay(torch, bd):
    c = synth.CONFIGS[4]
    H, W, n_img, per = 600, 800, 3, 700
    imgs = torch.from_numpy(synth.images(61, range(n_img), H, W)).cuda()
    kp_a = synth.keypoints_random_batch(61, range(n_img), per, H, W, 40, c["scale_max"] / 2)
    kp_b = synth.keypoints_random_batch(62, range(n_img), per, H, W, 40, c["scale_max"] / 2)
    kpi = torch.from_numpy(np.repeat(np.arange(n_img, dtype=np.int32), per)).cuda()
    kp = torch.from_numpy(kp_a).cuda()
    mb, mh = bd.BadModel(*synth.bad_tests(61, 512)), bd.HashSiftModel(synth.hashsift_matrix(61, 256))
    m = n_img * per
    ob = torch.empty((m, 16), dtype=torch.int32, device="cuda")
    oh = torch.empty((m, 8), dtype=torch.int32, device="cuda")
    st = torch.empty(m, dtype=torch.uint8, device="cuda")
    g = _capture(torch, lambda: bd.describe_warped(mb, mh, imgs, kp, kpi, out_bad=ob, out_hs=oh, status=st))
    for kp_np in (kp_b, kp_a):
        kp.copy_(torch.from_numpy(kp_np))
        ob.zero_()
        oh.zero_()
        g.replay()
        torch.cuda.synchronize()
        rb, rh = bd.describe_warped(mb, mh, imgs, torch.from_numpy(kp_np).cuda(), kpi)
        torch.cuda.synchronize()
        assert torch.equal(ob, rb) and torch.equal(oh, rh)
        assert int(st.sum().item()) == 0


def test_bad_compute_graph_replay(torch, bd):
    c = synth.CONFIGS[0]
    img = torch.from_numpy(synth.image(0, 0, c["H"], c["W"])).cuda()
    kp = torch.from_numpy(synth.keypoints_as_array(synth.config_keypoints(0, 0))).cuda()
    m = bd.BadModel(*synth.bad_tests(0, 256))
    out = torch.empty((kp.shape[0], 8), dtype=torch.int32, device="cuda")
    g = _capture(torch, lambda: bd.bad_compute(m, img, kp, None, out=out))
    ref = bd.bad_compute(m, img, kp)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
