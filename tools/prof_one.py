#!/usr/bin/env python
"""Run one workload's C-ABI call a few times (for ncu captures of a single kernel).

  python tools/prof_one.py c3 [reps]     # hashsift_compute_patches on configs[3]
  python tools/prof_one.py c2 [reps]     # bad_compute_patches on configs[2]
  python tools/prof_one.py c1 [reps]     # bad_compute on configs[1]
  python tools/prof_one.py c4 [reps]     # describe_warped on 64 configs[4] images
  python tools/prof_one.py m1 [reps]     # match_hamming, 64 pairs of 4000 x 4000, K = 512
  python tools/prof_one.py c4b [reps]    # bilinear warp only, 64 configs[4] images
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_08380_b200 as bd  # noqa: E402
import synth  # noqa: E402
import synth.gpu as sg  # noqa: E402

which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if which == "c3":
    P = sg.patches(3, 0, 1_000_000)
    m = bd.HashSiftModel(synth.hashsift_matrix(3, 256))
    fn = lambda: bd.hashsift_compute_patches(m, P)  # noqa: E731
elif which == "c2":
    P = sg.patches(2, 0, 4_000_000)
    m = bd.BadModel(*synth.bad_tests(2, 256))
    fn = lambda: bd.bad_compute_patches(m, P)  # noqa: E731
elif which == "c1":
    c = synth.CONFIGS[1]
    imgs = sg.images(1, 0, c["n_images"], c["H"], c["W"])
    kp = torch.from_numpy(synth.keypoints_random_batch(1, range(c["n_images"]), c["kp_per_image"], c["H"], c["W"],
                                                       c["margin"], c["scale_max"])).cuda()
    kpi = torch.from_numpy(np.repeat(np.arange(c["n_images"], dtype=np.int32), c["kp_per_image"])).cuda()
    m = bd.BadModel(*synth.bad_tests(1, 512))
    fn = lambda: bd.bad_compute(m, imgs, kp, kpi)  # noqa: E731
elif which == "m1":
    rng = np.random.default_rng(5)
    n_pairs, n, K = 64, 4000, 512
    b = rng.integers(0, 2**32, size=(n_pairs * n, K // 32), dtype=np.uint64).astype(np.uint32)
    ta = torch.from_numpy(b.view(np.int32)).cuda()
    off = np.arange(n_pairs + 1, dtype=np.int64) * n
    fn = lambda: bd.match_hamming(ta, ta, off, off, K)  # noqa: E731
elif which == "c4b":
    c = synth.CONFIGS[4]
    n = 64
    imgs = sg.images(4, 0, n, c["H"], c["W"])
    kp = torch.from_numpy(synth.keypoints_random_batch(4, range(n), c["kp_per_image"], c["H"], c["W"], c["margin"],
                                                       c["scale_max"])).cuda()
    kpi = torch.from_numpy(np.repeat(np.arange(n, dtype=np.int32), c["kp_per_image"])).cuda()
    fn = lambda: bd.warp_patches(imgs, kp, kpi, mode="bilinear")  # noqa: E731
else:
    c = synth.CONFIGS[4]
    n = 64
    imgs = sg.images(4, 0, n, c["H"], c["W"])
    kp = torch.from_numpy(synth.keypoints_random_batch(4, range(n), c["kp_per_image"], c["H"], c["W"], c["margin"],
                                                       c["scale_max"])).cuda()
    kpi = torch.from_numpy(np.repeat(np.arange(n, dtype=np.int32), c["kp_per_image"])).cuda()
    mb, mh = bd.BadModel(*synth.bad_tests(4, 512)), bd.HashSiftModel(synth.hashsift_matrix(4, 256))
    fn = lambda: bd.describe_warped(mb, mh, imgs, kp, kpi)  # noqa: E731
for _ in range(reps):
    fn()
torch.cuda.synchronize()
print("ok", which)
