#!/usr/bin/env python
"""Per-workload device timing of the C-ABI entry points (configs[1], [2], [3], [4-slice]).

  python tools/kbench.py [--which c1,c2,c3,c4] [--reps 10]

Prints one JSON object per workload: ms per call (CUDA events, after 3 warm-ups), per-kernel
breakdown from the library's tracing, Mdesc/s and the HBM-roofline fraction of the
algorithmic bytes."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2108_08380_b200 as bd
import synth
import synth.gpu as sg

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bd.profile_start()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    prof = bd.profile_stop()
    ms = e0.elapsed_time(e1) / reps
    return ms, {k: round(v[1] / reps, 4) for k, v in prof.items()}


def report(name, ms, prof, n_desc, alg_bytes):
    r = {"workload": name, "ms": round(ms, 4), "Mdesc_s": round(n_desc / ms / 1e3, 2),
         "alg_GBps": round(alg_bytes / ms / 1e6, 1), "hbm_frac": round(alg_bytes / ms / 1e6 / HBM, 4),
         "kernels_ms": prof}
    print(json.dumps(r), flush=True)
    return r


def c1(reps):
    c = synth.CONFIGS[1]
    n, H, W, per = c["n_images"], c["H"], c["W"], c["kp_per_image"]
    imgs = sg.images(1, 0, n, H, W)
    kp = torch.from_numpy(synth.keypoints_random_batch(1, range(n), per, H, W, c["margin"], c["scale_max"])).cuda()
    kpi = torch.from_numpy(np.repeat(np.arange(n, dtype=np.int32), per)).cuda()
    m = bd.BadModel(*synth.bad_tests(1, 512))
    out = torch.empty((n * per, 16), dtype=torch.int32, device="cuda")
    ms, prof = timeit(lambda: bd.bad_compute(m, imgs, kp, kpi, out=out), reps)
    return report("c1 BAD-512 images", ms, prof, n * per, n * H * W + n * per * 64)


def c2(reps):
    n = synth.CONFIGS[2]["n_patches"]
    P = sg.patches(2, 0, n)
    m = bd.BadModel(*synth.bad_tests(2, 256))
    out = torch.empty((n, 8), dtype=torch.int32, device="cuda")
    ms, prof = timeit(lambda: bd.bad_compute_patches(m, P, out=out), reps)
    return report("c2 BAD-256 patches", ms, prof, n, n * (1024 + 32))


def c3(reps):
    n = synth.CONFIGS[3]["n_patches"]
    P = sg.patches(3, 0, n)
    m = bd.HashSiftModel(synth.hashsift_matrix(3, 256))
    out = torch.empty((n, 8), dtype=torch.int32, device="cuda")
    ms, prof = timeit(lambda: bd.hashsift_compute_patches(m, P, out=out), reps)
    return report("c3 HashSIFT-256 patches", ms, prof, n, n * (1024 + 32))


def c4(reps, n_img=256):
    c = synth.CONFIGS[4]
    H, W, per = c["H"], c["W"], c["kp_per_image"]
    imgs = sg.images(4, 0, n_img, H, W)
    kp = torch.from_numpy(synth.keypoints_random_batch(4, range(n_img), per, H, W, c["margin"], c["scale_max"])).cuda()
    kpi = torch.from_numpy(np.repeat(np.arange(n_img, dtype=np.int32), per)).cuda()
    mb, mh = bd.BadModel(*synth.bad_tests(4, 512)), bd.HashSiftModel(synth.hashsift_matrix(4, 256))
    m = n_img * per
    ob = torch.empty((m, 16), dtype=torch.int32, device="cuda")
    oh = torch.empty((m, 8), dtype=torch.int32, device="cuda")
    ms, prof = timeit(lambda: bd.describe_warped(mb, mh, imgs, kp, kpi, out_bad=ob, out_hs=oh), reps)
    return report(f"c4 slice ({n_img} images)", ms, prof, m, m * (2074 + 96))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="c1,c2,c3,c4")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    for w in a.which.split(","):
        globals()[w](a.reps)
        torch.cuda.empty_cache()
