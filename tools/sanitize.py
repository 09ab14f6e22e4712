#!/usr/bin/env python
"""One small invocation of a C-ABI entry point for compute-sanitizer (VERDICT r01 #8,
SURVEY §5; SPEC.md:255 concurrency contract).  Inputs are the seeded synthetic workloads at
reduced size; the outputs are checked against the oracle so a sanitizer run is also a parity
run.

  compute-sanitizer --tool racecheck python tools/sanitize.py c2
cases: c0, c1s (1 image of configs[1]), c2 (4096 patches), c3 (4096 patches),
       c4 (a 2-image configs[4] slice), m1 (matcher), s1 (feature selection)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import paper_2108_08380_b200 as bd
import synth


def _bytes(w):
    return bd.bits_to_bytes(w)


def c0():
    c = synth.CONFIGS[0]
    img = synth.image(0, 0, c["H"], c["W"])
    kp = synth.keypoints_as_array(synth.config_keypoints(0, 0))
    pairs, radii, thr = synth.bad_tests(0, 256)
    out = bd.bad_compute(bd.BadModel(pairs, radii, thr), torch.from_numpy(img).cuda(), torch.from_numpy(kp).cuda())
    torch.cuda.synchronize()
    assert (_bytes(out) == oracle.bad_image(img, kp, pairs, radii, thr)).all()


def c1s():
    c = synth.CONFIGS[1]
    img = synth.image(1, 0, c["H"], c["W"])
    kp = synth.keypoints_random_batch(1, [0], 300, c["H"], c["W"], c["margin"], c["scale_max"])
    pairs, radii, thr = synth.bad_tests(1, 512)
    out = bd.bad_compute(bd.BadModel(pairs, radii, thr), torch.from_numpy(img).cuda(), torch.from_numpy(kp).cuda())
    torch.cuda.synchronize()
    assert (_bytes(out) == oracle.bad_image(img, kp, pairs, radii, thr)).all()


def c2():
    P = synth.patches(2, range(4096 + 17))
    pairs, radii, thr = synth.bad_tests(2, 256)
    out = bd.bad_compute_patches(bd.BadModel(pairs, radii, thr), torch.from_numpy(P).cuda())
    torch.cuda.synchronize()
    assert (_bytes(out) == oracle.bad_patches(P, pairs, radii, thr)).all()
    pairs, radii, thr = synth.bad_tests(22, 512)
    out = bd.bad_compute_patches(bd.BadModel(pairs, radii, thr), torch.from_numpy(P).cuda())
    torch.cuda.synchronize()
    assert (_bytes(out) == oracle.bad_patches(P, pairs, radii, thr)).all()


def c3():
    P = synth.patches(3, range(4096 + 17))
    B = synth.hashsift_matrix(3, 256)
    out = bd.hashsift_compute_patches(bd.HashSiftModel(B), torch.from_numpy(P).cuda())
    torch.cuda.synchronize()
    ref, proj = oracle.project(oracle.sift(P), B, want_proj=True)
    mism = np.unpackbits(_bytes(out), axis=1, bitorder="little") != np.unpackbits(ref, axis=1, bitorder="little")
    assert not (mism & (np.abs(proj) >= 1e-3)).any()


def c4():
    c = synth.CONFIGS[4]
    H, W, per = c["H"], c["W"], c["kp_per_image"]
    imgs = synth.images(4, range(2), H, W)
    kp = synth.keypoints_random_batch(4, range(2), per, H, W, c["margin"], c["scale_max"])
    kpi = np.repeat(np.arange(2, dtype=np.int32), per)
    pairs, radii, thr = synth.bad_tests(4, 512)
    B = synth.hashsift_matrix(4, 256)
    ob, oh = bd.describe_warped(bd.BadModel(pairs, radii, thr), bd.HashSiftModel(B), torch.from_numpy(imgs).cuda(),
                                torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda())
    torch.cuda.synchronize()
    P = oracle.warp_nn(imgs, kp, kp_image=kpi)
    assert (_bytes(ob) == oracle.bad_patches(P, pairs, radii, thr)).all()


def m1():
    rng = np.random.default_rng(5)
    n, K = 700, 512
    b = rng.integers(0, 2 ** 32, size=(2 * n, K // 32), dtype=np.uint64).astype(np.uint32)
    a = b.copy()
    a[:, 3] ^= np.uint32(0x10101)
    off = np.array([0, n, 2 * n], np.int64)
    r = bd.match_hamming(torch.from_numpy(a.view(np.int32)).cuda(), torch.from_numpy(b.view(np.int32)).cuda(),
                         off, off, K)
    torch.cuda.synchronize()
    assert (r["nn_ab"].cpu().numpy() == np.tile(np.arange(n), 2)).all()


def s1():
    N = 500
    P = synth.patches(7, range(3 * N))
    trip = np.stack([np.arange(N), N + np.arange(N), 2 * N + np.arange(N)], 1).astype(np.int32)
    rng = np.random.default_rng(6)
    sap = (2 * rng.integers(0, 5, N) - 4).astype(np.int32)
    san = (2 * rng.integers(0, 5, N) - 4).astype(np.int32)
    pairs, radii, _ = synth.bad_tests(9, 64, rmin=0, rmax=7)
    loss, bucket = bd.select_features(torch.from_numpy(P).cuda(), torch.from_numpy(trip).cuda(),
                                      torch.from_numpy(sap).cuda(), torch.from_numpy(san).cuda(), 4, pairs, radii)
    torch.cuda.synchronize()
    rl, rb = oracle.select_features(P, trip, sap, san, 4, pairs, radii)
    assert (loss.cpu().numpy() == rl).all() and (bucket.cpu().numpy() == rb).all()


if __name__ == "__main__":
    for name in sys.argv[1:]:
        globals()[name]()
        print(f"{name}: ok", flush=True)
