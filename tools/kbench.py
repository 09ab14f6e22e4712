#!/usr/bin/env python
"""Per-workload device timing of the C-ABI entry points (configs[1], [2], [3], [4-slice]).

  python tools/kbench.py [--which c0,c1,c2,c3,c4] [--reps 10]

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
from bench import ClockSampler  # NVML SM-clock / throttle-reason sampling (the bench's)

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


LAST = {}  # median / best of the last timeit (report median and best)


def timeit(fn, reps):
    """3 warm-ups, then `reps` back-to-back calls between two events (the reported mean, the
    figure the bench's per-step numbers compare with), plus each call timed on its own for the
    median and the best."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bd.profile_start()
    with ClockSampler(torch.cuda.current_device()) as clk:  # clocks during the timed calls
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
    prof = bd.profile_stop()
    LAST["clocks"] = clk.summary()
    ms = e0.elapsed_time(e1) / reps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    each = sorted(a.elapsed_time(b) for a, b in ev)
    LAST.update(median=round(each[len(each) // 2], 4), best=round(each[0], 4))
    return ms, {k: round(v[1] / reps, 4) for k, v in prof.items()}


def report(name, ms, prof, n_desc, alg_bytes):
    r = {"workload": name, "ms": round(ms, 4), "ms_median": LAST.get("median"), "ms_best": LAST.get("best"),
         "Mdesc_s": round(n_desc / ms / 1e3, 2),
         "alg_GBps": round(alg_bytes / ms / 1e6, 1), "hbm_frac": round(alg_bytes / ms / 1e6 / HBM, 4),
         "kernels_ms": prof, "clocks": LAST.get("clocks")}
    print(json.dumps(r), flush=True)
    return r


def c0(reps, n_lat=200):
    """configs[0] (one 640x480 image, 500 kp, BAD-256): a latency workload.
    Reports the device time of ONE bad_compute call (integral + bad_image, median of n_lat
    calls each bracketed by events on an idle stream), the same call replayed from a CUDA
    graph (launch overhead amortised by the graph), and back-to-back throughput."""
    c = synth.CONFIGS[0]
    img = torch.from_numpy(synth.image(0, 0, c["H"], c["W"])).cuda()
    kp = torch.from_numpy(synth.keypoints_as_array(synth.config_keypoints(0, 0))).cuda()
    m = bd.BadModel(*synth.bad_tests(0, 256))
    out = torch.empty((kp.shape[0], 8), dtype=torch.int32, device="cuda")
    fn = lambda: bd.bad_compute(m, img, kp, None, out=out)  # noqa: E731
    ms, prof = timeit(fn, reps)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()

    def lat(call):
        t = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(n_lat):
            torch.cuda.synchronize()
            e0.record()
            call()
            e1.record()
            e1.synchronize()
            t.append(e0.elapsed_time(e1) * 1e3)
        return float(np.median(t))

    us_call = lat(fn)
    us_graph = lat(g.replay)
    r = {"workload": "c0 BAD-256 one 640x480 image, 500 kp (latency)", "ms": round(ms, 4),
         "Mdesc_s": round(kp.shape[0] / ms / 1e3, 3), "latency_us": round(us_call, 2),
         "graph_latency_us": round(us_graph, 2), "kernels_ms": prof, "clocks": LAST.get("clocks")}
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


def c4b(reps):
    return c4(reps, mode="bilinear")


def c4(reps, n_img=256, mode="nn"):
    c = synth.CONFIGS[4]
    H, W, per = c["H"], c["W"], c["kp_per_image"]
    imgs = sg.images(4, 0, n_img, H, W)
    kp = torch.from_numpy(synth.keypoints_random_batch(4, range(n_img), per, H, W, c["margin"], c["scale_max"])).cuda()
    kpi = torch.from_numpy(np.repeat(np.arange(n_img, dtype=np.int32), per)).cuda()
    mb, mh = bd.BadModel(*synth.bad_tests(4, 512)), bd.HashSiftModel(synth.hashsift_matrix(4, 256))
    m = n_img * per
    ob = torch.empty((m, 16), dtype=torch.int32, device="cuda")
    oh = torch.empty((m, 8), dtype=torch.int32, device="cuda")
    ms, prof = timeit(lambda: bd.describe_warped(mb, mh, imgs, kp, kpi, out_bad=ob, out_hs=oh, mode=mode), reps)
    return report(f"c4 slice ({n_img} images, {mode} warp)", ms, prof, m, m * (2074 + 96))


def m1(reps, n_pairs=64, n=4000, K=512):
    """NEXT-1 matcher: n_pairs image pairs of n x n BAD-512 descriptor sets (near-duplicate
    structure), both NN directions + mutual flags.  Tensor roofline: 2*n*n*K ops per direction
    per pair vs the dense FP4 peak the kernel runs at (tcgen05 kind::mxf4: 4 x the measured bf16
    peak, the guide's nominal 9 / 2.25 PFLOP/s ratio)."""
    rng = np.random.default_rng(5)
    b = rng.integers(0, 2**32, size=(n_pairs * n, K // 32), dtype=np.uint64).astype(np.uint32)
    a = b.copy()
    flips = rng.integers(0, K, size=(a.shape[0], 24))
    for j in range(24):
        a[np.arange(a.shape[0]), flips[:, j] // 32] ^= (np.uint32(1) << (flips[:, j] % 32).astype(np.uint32))
    ta = torch.from_numpy(a.view(np.int32)).cuda()
    tb = torch.from_numpy(b.view(np.int32)).cuda()
    off = np.arange(n_pairs + 1, dtype=np.int64) * n
    ms, prof = timeit(lambda: bd.match_hamming(ta, tb, off, off, K), reps)
    ops = 2.0 * 2 * n * n * K * n_pairs
    peak = 4 * json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6360.0
    r = {"workload": f"m1 match {n_pairs} pairs {n}x{n} K={K} (both directions + mutual)", "ms": round(ms, 4),
         "pairs_per_s": round(n_pairs / ms * 1e3, 1), "TOPS": round(ops / ms / 1e9, 1),
         "tensor_frac": round(ops / ms / 1e9 / peak, 4), "kernels_ms": prof, "clocks": LAST.get("clocks")}
    print(json.dumps(r), flush=True)
    return r


def s1(reps, M=30000, N=10000, J=1000, t=20, tau=4):
    """NEXT-4: one feature-selection iteration: J = 1000 candidates over N triplets of
    3N synthetic patches (positives = the same noise field at another contrast gain)."""
    rng = np.random.default_rng(6)
    units = np.arange(N)
    a = synth.patches(7, units)
    g = synth.patch_gain(8, units)  # a second gain for the positive view of each "3D point"
    p = synth._quantise(synth._fields(7, units, 32, 32), g)
    neg = synth.patches(7, N + rng.permutation(N))
    P = np.concatenate([a, p, neg])[:M]
    trip = np.stack([units, N + units, 2 * N + units], 1).astype(np.int32)
    sap = (2 * rng.integers(0, t, N) - (t - 1)).astype(np.int32)
    san = (2 * rng.integers(0, t, N) - (t - 1)).astype(np.int32)
    pairs, radii, _ = synth.bad_tests(9, J, rmin=0, rmax=7)
    tP, tt = torch.from_numpy(P).cuda(), torch.from_numpy(trip).cuda()
    ta, tn = torch.from_numpy(sap).cuda(), torch.from_numpy(san).cuda()
    ms, prof = timeit(lambda: bd.select_features(tP, tt, ta, tn, tau, pairs, radii), reps)
    r = {"workload": f"s1 feature selection: J={J} candidates x N={N} triplets (M={M} patches)", "ms": round(ms, 4),
         "candidate_triplets_per_s": round(J * N / ms * 1e3 / 1e9, 3), "unit": "G candidate-triplets/s",
         "kernels_ms": prof, "clocks": LAST.get("clocks")}
    print(json.dumps(r), flush=True)
    return r


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="c0,c1,c2,c3,c4,c4b,m1,s1")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    for w in a.which.split(","):
        globals()[w](a.reps)
        torch.cuda.empty_cache()
