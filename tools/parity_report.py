#!/usr/bin/env python
"""Parity report (SURVEY §8(c) "Parity report fields") for every BASELINE config, written as
JSON: the GPU path through the C ABI against the CPU oracle on the same seeded inputs.

  python tools/parity_report.py [--out profiles/parity_r01.json]

BAD: bits compared, mismatches, mismatches on R6-fragile keypoints, exact ties (swap test).
HashSIFT: max SIFT error relative to ||o|| (R14), mismatching bits inside / outside the
|p| < 1e-3 band (R13), band populations at 1e-3 and 1e-4.  Sharding: per-image SHA-256 of
the descriptors computed with the images split over P = 1, 2, 4, 8 shards (the bench's
contiguous ranges; each shard a separate call) must agree.  Large configs are sampled (the
sample is recorded).  Test infrastructure: imports oracle/ (like tests/)."""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2108_08380_b200 as bd  # noqa: E402
import synth  # noqa: E402
import synth.gpu as sg  # noqa: E402


def to_bytes(words):
    w = np.ascontiguousarray(words.cpu().numpy()).view(np.uint32).astype("<u4")
    return w.view(np.uint8).reshape(w.shape[0], -1)


def bad_stats(gpu_words, ref, fragile, ties, K):
    g = to_bytes(gpu_words)
    gb = np.unpackbits(g, axis=1, bitorder="little")[:, :K]
    rb = np.unpackbits(ref, axis=1, bitorder="little")[:, :K]
    mism = gb != rb
    rows_bad = mism.any(1)
    return {"bits_compared": int(gb.size), "mismatches": int(mism.sum()),
            "mismatches_on_fragile_keypoints": int(mism[fragile.astype(bool)].sum()) if fragile is not None else 0,
            "fragile_keypoints": int(fragile.sum()) if fragile is not None else 0,
            "exact_ties": int(ties.sum()) if ties is not None else 0, "rows_differing": int(rows_bad.sum())}


def hs_stats(gpu_words, ref, proj, N, gpu_sift=None, ref_sift=None):
    gb = np.unpackbits(to_bytes(gpu_words), axis=1, bitorder="little")[:, :N]
    rb = np.unpackbits(ref, axis=1, bitorder="little")[:, :N]
    mism = gb != rb
    inside = mism & (np.abs(proj) < 1e-3)
    r = {"bits_compared": int(gb.size), "mismatches": int(mism.sum()), "mismatches_inside_band": int(inside.sum()),
         "mismatches_outside_band": int((mism & ~inside).sum()),
         "band_population_1e-3": float((np.abs(proj) < 1e-3).mean()),
         "band_population_1e-4": float((np.abs(proj) < 1e-4).mean())}
    if gpu_sift is not None:
        g = gpu_sift.cpu().numpy().astype(np.float64)
        nrm = np.linalg.norm(ref_sift, axis=1)
        nz = nrm > 0
        r["max_sift_error_rel"] = float((np.abs(g - ref_sift).max(1)[nz] / nrm[nz]).max())
        r["zero_descriptors_exact"] = bool((g[~nz] == 0).all())
    return r


def c0():
    c = synth.CONFIGS[0]
    img = synth.image(0, 0, c["H"], c["W"])
    kp = synth.keypoints_as_array(synth.config_keypoints(0, 0))
    pairs, radii, thr = synth.bad_tests(0, 256)
    ref, _, fragile, ties = oracle.bad_image(img[None], kp, pairs, radii, thr, want_aux=True)
    out = bd.bad_compute(bd.BadModel(pairs, radii, thr), torch.from_numpy(img).cuda(), torch.from_numpy(kp).cuda())
    return {"config": c["name"], "sample": "all 500 keypoints", "bad": bad_stats(out, ref, fragile, ties, 256)}


def c1(n_check=2):
    c = synth.CONFIGS[1]
    n, H, W, per = c["n_images"], c["H"], c["W"], c["kp_per_image"]
    imgs = sg.images(1, 0, n, H, W)
    kp = synth.keypoints_random_batch(1, range(n), per, H, W, c["margin"], c["scale_max"])
    kpi = np.repeat(np.arange(n, dtype=np.int32), per)
    pairs, radii, thr = synth.bad_tests(1, 512)
    out = bd.bad_compute(bd.BadModel(pairs, radii, thr), imgs, torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda())
    torch.cuda.synchronize()
    agg = None
    for i in (0, n - 1)[:n_check]:
        sl = slice(i * per, (i + 1) * per)
        ref, _, fragile, ties = oracle.bad_image(synth.image(1, i, H, W)[None], kp[sl], pairs, radii, thr,
                                                 want_aux=True)
        s = bad_stats(out[sl], ref, fragile, ties, 512)
        agg = s if agg is None else {k: agg[k] + s[k] for k in s}
    return {"config": c["name"], "sample": f"full launch (64 images); images 0 and {n - 1} checked in full",
            "bad": agg}


def c2(n_sample=20000):
    c = synth.CONFIGS[2]
    n = c["n_patches"]
    P = sg.patches(2, 0, n)
    pairs, radii, thr = synth.bad_tests(2, 256)
    out = bd.bad_compute_patches(bd.BadModel(pairs, radii, thr), P)
    idx = np.random.default_rng(0).choice(n, n_sample, replace=False)
    Ps = synth.patches(2, idx)
    ref = oracle.bad_patches(Ps, pairs, radii, thr)
    return {"config": c["name"], "sample": f"full 4M launch; {n_sample} random patches checked",
            "bad": bad_stats(out[torch.from_numpy(idx).cuda()], ref, None, None, 256)}


def c3(n_sample=20000):
    c = synth.CONFIGS[3]
    n = c["n_patches"]
    P = sg.patches(3, 0, n)
    B = synth.hashsift_matrix(3, 256)
    sift = torch.empty((n, 128), dtype=torch.float32, device="cuda")
    out = bd.hashsift_compute_patches(bd.HashSiftModel(B), P, sift=sift, want_sift=True)[0]
    idx = np.random.default_rng(1).choice(n, n_sample, replace=False)
    v = oracle.sift(synth.patches(3, idx))
    ref, proj = oracle.project(v, B, want_proj=True)
    ti = torch.from_numpy(idx).cuda()
    return {"config": c["name"], "sample": f"full 1M launch; {n_sample} random patches checked",
            "hashsift": hs_stats(out[ti], ref, proj, 256, sift[ti], v)}


def c4(n_img=64, n_check=2):
    c = synth.CONFIGS[4]
    H, W, per = c["H"], c["W"], c["kp_per_image"]
    imgs = sg.images(4, 0, n_img, H, W)
    kp = synth.keypoints_random_batch(4, range(n_img), per, H, W, c["margin"], c["scale_max"])
    kpi = np.repeat(np.arange(n_img, dtype=np.int32), per)
    pairs, radii, thr = synth.bad_tests(4, 512)
    B = synth.hashsift_matrix(4, 256)
    mb, mh = bd.BadModel(pairs, radii, thr), bd.HashSiftModel(B)
    tkp, tki = torch.from_numpy(kp).cuda(), torch.from_numpy(kpi).cuda()
    ob, oh = bd.describe_warped(mb, mh, imgs, tkp, tki)
    torch.cuda.synchronize()
    bad_agg = hs_agg = None
    for i in (0, n_img - 1)[:n_check]:
        sl = slice(i * per, (i + 1) * per)
        P = oracle.warp_nn(synth.image(4, i, H, W), kp[sl])
        s = bad_stats(ob[sl], oracle.bad_patches(P, pairs, radii, thr), None, None, 512)
        ref, proj = oracle.project(oracle.sift(P), B, want_proj=True)
        h = hs_stats(oh[sl], ref, proj, 256)
        bad_agg = s if bad_agg is None else {k: bad_agg[k] + s[k] for k in s}
        hs_agg = h if hs_agg is None else {k: (hs_agg[k] + h[k]) if "population" not in k else max(hs_agg[k], h[k])
                                           for k in h}
    # sharding invariance: the bench's contiguous image ranges, one call per shard
    import bench
    digests = {}
    for P_ in (1, 2, 4, 8):
        per_img = []
        for r in range(P_):
            i0, i1 = bench.shard(n_img, r, P_)
            a, b = i0 * per, i1 * per
            sb, sh = bd.describe_warped(mb, mh, imgs[i0:i1], tkp[a:b], tki[a:b] - i0)
            torch.cuda.synchronize()
            for i in range(i1 - i0):
                q = slice(i * per, (i + 1) * per)
                per_img.append(hashlib.sha256(sb[q].cpu().numpy().tobytes() + sh[q].cpu().numpy().tobytes())
                               .hexdigest())
        digests[P_] = per_img
    agree = all(digests[P_] == digests[1] for P_ in digests)
    return {"config": c["name"], "sample": f"{n_img} images; images 0 and {n_img - 1} checked in full",
            "bad": bad_agg, "hashsift": hs_agg,
            "sharding": {"shards": [1, 2, 4, 8], "images": n_img, "per_image_sha256_agree": agree}}


def m1(n_pairs=64, n=4000, K=512, n_sample=2000):
    """NEXT-1 at the kbench size (tools/kbench.py m1): the full launch, sampled query rows of
    both directions checked against the oracle's brute-force NN (indices, distances, mutual)."""
    rng = np.random.default_rng(5)
    b = rng.integers(0, 2**32, size=(n_pairs * n, K // 32), dtype=np.uint64).astype(np.uint32)
    a = b.copy()
    flips = rng.integers(0, K, size=(a.shape[0], 24))
    for j in range(24):
        a[np.arange(a.shape[0]), flips[:, j] // 32] ^= (np.uint32(1) << (flips[:, j] % 32).astype(np.uint32))
    off = np.arange(n_pairs + 1, dtype=np.int64) * n
    r = bd.match_hamming(torch.from_numpy(a.view(np.int32)).cuda(), torch.from_numpy(b.view(np.int32)).cuda(),
                         off, off, K)
    torch.cuda.synchronize()
    r = {k: v.cpu().numpy() for k, v in r.items()}
    bad = {"nn_ab": 0, "dist_ab": 0, "nn_ba": 0, "dist_ba": 0, "mutual": 0}
    qs = np.random.default_rng(6).choice(n_pairs * n, n_sample, replace=False)
    for q in qs:  # one query row against its pair's train block, both directions
        p = int(q // n)
        for d, (x, y, tag) in enumerate(((a, b, "ab"), (b, a, "ba"))):
            nn, dist = oracle.match(x[q:q + 1], [0, 1], y[p * n:(p + 1) * n], [0, n], K)
            bad["nn_" + tag] += int(r["nn_" + tag][q] != nn[0])
            bad["dist_" + tag] += int(r["dist_" + tag][q] != dist[0])
        j = int(r["nn_ab"][q])
        bad["mutual"] += int(r["mutual"][q] != (r["nn_ba"][p * n + j] == q - p * n))
    return {"config": f"m1 matcher: {n_pairs} pairs of {n} x {n}, K = {K}",
            "sample": f"full launch; {n_sample} random query rows checked in both directions",
            "mismatches": bad}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity.json"))
    a = ap.parse_args()
    rep = {"device": torch.cuda.get_device_name(0), "configs": [c0(), c1(), c2(), c3(), c4(), m1()]}
    json.dump(rep, open(a.out, "w"), indent=1)
    print(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
