"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 bench path.

bench.py shards configs[4] by contiguous image ranges with no data-path collective; the only
collectives are the barrier, the max-over-ranks time and the sum of keypoints.  These tests
run that host logic in two real processes over gloo on 127.0.0.1 and check sharding
invariance: the per-image descriptor digests gathered from the ranks equal the single-process
digests (R21: image i's inputs depend only on (seed, i)).  The descriptors here come from the
CPU oracle on a reduced-size configs[4]-style workload — the GPU path's parity with the oracle
is tested separately (tests/test_gpu_*.py)."""
import os
import socket

import numpy as np
import pytest

import bench
import oracle
import synth

H, W, PER, N_IMG, SEED = 96, 128, 24, 5, 4


def _words(i):
    """image i's descriptors in the GPU path's layout: uint32 words (PER, K/32), LSB-first (R16)
    — BAD-64 and HashSIFT-32 computed by the oracle on a reduced configs[4]-style image."""
    pairs, radii, thr = synth.bad_tests(SEED, 64)
    B = synth.hashsift_matrix(SEED, 32)
    img = synth.image(SEED, i, H, W)
    kp = synth.keypoints_as_array(synth.keypoints_random(SEED, i, PER, H, W, 20, 1.0))
    P = oracle.warp_nn(img, kp, nthreads=1)
    b = oracle.bad_patches(P, pairs, radii, thr, nthreads=1)
    h = oracle.hashsift_patches(P, B, nthreads=1)
    return b.view("<u4"), h.view("<u4")


def _digests(i0, i1):
    """bench.image_digests over the shard's concatenated GPU-shaped output rows (the same
    function bench.py applies to the device outputs)."""
    if i1 <= i0:
        return []
    bw, hw = zip(*[_words(i) for i in range(i0, i1)])
    return bench.image_digests(np.concatenate(bw), np.concatenate(hw), PER)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        i0, i1 = bench.shard(N_IMG, rank, world)
        dig = bench.gather_digests(_digests(i0, i1), i0, world)  # bench.py's all-gather
        ms = bench.allreduce_max(float(10 + rank), world)
        kps = bench.allreduce_sum(float((i1 - i0) * PER), world)
        bench.barrier(world)
        if rank == 0:
            # bench.py's P = 1 check: sampled images recomputed alone on rank 0
            chk = bench.check_sharding(dig, lambda i: bench.image_digests(*_words(i), PER)[0],
                                       bench.sample_images(N_IMG, world))
            q.put((dig, ms, kps, chk))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_partition():
    for n in (1, 5, 8, 8192):
        for world in (1, 2, 3, 4, 8):
            r = [bench.shard(n, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1


def test_two_rank_gloo_sharding_invariance():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    dig, ms, kps, chk = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert dig == _digests(0, N_IMG)     # sharding invariance (R21), in image order
    assert chk["mismatches"] == 0 and chk["checked"] >= 3 and chk["images"] == N_IMG
    assert ms == 11.0                    # max over ranks
    assert kps == N_IMG * PER            # sum over ranks


def test_digest_detects_a_flipped_bit():
    bw, hw = _words(0)
    d0 = bench.image_digests(bw, hw, PER)
    bw2 = bw.copy()
    bw2[3, 1] ^= np.uint32(1 << 7)
    assert bench.image_digests(bw2, hw, PER) != d0
    chk = bench.check_sharding(d0, lambda i: bench.image_digests(bw2, hw, PER)[i], [0])
    assert chk["mismatches"] == 1


def test_sample_images_cover_every_shard_edge():
    for n, world in ((8192, 8), (5, 2), (64, 4)):
        s = bench.sample_images(n, world)
        for r in range(world):
            a, b = bench.shard(n, r, world)
            assert a in s and b - 1 in s
