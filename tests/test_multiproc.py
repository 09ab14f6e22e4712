"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 bench path.

bench.py shards configs[4] by contiguous image ranges with no data-path collective; the only
collectives are the barrier, the max-over-ranks time and the sum of keypoints.  These tests
run that host logic in two real processes over gloo on 127.0.0.1 and check sharding
invariance: the per-image descriptor digests gathered from the ranks equal the single-process
digests (R21: image i's inputs depend only on (seed, i)).  The descriptors here come from the
CPU oracle on a reduced-size configs[4]-style workload — the GPU path's parity with the oracle
is tested separately (tests/test_gpu_*.py)."""
import hashlib
import os
import socket

import numpy as np
import pytest

import bench
import oracle
import synth

H, W, PER, N_IMG, SEED = 96, 128, 24, 5, 4


def _digests(i0, i1):
    """sha256 of (BAD-64 bits, HashSIFT-32 bits) of every keypoint of images [i0, i1)."""
    pairs, radii, thr = synth.bad_tests(SEED, 64)
    B = synth.hashsift_matrix(SEED, 32)
    out = []
    for i in range(i0, i1):
        img = synth.image(SEED, i, H, W)
        kp = synth.keypoints_as_array(synth.keypoints_random(SEED, i, PER, H, W, 20, 1.0))
        P = oracle.warp_nn(img, kp, nthreads=1)
        b = oracle.bad_patches(P, pairs, radii, thr, nthreads=1)
        h = oracle.hashsift_patches(P, B, nthreads=1)
        out.append(hashlib.sha256(b.tobytes() + h.tobytes()).hexdigest())
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        i0, i1 = bench.shard(N_IMG, rank, world)
        dig = _digests(i0, i1)
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, i0, i1, dig))
        ms = bench.allreduce_max(float(10 + rank), world)
        kps = bench.allreduce_sum(float((i1 - i0) * PER), world)
        bench.barrier(world)
        if rank == 0:
            q.put((gathered, ms, kps))
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
    gathered, ms, kps = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered.sort()
    assert [g[0] for g in gathered] == [0, 1]
    assert gathered[0][1] == 0 and gathered[0][2] == gathered[1][1] and gathered[1][2] == N_IMG
    multi = gathered[0][3] + gathered[1][3]
    assert multi == _digests(0, N_IMG)   # sharding invariance (R21)
    assert ms == 11.0                    # max over ranks
    assert kps == N_IMG * PER            # sum over ranks
