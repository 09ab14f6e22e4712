"""GPU parity of the NEXT-1 matcher (bd_match_hamming, tcgen05 kind::mxf4 +-1 GEMM) against the
oracle: nearest-neighbour indices and distances bit-exact (integer work), ties -> lowest index,
mutual flags, ragged sizes, several pairs per call."""
import numpy as np
import pytest

import oracle

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


def _bits(n, K, rng):
    return rng.integers(0, 2**32, size=(n, K // 32), dtype=np.uint64).astype(np.uint32)


def _near(x, flips, rng):
    """copies of x with `flips` random bits flipped (makes NN structure non-trivial)"""
    y = x.copy()
    K = x.shape[1] * 32
    for r in range(len(y)):
        for k in rng.choice(K, flips, replace=False):
            y[r, k // 32] ^= np.uint32(1 << (k % 32))
    return y


def _run(torch, bd, a, a_off, b, b_off, K):
    ta = torch.from_numpy(a.view(np.int32)).cuda()
    tb = torch.from_numpy(b.view(np.int32)).cuda()
    r = bd.match_hamming(ta, tb, a_off, b_off, K)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in r.items()}


@pytest.mark.parametrize("na,nb,K", [(1, 1, 32), (5, 300, 64), (127, 129, 256), (300, 257, 512), (1000, 1000, 512),
                                     (200, 3, 96), (333, 450, 160), (257, 225, 320), (90, 700, 480)])
def test_single_pair(torch, bd, na, nb, K):
    rng = np.random.default_rng(na * 7 + nb + K)
    b = _bits(nb, K, rng)
    a = _near(b[rng.integers(0, nb, na)], K // 16, rng)
    r = _run(torch, bd, a, [0, na], b, [0, nb], K)
    nn, dist = oracle.match(a, [0, na], b, [0, nb], K)
    nn2, dist2 = oracle.match(b, [0, nb], a, [0, na], K)
    assert (r["nn_ab"] == nn).all() and (r["dist_ab"] == dist).all()
    assert (r["nn_ba"] == nn2).all() and (r["dist_ba"] == dist2).all()
    assert (r["mutual"] == oracle.mutual(nn, nn2, [0, na], [0, nb])).all()


def test_ties_and_duplicates(torch, bd):
    rng = np.random.default_rng(9)
    K = 256
    base = _bits(40, K, rng)
    b = np.concatenate([base, base, base[::-1]])     # every train appears 3 times
    a = np.concatenate([base, _near(base, 3, rng)])
    r = _run(torch, bd, a, [0, len(a)], b, [0, len(b)], K)
    nn, dist = oracle.match(a, [0, len(a)], b, [0, len(b)], K)
    assert (r["nn_ab"] == nn).all() and (r["dist_ab"] == dist).all()
    assert (r["nn_ab"][:40] == np.arange(40)).all()  # exact duplicates: lowest index wins


def test_many_pairs(torch, bd):
    rng = np.random.default_rng(10)
    K = 512
    sizes = [(130, 260), (1, 5), (400, 129), (77, 77), (256, 1)]
    a_off = np.cumsum([0] + [s[0] for s in sizes])
    b_off = np.cumsum([0] + [s[1] for s in sizes])
    b = _bits(int(b_off[-1]), K, rng)
    a = np.concatenate([_near(b[b_off[p] + rng.integers(0, sizes[p][1], sizes[p][0])], 20, rng)
                        for p in range(len(sizes))])
    r = _run(torch, bd, a, a_off, b, b_off, K)
    nn, dist = oracle.match(a, a_off, b, b_off, K)
    nn2, _ = oracle.match(b, b_off, a, a_off, K)
    assert (r["nn_ab"] == nn).all() and (r["dist_ab"] == dist).all() and (r["nn_ba"] == nn2).all()
    assert (r["mutual"] == oracle.mutual(nn, nn2, a_off, b_off)).all()


def test_ties_across_halves_and_tiles(torch, bd):
    """A query's exact duplicates planted in both column halves of a 256-row train tile
    (held by the two CTAs of a pair) and in later tiles: the lowest index must win whichever
    half or tile it sits in (the halves merge with an explicit index tie-break)."""
    rng = np.random.default_rng(11)
    K = 64
    b = _bits(1100, K, rng)
    q = _bits(6, K, rng)
    plants = [[100, 200, 300, 500], [130, 300, 1000], [255, 256, 700], [256, 511, 512], [600, 1099], [5, 1050]]
    for i, pos in enumerate(plants):
        for p in pos:
            b[p] = q[i]
    a = np.concatenate([q, _near(q, 2, rng)])
    r = _run(torch, bd, a, [0, len(a)], b, [0, len(b)], K)
    nn, dist = oracle.match(a, [0, len(a)], b, [0, len(b)], K)
    nn2, dist2 = oracle.match(b, [0, len(b)], a, [0, len(a)], K)
    assert (r["nn_ab"][:6] == [pos[0] for pos in plants]).all() and (r["dist_ab"][:6] == 0).all()
    assert (r["nn_ab"] == nn).all() and (r["dist_ab"] == dist).all()
    assert (r["nn_ba"] == nn2).all() and (r["dist_ba"] == dist2).all()


def test_many_work_items(torch, bd):
    """More 256-row query tiles than CTA pairs (74 on a B200): every pair loops over several
    items in both directions, with the query tile double buffered across items."""
    rng = np.random.default_rng(12)
    K = 128
    sizes = [(int(rng.integers(1, 600)), int(rng.integers(1, 600))) for _ in range(160)]
    a_off = np.cumsum([0] + [s[0] for s in sizes])
    b_off = np.cumsum([0] + [s[1] for s in sizes])
    b = _bits(int(b_off[-1]), K, rng)
    a = np.concatenate([_near(b[b_off[p] + rng.integers(0, sizes[p][1], sizes[p][0])], 6, rng)
                        for p in range(len(sizes))])
    r = _run(torch, bd, a, a_off, b, b_off, K)
    nn, dist = oracle.match(a, a_off, b, b_off, K)
    nn2, dist2 = oracle.match(b, b_off, a, a_off, K)
    assert (r["nn_ab"] == nn).all() and (r["dist_ab"] == dist).all()
    assert (r["nn_ba"] == nn2).all() and (r["dist_ba"] == dist2).all()
    assert (r["mutual"] == oracle.mutual(nn, nn2, a_off, b_off)).all()


def test_one_direction(torch, bd):
    """mutual=False: only a -> b is computed (the work list holds direction 0 only)."""
    rng = np.random.default_rng(13)
    K = 512
    b = _bits(900, K, rng)
    a = _near(b[rng.integers(0, 900, 700)], 30, rng)
    ta = torch.from_numpy(a.view(np.int32)).cuda()
    tb = torch.from_numpy(b.view(np.int32)).cuda()
    r = bd.match_hamming(ta, tb, [0, 300, 700], [0, 450, 900], K, mutual=False)
    torch.cuda.synchronize()
    assert set(r) == {"nn_ab", "dist_ab"}
    nn, dist = oracle.match(a, [0, 300, 700], b, [0, 450, 900], K)
    assert (r["nn_ab"].cpu().numpy() == nn).all() and (r["dist_ab"].cpu().numpy() == dist).all()
