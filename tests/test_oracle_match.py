"""Pins for the NEXT-1 matcher oracle (or_match).

The oracle counts differing bits one by one; these tests pin it against independent
computations (numpy unpackbits + argmin, whose first-occurrence rule is the S:530 tie rule),
the closed forms a = b -> 0 and complement -> K, the similarity identity of P:123
(h(x)^T h(y) = K - 2 Hamming with h in {-1,+1}^K) and SPEC's mutual-NN asymmetry example
(S:536)."""
import numpy as np
import pytest

import oracle


def _bits(n, K, rng):
    return rng.integers(0, 2**32, size=(n, K // 32), dtype=np.uint64).astype(np.uint32)


def _dmat(a, b, K):
    ua = np.unpackbits(a.view(np.uint8), axis=1, bitorder="little")[:, :K].astype(np.int64)
    ub = np.unpackbits(b.view(np.uint8), axis=1, bitorder="little")[:, :K].astype(np.int64)
    return (ua[:, None, :] != ub[None, :, :]).sum(-1)


@pytest.mark.parametrize("K", [32, 64, 256, 512])
def test_nn_equals_numpy_argmin(K):
    rng = np.random.default_rng(K)
    a, b = _bits(57, K, rng), _bits(43, K, rng)
    nn, dist = oracle.match(a, [0, 57], b, [0, 43], K)
    D = _dmat(a, b, K)
    assert (nn == D.argmin(1)).all() and (dist == D.min(1)).all()


def test_self_and_complement():
    rng = np.random.default_rng(1)
    K = 256
    a = _bits(40, K, rng)
    nn, dist = oracle.match(a, [0, 40], a, [0, 40], K)
    assert (dist == 0).all() and (nn == np.arange(40)).all()
    nn, dist = oracle.match(a, [0, 40], ~a, [0, 40], K)
    D = _dmat(a, ~a, K)
    assert (np.diag(D) == K).all() and (dist == D.min(1)).all()


def test_ties_lowest_index():
    rng = np.random.default_rng(2)
    K = 64
    q = _bits(1, K, rng)
    b = np.repeat(_bits(1, K, rng), 5, axis=0)   # five identical trains
    nn, dist = oracle.match(q, [0, 1], b, [0, 5], K)
    assert nn[0] == 0
    b[3] = q[0]                                  # one exact match -> chosen
    nn, dist = oracle.match(q, [0, 1], b, [0, 5], K)
    assert nn[0] == 3 and dist[0] == 0


def test_similarity_identity():
    rng = np.random.default_rng(3)
    K = 512
    a, b = _bits(20, K, rng), _bits(30, K, rng)
    ha = 2 * np.unpackbits(a.view(np.uint8), axis=1, bitorder="little")[:, :K].astype(np.int64) - 1
    hb = 2 * np.unpackbits(b.view(np.uint8), axis=1, bitorder="little")[:, :K].astype(np.int64) - 1
    S = ha @ hb.T
    nn, dist = oracle.match(a, [0, 20], b, [0, 30], K)
    assert (dist == (K - S.max(1)) // 2).all() and (nn == S.argmax(1)).all()


def test_mutual_asymmetry_example():
    # q0 -> t0 but t0's NN is q1 -> q0 unmatched
    K = 32
    t0 = np.uint32(0)
    q1 = np.uint32(0)            # identical to t0
    q0 = np.uint32(0b1)          # one bit from t0
    a = np.array([[q0], [q1]], np.uint32)
    b = np.array([[t0], [np.uint32(0xFFFFFFFF)]], np.uint32)
    nn_ab, _ = oracle.match(a, [0, 2], b, [0, 2], K)
    nn_ba, _ = oracle.match(b, [0, 2], a, [0, 2], K)
    assert list(nn_ab) == [0, 0] and nn_ba[0] == 1
    assert list(oracle.mutual(nn_ab, nn_ba, [0, 2], [0, 2])) == [0, 1]


def test_pairs_are_independent_and_relative():
    rng = np.random.default_rng(4)
    K = 128
    a1, a2, b1, b2 = _bits(9, K, rng), _bits(7, K, rng), _bits(5, K, rng), _bits(11, K, rng)
    nn, dist = oracle.match(np.concatenate([a1, a2]), [0, 9, 16], np.concatenate([b1, b2]), [0, 5, 16], K)
    n1, d1 = oracle.match(a1, [0, 9], b1, [0, 5], K)
    n2, d2 = oracle.match(a2, [0, 7], b2, [0, 11], K)
    assert (nn == np.concatenate([n1, n2])).all() and (dist == np.concatenate([d1, d2])).all()
