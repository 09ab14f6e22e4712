"""Pins for the NEXT-4 feature-selection oracle (or_select_features; Alg. 1 lines 4-12 and
Alg. 2; readings R29-R31).

* L* of every candidate equals the loss evaluated BY DEFINITION (or_feature_loss_at: h = +1 iff
  f <= theta, Eq. 2 summed over triplets) at the threshold the sweep reports, and no other
  threshold realisable on the bucket grid (or at -inf / +inf) does better (brute force).
* Integer-valued features (radius-0 boxes: f = pixel difference): the bucketed optimum equals
  the exact optimum over all real thresholds (SPEC: "with precision 0.1 and integer-valued
  features, exactly matches find_threshold").
* SPEC's worked example (one triplet, f = 0, 1, 10, tau = 1 -> L* = 0 with theta in [1, 10)).
* Zero-margin / cancellation cases of Eq. 2 and thread-count invariance."""
import numpy as np

import oracle
import synth


def _problem(seed, M=90, N=40, J=25, t=7, tau=3, rmax=3):
    rng = np.random.default_rng(seed)
    P = synth.patches(seed, range(M))
    trip = rng.integers(0, M, size=(N, 3)).astype(np.int32)
    # prior similarities: sums of t-1 products of +-1 -> parity of t-1
    sap = (2 * rng.integers(0, t, N) - (t - 1)).astype(np.int32)
    san = (2 * rng.integers(0, t, N) - (t - 1)).astype(np.int32)
    pairs, radii, _ = synth.bad_tests(seed, 32 * ((J + 31) // 32), rmin=0, rmax=rmax)
    return P, trip, sap, san, tau, pairs[:J], radii[:J]


def test_sweep_loss_equals_definition_and_brute_force():
    P, trip, sap, san, tau, pairs, radii = _problem(1)
    loss, bucket = oracle.select_features(P, trip, sap, san, tau, pairs, radii)
    for j in range(len(radii)):
        th = oracle.bucket_theta(bucket[j])
        assert loss[j] == oracle.feature_loss_at(P, trip, sap, san, tau, pairs[j], radii[j], th)
        # brute force over every bucket edge that holds a feature value, plus -inf and +inf
        vals = set()
        for q in trip.reshape(-1):
            S = []
            for k in (0, 2):
                x, y, r = 16 + pairs[j][k], 16 + pairs[j][k + 1], radii[j]
                box = P[q][max(y - r, 0):min(y + r, 31) + 1, max(x - r, 0):min(x + r, 31) + 1]
                S.append((int(box.sum()), box.size))
            f = S[0][0] / S[0][1] - S[1][0] / S[1][1]
            vals.add(int(np.floor((f + 255) * 10 + 1e-9)))
        cands = [-np.inf, np.inf] + [oracle.bucket_theta(b) for b in vals]
        bf = min(oracle.feature_loss_at(P, trip, sap, san, tau, pairs[j], radii[j], th) for th in cands)
        assert loss[j] == bf, (j, loss[j], bf)


def test_integer_features_match_exact_optimum():
    P, trip, sap, san, tau, pairs, _ = _problem(2, rmax=0)
    radii = np.zeros(len(pairs), np.uint8)
    loss, bucket = oracle.select_features(P, trip, sap, san, tau, pairs, radii)
    for j in range(len(radii)):
        vals = {int(P[q][16 + pairs[j][1], 16 + pairs[j][0]]) - int(P[q][16 + pairs[j][3], 16 + pairs[j][2]])
                for q in trip.reshape(-1)}
        exact = min(oracle.feature_loss_at(P, trip, sap, san, tau, pairs[j], 0, th)
                    for th in [-np.inf] + sorted(float(v) for v in vals))
        assert loss[j] == exact


def test_spec_worked_example():
    # f(a) = 0, f(p) = 1, f(n) = 10 with radius-0 boxes at offsets (0,0) and (1,0)
    P = np.full((3, 32, 32), 100, np.uint8)
    P[1, 16, 16] = 101
    P[2, 16, 16] = 110
    pairs = np.array([[0, 0, 1, 0]], np.int8)
    loss, bucket = oracle.select_features(P, [[0, 1, 2]], [0], [0], 1, pairs, np.array([0], np.uint8))
    assert loss[0] == 0
    th = oracle.bucket_theta(bucket[0])
    assert 1 <= th < 10


def test_eq2_cancellation_and_zero_margin():
    P, trip, sap, san, tau, pairs, radii = _problem(3)
    # identical members: h_a h_p = h_a h_n for every theta -> loss = sum [tau - S_ap + S_an]_+ for all theta
    same = np.stack([trip[:, 0]] * 3, 1)
    loss, bucket = oracle.select_features(P, same, sap, san, tau, pairs, radii)
    base = np.maximum(0, tau - sap.astype(np.int64) + san).sum()
    assert (loss == base).all() and (bucket == -1).all()
    # the optimum is never worse than the constant bits (-inf and +inf)
    loss, _ = oracle.select_features(P, trip, sap, san, tau, pairs, radii)
    for j in range(len(radii)):
        for th in (-np.inf, np.inf):
            assert loss[j] <= oracle.feature_loss_at(P, trip, sap, san, tau, pairs[j], radii[j], th)


def test_thread_invariance():
    P, trip, sap, san, tau, pairs, radii = _problem(4)
    a = oracle.select_features(P, trip, sap, san, tau, pairs, radii, nthreads=1)
    b = oracle.select_features(P, trip, sap, san, tau, pairs, radii, nthreads=4)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
