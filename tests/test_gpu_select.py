"""GPU parity of NEXT-4 (bd_select_features: one feature-selection iteration, Alg. 1 lines
4-12 + Alg. 2 integer sort) against the oracle: L* and b* of every candidate EXACT (all
arithmetic is integer, R29-R31), at small and benchmark-like sizes, with ties (duplicate
patches, radius-0 integer features) and every radius 0..7."""
import numpy as np
import pytest

import oracle
import synth

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


def _problem(seed, M, N, J, t, tau, rmin=0, rmax=7, dup=False):
    rng = np.random.default_rng(seed)
    P = synth.patches(seed, range(M))
    if dup:
        P[M // 2:] = P[: M - M // 2]       # exact duplicate patches -> tied feature values
    trip = rng.integers(0, M, size=(N, 3)).astype(np.int32)
    sap = (2 * rng.integers(0, t, N) - (t - 1)).astype(np.int32)
    san = (2 * rng.integers(0, t, N) - (t - 1)).astype(np.int32)
    pairs, radii, _ = synth.bad_tests(seed, 32 * ((J + 31) // 32), rmin=rmin, rmax=rmax)
    return P, trip, sap, san, tau, pairs[:J], radii[:J]


@pytest.mark.parametrize("seed,M,N,J,t,tau,rmax,dup", [
    (1, 50, 30, 10, 1, 1, 7, False),
    (2, 600, 400, 70, 9, 3, 7, True),
    (3, 3000, 1000, 150, 25, 5, 0, False),   # integer features (radius 0)
    (4, 30000, 10000, 300, 40, 4, 5, False),  # benchmark-like sizes
])
def test_select_parity(torch, bd, seed, M, N, J, t, tau, rmax, dup):
    P, trip, sap, san, tau, pairs, radii = _problem(seed, M, N, J, t, tau, rmax=rmax, dup=dup)
    ref_loss, ref_b = oracle.select_features(P, trip, sap, san, tau, pairs, radii)
    loss, b = bd.select_features(torch.from_numpy(P).cuda(), torch.from_numpy(trip).cuda(),
                                 torch.from_numpy(sap).cuda(), torch.from_numpy(san).cuda(), tau, pairs, radii)
    torch.cuda.synchronize()
    assert (loss.cpu().numpy() == ref_loss).all()
    assert (b.cpu().numpy() == ref_b).all()
