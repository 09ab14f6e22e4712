"""Pins for the SIFT / HashSIFT oracle (or_sift, or_project, or_hashsift_patches).

The paper only says "SIFT" and prints no SIFT values, so the conventions (R10)
are pinned by closed forms and exact invariants: the zero rule, a step edge
(closed-form 1-D sums), a single bright pixel (hand-placed trilinear weights),
90-degree rotation and mirror permutations, contrast invariance, and the projection
special cases of P:242 / S:436-441 (W = 0, signed identity rows).
"""
import math

import numpy as np
import pytest

import oracle
import synth


def tri(c, k):
    return max(0.0, 1.0 - abs(c - k))


def gauss1(t):
    return math.exp(-((t - 15.5) ** 2) / 512.0)


def step_edge(bright_right=True, vertical=True):
    P = np.zeros((32, 32), np.uint8)
    if vertical:
        if bright_right:
            P[:, 16:] = 255
        else:
            P[:, :16] = 255
    else:
        P[16:, :] = 255
    return P


def test_constant_patch_is_zero():
    v, raw = oracle.sift(np.full((2, 32, 32), 93, np.uint8), want_raw=True)
    assert (v == 0).all() and (raw == 0).all()


def test_vertical_step_edge_closed_form():
    v, raw = oracle.sift(step_edge()[None], want_raw=True)
    v, raw = v[0], raw[0]
    # gx = 255 at columns 15 and 16 (central difference, not halved), gy = 0, theta = 0 -> o = 0.
    # tri_x(15, cell 1) + tri_x(16, cell 1) = 0.5625 + 0.4375 = 1 (cells 1 and 2 alike)
    gx = math.exp(-0.25 / 512.0)
    R = [sum(gauss1(y) * tri((y - 3.5) / 8.0, j) for y in range(32)) for j in range(4)]
    expect = np.zeros(128)
    for j in range(4):
        for i in (1, 2):
            expect[(j * 4 + i) * 8 + 0] = 255.0 * gx * R[j]
    np.testing.assert_allclose(raw, expect, rtol=1e-12, atol=1e-9)
    # after clip (all 8 pre-clip values > 0.2) and renormalisation: 8 entries of 1/sqrt(8)
    nz = [(j * 4 + i) * 8 for j in range(4) for i in (1, 2)]
    np.testing.assert_allclose(v[nz], 1 / math.sqrt(8), rtol=1e-12)
    assert np.count_nonzero(v) == 8
    # pre-clip values (clip disabled): R0/N and R1/N, N = sqrt(4 R0^2 + 4 R1^2)
    u = oracle.sift(step_edge()[None], clip=2.0)[0]
    N = math.sqrt(4 * R[0] ** 2 + 4 * R[1] ** 2)
    assert abs(u[(0 * 4 + 1) * 8] - R[0] / N) < 1e-12 and abs(u[(1 * 4 + 1) * 8] - R[1] / N) < 1e-12
    assert abs(R[0] / N - 0.2905) < 1e-4 and abs(R[1] / N - 0.4070) < 1e-4


def test_edge_orientations():
    for P, o in ((step_edge(bright_right=False), 4), (step_edge(vertical=False), 2)):
        v = oracle.sift(P[None])[0].reshape(16, 8)
        assert v[:, o].sum() > 0 and np.allclose(np.delete(v, o, axis=1), 0)


# single bright pixel at (y0, x0) = (11, 10): 4 gradient pixels, hand-placed contributions
# (pixel y, x, orientation bin, m = 255):
#   (11,  9): gx=+255 -> theta 0     -> o 0     (11, 11): gx=-255 -> theta pi   -> o 4
#   (10, 10): gy=+255 -> theta pi/2  -> o 2     (12, 10): gy=-255 -> theta 3pi/2 -> o 6
# cell weights: cx = (x-3.5)/8, cy = (y-3.5)/8 (R10):
#   x= 9: cx=0.6875 -> i0 0.3125, i1 0.6875     x=10: cx=0.8125 -> i0 0.1875, i1 0.8125
#   x=11: cx=0.9375 -> i0 0.0625, i1 0.9375
#   y=10: cy=0.8125 -> j0 0.1875, j1 0.8125     y=11: cy=0.9375 -> j0 0.0625, j1 0.9375
#   y=12: cy=1.0625 -> j1 0.9375, j2 0.0625
SINGLE = [  # (y, x, o, {i: wx}, {j: wy})
    (11, 9, 0, {0: 0.3125, 1: 0.6875}, {0: 0.0625, 1: 0.9375}),
    (11, 11, 4, {0: 0.0625, 1: 0.9375}, {0: 0.0625, 1: 0.9375}),
    (10, 10, 2, {0: 0.1875, 1: 0.8125}, {0: 0.1875, 1: 0.8125}),
    (12, 10, 6, {0: 0.1875, 1: 0.8125}, {1: 0.9375, 2: 0.0625}),
]


def test_single_pixel_trilinear_weights():
    P = np.zeros((32, 32), np.uint8)
    P[11, 10] = 255
    _, raw = oracle.sift(P[None], want_raw=True)
    expect = np.zeros(128)
    for y, x, o, wxs, wys in SINGLE:
        g = math.exp(-((x - 15.5) ** 2 + (y - 15.5) ** 2) / 512.0)
        for i, wx in wxs.items():
            for j, wy in wys.items():
                expect[(j * 4 + i) * 8 + o] += 255.0 * g * wx * wy
    np.testing.assert_allclose(raw[0], expect, rtol=1e-12, atol=1e-12)


def test_orientation_interpolation_half_bin():
    # gx = gy everywhere inside a diagonal ramp -> theta = 45 deg -> co = 1 exactly (bin 1 only);
    # P = 4x + 2y would give theta = atan2(1,2)... use the exact 45-degree case + 22.5 via mirror
    y, x = np.mgrid[0:32, 0:32]
    P = (3 * x + 3 * y + 20).astype(np.uint8)
    _, raw = oracle.sift(P[None], want_raw=True)
    raw = raw[0].reshape(16, 8)
    # interior pixels put all their mass in bin 1; border pixels (one-sided) have angles
    # atan2(6,3) or atan2(3,6): 63.4 / 26.6 deg -> bins 1-2 / 0-1.  Nothing in bins 3..7.
    assert np.allclose(raw[:, 3:], 0)
    assert raw[:, 1].sum() > 10 * (raw[:, 0].sum() + raw[:, 2].sum())


def _rot90_perm():
    # Q = np.rot90(P): Q[i, j] = P[j, 31 - i]; (gxQ, gyQ) = (gyP, -gxP) -> thetaQ = thetaP - 90deg;
    # cells: P cell (jp, ip) = (iq, 3 - jq); bins: oP = oQ + 2
    perm = np.zeros(128, int)
    for jq in range(4):
        for iq in range(4):
            for oq in range(8):
                jp, ip, op = iq, 3 - jq, (oq + 2) % 8
                perm[(jq * 4 + iq) * 8 + oq] = (jp * 4 + ip) * 8 + op
    return perm


def test_rot90_is_a_fixed_permutation():
    P = synth.patches(21, range(8))
    v = oracle.sift(P)
    q = oracle.sift(np.stack([np.rot90(p) for p in P]))
    np.testing.assert_allclose(q, v[:, _rot90_perm()], atol=1e-12)


def test_horizontal_mirror():
    P = synth.patches(22, range(8))
    v = oracle.sift(P)
    q = oracle.sift(P[:, :, ::-1])
    perm = np.zeros(128, int)
    for j in range(4):
        for i in range(4):
            for o in range(8):
                perm[(j * 4 + i) * 8 + o] = (j * 4 + 3 - i) * 8 + (4 - o) % 8
    np.testing.assert_allclose(q, v[:, perm], atol=1e-12)


def test_contrast_invariance_and_unit_norm():
    P = synth.patches(23, range(16)).astype(np.int32)
    P = np.clip(P, 64, 191)
    v = oracle.sift(P.astype(np.uint8))
    w = oracle.sift((2 * P - 128).astype(np.uint8))
    np.testing.assert_allclose(v, w, atol=1e-12)
    n = np.linalg.norm(v, axis=1)
    assert np.all(np.abs(n - 1) < 1e-12)
    # R11: entries <= 0.2 before renormalisation -> after it, max <= 0.2 * (renorm factor)
    u = oracle.sift(P.astype(np.uint8), clip=2.0)
    pre = np.minimum(u, 0.2)
    np.testing.assert_allclose(v, pre / np.linalg.norm(pre, axis=1, keepdims=True), atol=1e-12)


def test_projection_special_cases():
    rng = np.random.default_rng(5)
    v = oracle.sift(synth.patches(24, range(10)))
    N = 256
    # W = 0 -> bits = [b >= 0], including b == 0 exactly (sgn(0) = +1)
    B = np.zeros((N, 129), np.float32)
    B[:, 128] = rng.standard_normal(N).astype(np.float32)
    B[:5, 128] = 0.0
    bits = np.unpackbits(oracle.project(v, B), axis=1, bitorder="little")
    assert (bits == (B[:, 128] >= 0)[None, :]).all()
    # signed identity rows: p_k = s_k * v_{k mod 128}, v >= 0 -> bit = 1 if s = +1 else [v == 0]
    B = np.zeros((N, 129), np.float32)
    s = np.where(np.arange(N) < 128, 1.0, -1.0)
    B[np.arange(N), np.arange(N) % 128] = s
    bits = np.unpackbits(oracle.project(v, B), axis=1, bitorder="little")
    expect = np.concatenate([np.ones((10, 128)), (v == 0)], axis=1)
    assert (bits == expect).all()
    # constant patch -> bits = sgn(bias)
    B = synth.hashsift_matrix(3, N)
    c = oracle.hashsift_patches(np.full((1, 32, 32), 50, np.uint8), B)
    assert (np.unpackbits(c, bitorder="little") == (B[:, 128] >= 0)).all()


def test_projection_against_numpy_float64():
    v = oracle.sift(synth.patches(25, range(64)))
    B = synth.hashsift_matrix(25, 256)
    bits, proj = oracle.project(v, B, want_proj=True)
    ref = v @ B[:, :128].astype(np.float64).T + B[:, 128].astype(np.float64)
    np.testing.assert_allclose(proj, ref, atol=1e-13)
    assert (np.unpackbits(bits, axis=1, bitorder="little") == (proj >= 0)).all()
    assert (oracle.hashsift_patches(synth.patches(25, range(64)), B) == bits).all()


def test_sift_thread_invariance():
    P = synth.patches(26, range(100))
    assert (oracle.sift(P, nthreads=1) == oracle.sift(P, nthreads=8)).all()
