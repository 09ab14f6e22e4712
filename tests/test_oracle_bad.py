"""Pins for the BAD oracle (oracle/bindesc_oracle.c: or_bad_image, or_bad_patches).

Each test checks the oracle against something other than itself: hand-derived closed
forms (tests/golden/bad_ramp_8x8.txt), special cases the paper fixes, invariants
(swap, 90-degree rotation, scale, crop equivalence) and an independent exact-rational
integral-image evaluation.  Definitions: PAPER.md P:117-118; SPEC.md S:53-61,
S:88; readings R1-R9, R16.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def ramp8():
    y, x = np.mgrid[0:8, 0:8]
    return (16 * x + 2 * y + 10).astype(np.uint8)


def _bits(out, K):
    return np.unpackbits(out, axis=1, bitorder="little")[:, :K]


def test_ramp_worked_examples():
    img = ramp8()
    rows = []
    for line in open(os.path.join(GOLD, "bad_ramp_8x8.txt")):
        line = line.split("#")[0].strip()
        if line:
            rows.append([float(t) for t in line.split()])
    assert len(rows) == 14
    for kx, ky, ang, sc, dx1, dy1, dx2, dy2, r, th, exp in rows:
        kp = np.array([[kx, ky, np.float32(ang), sc]], dtype=np.float32)
        pairs = np.array([[dx1, dy1, dx2, dy2]], dtype=np.int8)
        out = oracle.bad_image(img, kp, pairs, np.array([r], np.uint8), np.array([th], np.float32))
        assert _bits(out, 1)[0, 0] == int(exp), (kx, ky, ang, sc, dx1, dy1, dx2, dy2, r, th)


def test_pack_k12_golden():
    lines = {l.split(":")[0]: l.split(":")[1] for l in open(os.path.join(GOLD, "bad_pack_k12.txt"))
             if ":" in l and not l.startswith("#")}
    thr = np.array([float(t) for t in lines["thresholds"].split()], dtype=np.float32)
    exp = [int(t, 16) for t in lines["bytes"].split()]
    img = np.full((40, 40), 77, np.uint8)
    rng = np.random.default_rng(0)
    pairs = rng.integers(-16, 16, size=(12, 4)).astype(np.int8)
    radii = rng.integers(1, 6, size=12).astype(np.uint8)
    out = oracle.bad_image(img, np.array([[20, 20, 0.3, 1.5]], np.float32), pairs, radii, thr)
    assert out.shape == (1, 2)
    assert list(out[0]) == exp


def test_constant_image_bits_are_sign_of_minus_threshold():
    # BJ.ns: "a constant image gives zero differences, so every bit equals the sign of
    # minus its threshold".
    img = np.full((100, 120), 201, np.uint8)
    pairs, radii, thr = synth.bad_tests(11, 256)
    thr = thr.copy()
    thr[:8] = 0.0  # f = 0 = theta -> tie -> bit 1
    kp = synth.keypoints_as_array(synth.keypoints_random(5, 0, 50, 100, 120, 0, 3.0))
    out = oracle.bad_image(img, kp, pairs, radii, thr)
    expect = (thr >= 0).astype(np.uint8)
    assert (_bits(out, 256) == expect[None, :]).all()


def test_swap_symmetry():
    # swapping p1 <-> p2 and theta -> -theta flips the bit except at exact ties (BJ.ns)
    img = synth.image(7, 0, 120, 160)
    pairs, radii, thr = synth.bad_tests(7, 256)
    kp = synth.keypoints_as_array(synth.keypoints_random(7, 0, 64, 120, 160, 0, 2.0))
    a, _, _, ties = oracle.bad_image(img, kp, pairs, radii, thr, want_aux=True)
    b = oracle.bad_image(img, kp, pairs[:, [2, 3, 0, 1]], radii, -thr)
    assert ties.sum() == 0
    assert (_bits(a, 256) ^ _bits(b, 256)).all()


def test_swap_symmetry_with_ties():
    # integer thresholds on a quantised image produce ties; both sides give 1 there
    img = (synth.image(8, 0, 64, 64) // 32).astype(np.uint8)
    pairs, radii, _ = synth.bad_tests(8, 256)
    thr = np.zeros(256, np.float32)
    kp = np.array([[32, 32, 0, 1]], np.float32)
    a, _, _, ties = oracle.bad_image(img, kp, pairs, radii, thr, want_aux=True)
    b = oracle.bad_image(img, kp, pairs[:, [2, 3, 0, 1]], radii, -thr)
    ba, bb = _bits(a, 256)[0], _bits(b, 256)[0]
    assert ties[0] > 0
    n_both_one = int(((ba == 1) & (bb == 1)).sum())
    assert n_both_one == ties[0]
    assert ((ba ^ bb) | (ba & bb)).all()


def test_rotation_90_equals_rotated_table():
    # BJ.ns: "a 90-degree keypoint rotation equals evaluating the 90-degree-rotated pair
    # table".  angle = (float)(pi/2): a = -4.4e-8, b = 1 -> p = (x - dy, y + dx) (R9).
    img = synth.image(9, 0, 96, 96)
    pairs, radii, thr = synth.bad_tests(9, 512)
    rng = np.random.default_rng(1)
    xy = rng.integers(20, 76, size=(40, 2)).astype(np.float32)
    kp_rot = np.column_stack([xy, np.full(40, np.float32(math.pi / 2)), np.ones(40)]).astype(np.float32)
    kp_id = np.column_stack([xy, np.zeros(40), np.ones(40)]).astype(np.float32)
    rot = np.column_stack([-pairs[:, 1], pairs[:, 0], -pairs[:, 3], pairs[:, 2]]).astype(np.int8)
    a = oracle.bad_image(img, kp_rot, pairs, radii, thr)
    b = oracle.bad_image(img, kp_id, rot, radii, thr)
    assert (a == b).all()


def test_scale_two_equals_doubled_offsets():
    img = synth.image(10, 0, 128, 128)
    pairs, radii, thr = synth.bad_tests(10, 256)
    rng = np.random.default_rng(2)
    xy = rng.integers(36, 92, size=(30, 2)).astype(np.float32)
    kp2 = np.column_stack([xy, np.zeros(30), np.full(30, 2.0)]).astype(np.float32)
    kp1 = np.column_stack([xy, np.zeros(30), np.ones(30)]).astype(np.float32)
    a = oracle.bad_image(img, kp2, pairs, radii, thr)
    b = oracle.bad_image(img, kp1, (2 * pairs.astype(np.int16)).astype(np.int8), radii, thr)
    assert (a == b).all()


def test_image_path_equals_patch_path_inside_crop():
    # identity keypoint: crop [x-16, x+15] and evaluate at (16, 16); same bits for every
    # test whose boxes stay inside the crop (SURVEY §8(c) pins)
    img = synth.image(12, 0, 200, 200)
    pairs, radii, thr = synth.bad_tests(12, 256)
    rng = np.random.default_rng(3)
    xy = rng.integers(40, 160, size=(25, 2))
    kp = np.column_stack([xy, np.zeros(25), np.ones(25)]).astype(np.float32)
    crops = np.stack([img[y - 16:y + 16, x - 16:x + 16] for x, y in xy])
    a = _bits(oracle.bad_image(img, kp, pairs, radii, thr), 256)
    b = _bits(oracle.bad_patches(crops, pairs, radii, thr), 256)
    p = pairs.astype(int) + 16
    r = radii.astype(int)
    inside = ((p - r[:, None]) >= 0).all(1) & ((p + r[:, None]) <= 31).all(1)
    assert inside.sum() > 50
    assert (a[:, inside] == b[:, inside]).all()


def _exact_bits_via_integral(img, kp, pairs, radii, thr):
    """independent route: exact-rational compare of box means from an integral image."""
    H, W = img.shape
    ii = np.zeros((H + 1, W + 1), np.int64)
    ii[1:, 1:] = img.astype(np.int64).cumsum(0).cumsum(1)
    x, y, ang, sc = [float(v) for v in kp]
    out = []
    for (dx1, dy1, dx2, dy2), r, th in zip(pairs.astype(int), radii.astype(int), thr):
        means = []
        for dx, dy in ((dx1, dy1), (dx2, dy2)):
            # angle 0, integer scale: exact integer sample point
            px = min(max(int(x) + int(sc) * dx, 0), W - 1)
            py = min(max(int(y) + int(sc) * dy, 0), H - 1)
            x0, x1 = max(px - r, 0), min(px + r, W - 1) + 1
            y0, y1 = max(py - r, 0), min(py + r, H - 1) + 1
            s = ii[y1, x1] - ii[y0, x1] - ii[y1, x0] + ii[y0, x0]
            means.append(Fraction(int(s), (x1 - x0) * (y1 - y0)))
        out.append(int(means[0] - means[1] <= Fraction(float(th))))
    return np.array(out, np.uint8)


def test_against_exact_rational_integral_image():
    img = synth.image(13, 0, 48, 56)
    pairs, radii, thr = synth.bad_tests(13, 128)
    rng = np.random.default_rng(4)
    for _ in range(12):
        kp = np.array([rng.integers(0, 56), rng.integers(0, 48), 0, rng.integers(1, 3)], np.float32)
        got = _bits(oracle.bad_image(img, kp[None], pairs, radii, thr), 128)[0]
        assert (got == _exact_bits_via_integral(img, kp, pairs, radii, thr)).all()


def test_similarity_identity_and_packing():
    # S(x, y) = h(x)^T h(y) = K - 2 * Hamming, K in {8, 256, 512}
    for K in (8, 256, 512):
        pairs, radii, thr = synth.bad_tests(14, K)
        P = synth.patches(14, range(6))
        d = oracle.bad_patches(P, pairs, radii, thr)
        h = 2.0 * _bits(d, K).astype(np.int64) - 1
        for i in range(6):
            for j in range(6):
                ham = int(np.unpackbits(d[i] ^ d[j]).sum())
                assert int(h[i] @ h[j]) == K - 2 * ham


def test_invalid_keypoints_give_zero_rows_and_status():
    img = synth.image(15, 0, 50, 60)
    pairs, radii, thr = synth.bad_tests(15, 64, tmax=-1.0)  # thresholds in [1, -1] range
    kp = np.array([[10, 10, 0, 1], [np.nan, 5, 0, 1], [5, 5, 0, 0], [60, 5, 0, 1], [5, -0.5, 0, 1],
                   [59, 49, 0, 1], [5, 5, np.inf, 1]], np.float32)
    out, status, _, _ = oracle.bad_image(img, kp, pairs, radii, thr, want_aux=True)
    assert list(status) == [0, 1, 1, 1, 1, 0, 1]
    assert (out[status == 1] == 0).all()
    kpi = np.array([0, 0, 0, 0, 0, 3, 0], np.int32)
    _, status2, _, _ = oracle.bad_image(img, kp, pairs, radii, thr, kp_image=kpi, want_aux=True)
    assert status2[5] == 1


def test_empty_batch():
    pairs, radii, thr = synth.bad_tests(0, 32)
    out = oracle.bad_patches(np.zeros((0, 32, 32), np.uint8), pairs, radii, thr)
    assert out.shape == (0, 4)


def test_thread_count_invariance():
    pairs, radii, thr = synth.bad_tests(16, 256)
    P = synth.patches(16, range(300))
    assert (oracle.bad_patches(P, pairs, radii, thr, nthreads=1)
            == oracle.bad_patches(P, pairs, radii, thr, nthreads=8)).all()


# ------------------------------------------------------------ R6 fragility flag pins --
# R6: the oracle flags a keypoint "fragile" when a float64 trig coefficient
# scale*cos / scale*sin lies within 4 float64-ulp of an fp32 rounding boundary, or when any
# sample X or Y lies within 1e-4 of a rounding boundary n + 1/2.  The GPU must match those
# rows bit-exactly too (no exemption); these pins make sure the flag itself is right, so the
# parity report's "fragile rows checked" count means what it says.
def _f32_midpoints(c: float):
    """the two fp32 rounding boundaries around float64 c, as exact rationals (numpy fp32)"""
    f = np.float32(c)
    lo, hi = np.nextafter(f, np.float32(-np.inf)), np.nextafter(f, np.float32(np.inf))
    return (Fraction(float(f)) + Fraction(float(lo))) / 2, (Fraction(float(f)) + Fraction(float(hi))) / 2


@pytest.mark.parametrize("base", [1.0, 3.0 * 2 ** 20, 0.7071067690849304, -1.0, 5.75])
def test_fragile_round_hand_built(base):
    f = np.float32(base)
    assert float(f) == base or base == 0.7071067690849304
    up = float(np.nextafter(f, np.float32(np.inf)))
    mid = (Fraction(float(f)) + Fraction(up)) / 2          # exact fp32 rounding midpoint
    m = float(mid)
    assert Fraction(m) == mid                             # representable in float64
    u = math.ulp(m)                                       # float64 ulp at the midpoint
    assert oracle.fragile_round(m)                        # exactly on the boundary
    assert oracle.fragile_round(m + 3 * u) and oracle.fragile_round(m - 3 * u)
    assert not oracle.fragile_round(m + 5 * u) and not oracle.fragile_round(m - 5 * u)
    assert not oracle.fragile_round(float(f)) and not oracle.fragile_round(up)  # fp32 values
    assert not oracle.fragile_round(0.0)


# Hand-built keypoints whose float64 coefficient scale*sin(angle) sits EXACTLY on an fp32
# rounding midpoint: for a tiny fp32 angle, sin(angle) == angle in float64 (angle^3/6 is far
# below half an ulp), and the product of two fp32 values is exact in float64.  With scale =
# 1 + 2^-23 and angle = 1.5 * 2^-30: b64 = 2^-30 * (1.5 + 2^-23 + 2^-24), exactly halfway
# between the fp32 values 2^-30 * (1.5 + 2^-23) and 2^-30 * (1.5 + 2^-22).  R6 rounds it to
# nearest-even.  angle = 1.25 * 2^-30 gives 2^-30 * (1.25 + 2^-23 + 2^-25): a quarter fp32-ulp
# from the boundary, not fragile.
MIDPOINT_KP = [100.0, 100.0, 1.5 * 2.0 ** -30, 1 + 2.0 ** -23]
SAFE_KP = [100.0, 100.0, 1.25 * 2.0 ** -30, 1 + 2.0 ** -23]


def test_kp_frame_flags_a_coefficient_on_a_midpoint():
    assert math.sin(MIDPOINT_KP[2]) == MIDPOINT_KP[2]
    c = MIDPOINT_KP[3] * MIDPOINT_KP[2]
    lo, hi = 2.0 ** -30 * (1.5 + 2.0 ** -23), 2.0 ** -30 * (1.5 + 2.0 ** -22)
    assert c == (lo + hi) / 2 and float(np.float32(lo)) == lo and float(np.float32(hi)) == hi
    a, b, fr = oracle.kp_frame(MIDPOINT_KP)
    assert fr and a == np.float32(1 + 2.0 ** -23)
    assert b == hi  # ties-to-even: 1.5 + 2^-22 has the even fp32 mantissa, 1.5 + 2^-23 the odd one
    assert (np.float32(b).view(np.uint32) & 1) == 0 and (np.float32(lo).view(np.uint32) & 1) == 1
    a2, b2, fr2 = oracle.kp_frame(SAFE_KP)
    assert not fr2 and b2 == 2.0 ** -30 * (1.25 + 2.0 ** -23)
    # angle 0: a = scale exactly, b = 0 -> never fragile
    assert oracle.kp_frame([5, 5, 0.0, 1.75]) == (1.75, 0.0, False)


@pytest.mark.parametrize("dx_frac,expect", [(5e-5, True), (-5e-5, True), (2e-4, False), (-2e-4, False),
                                            (0.0, True)])
def test_sample_margin_flag(dx_frac, expect):
    """samples at n + 1/2 +- 5e-5 are fragile (margin 1e-4), at +- 2e-4 they are not; the
    exact half (margin 0) is fragile.  angle 0, scale 1, integer y: only x decides."""
    img = synth.image(17, 0, 40, 40)
    pairs, radii, thr = synth.bad_tests(17, 32)
    kp = np.array([[np.float32(20.5 + dx_frac), 20.0, 0.0, 1.0]], np.float32)
    _, status, fragile, _ = oracle.bad_image(img, kp, pairs, radii, thr, want_aux=True)
    assert status[0] == 0
    assert bool(fragile[0]) == expect


def test_sample_half_rounds_up():
    """R6: p = floor(X + 1/2): a sample exactly at n + 1/2 goes to n + 1.  Ramp image
    I(y, x) = 16x + 2y + 10; test p1 = kp + (0, 0) with r = 1 against p2 = kp + (-16, 0),
    which clamps to column 0 (box cols 0..1, rows 3..5, A = 6, S = 6*10 + 3*16 + 2*(3+4+5)*2
    = 156 -> mean 26).  kp x = 3.5 -> p1 = (4, 4): mean 82 (unclamped odd box = I(centre));
    kp x = 3.49 -> p1 = (3, 4): mean 66.  The bit is [f <= theta]: with theta = f it is 1,
    with theta = f - 1/4 it is 0, for the f of the rounded-up point only."""
    img = ramp8()
    pairs = np.array([[0, 0, -16, 0]], np.int8)
    r = np.array([1], np.uint8)
    s2 = sum(16 * xx + 2 * yy + 10 for yy in (3, 4, 5) for xx in (0, 1))
    assert s2 == 156
    for x, m1 in ((3.5, 82.0), (3.49, 66.0)):
        kp = np.array([[x, 4.0, 0.0, 1.0]], np.float32)
        f = m1 - s2 / 6.0
        out_eq = oracle.bad_image(img, kp, pairs, r, np.array([f], np.float32))
        out_lt = oracle.bad_image(img, kp, pairs, r, np.array([f - 0.25], np.float32))
        assert _bits(out_eq, 1)[0, 0] == 1 and _bits(out_lt, 1)[0, 0] == 0, (x, f)
