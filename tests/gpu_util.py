"""Shared helpers of the -m gpu parity tests (comparison rules of DESIGN.md §4)."""
import numpy as np


def to_bytes(words):
    """device uint32 words (n, K/32) -> LSB-first bytes (n, K/8) (the oracle's packing)."""
    w = words.cpu().numpy() if hasattr(words, "cpu") else np.asarray(words)
    w = np.ascontiguousarray(w).view(np.uint32).astype("<u4")
    return w.view(np.uint8).reshape(w.shape[0], -1)


def bits(bytes_, K):
    return np.unpackbits(np.asarray(bytes_, np.uint8), axis=1, bitorder="little")[:, :K]


def assert_bad_exact(gpu_words, oracle_bytes, K, fragile=None, what=""):
    """BAD: bit-exact on EVERY row (BJ.ns), R6-fragile keypoints included — the GPU evaluates
    the identical fp32 sample-point rule, so no exemption applies.  When the oracle's fragility
    flags are passed, the message splits the mismatching rows into fragile / non-fragile
    (SURVEY §8(c) parity report fields) so a regression on the hard rows is visible.
    Returns the number of fragile rows checked (for the caller's coverage assertions)."""
    g = to_bytes(gpu_words)
    assert g.shape == oracle_bytes.shape, (g.shape, oracle_bytes.shape)
    bad_rows = np.nonzero((g != oracle_bytes).any(1))[0]
    n_frag = 0 if fragile is None else int(np.count_nonzero(fragile))
    if len(bad_rows):
        if fragile is not None:
            nf = int(np.count_nonzero(np.asarray(fragile)[bad_rows]))
            raise AssertionError(f"{what}: {len(bad_rows)} rows differ ({nf} of them R6-fragile, "
                                 f"{len(bad_rows) - nf} not), e.g. {bad_rows[:5].tolist()}")
        raise AssertionError(f"{what}: {len(bad_rows)} rows differ, e.g. {bad_rows[:5].tolist()}")
    return n_frag


def hashsift_compare(gpu_words, oracle_bytes, proj, N, band=1e-3, max_frac=1e-3):
    """R13: every mismatching bit must have oracle |p| < band and mismatches <= max_frac of bits."""
    gb = bits(to_bytes(gpu_words), N)
    ob = bits(oracle_bytes, N)
    mism = gb != ob
    outside = mism & (np.abs(proj) >= band)
    n_bits = gb.size
    stats = dict(bits=n_bits, mismatches=int(mism.sum()), outside_band=int(outside.sum()),
                 band_pop_1e3=float((np.abs(proj) < 1e-3).mean()), band_pop_1e4=float((np.abs(proj) < 1e-4).mean()))
    assert stats["outside_band"] == 0, stats
    assert stats["mismatches"] <= max_frac * n_bits, stats
    return stats


def assert_sift_close(gpu_sift, oracle_sift, rel=1e-4):
    """R14: per descriptor max_i |g_i - o_i| <= rel * ||o||_2; zero descriptors exactly zero."""
    g = gpu_sift.cpu().numpy().astype(np.float64) if hasattr(gpu_sift, "cpu") else np.asarray(gpu_sift, np.float64)
    o = np.asarray(oracle_sift, np.float64)
    nrm = np.linalg.norm(o, axis=1)
    err = np.abs(g - o).max(1)
    zero = nrm == 0
    assert (g[zero] == 0).all(), "zero descriptors must be exactly zero"
    worst = float((err[~zero] / nrm[~zero]).max()) if (~zero).any() else 0.0
    assert worst <= rel, f"max relative SIFT error {worst:.3g} > {rel}"
    return worst
