"""Model and descriptor text files (SURVEY §5 "optional loaders for SPEC's BADMODEL v1 /
HASHSIFT v1 formats"; the formats are S:257 and S:492 — UTF-8 text).  Host-side parsing only:
the parsed arrays go to the same create calls as any other model.

  BADMODEL v1   line 1 `BADMODEL v1`; line 2 `K <int>`; then K lines `x1 y1 x2 y2 s theta`:
                box centres in the 32x32 patch frame, box side s, real threshold.  This
                library's tests use offsets from the patch centre (16, 16) in [-16, 15] and a
                radius r with side 2r + 1 (R1), so s must be odd and <= 15.
  HASHSIFT v1   line 1 `HASHSIFT v1`; line 2 `K <int> rootsift <0|1>`; then K lines of 129
                decimals (B = [W | b]).
  DESC v1       line 1 `DESC v1 bits=<K> count=<n>`; then n lines of lowercase hex, the
                descriptor's LSB-first bytes (R16: bit k -> bit k % 8 of byte k / 8).
"""
from __future__ import annotations

import numpy as np

_CENTRE = 16  # patch centre of the 32x32 frame (R5: the keypoint sits at (16, 16))


def _lines(path):
    with open(path, "r", encoding="utf-8") as f:
        return [ln.strip() for ln in f if ln.strip()]


def read_bad_model(path):
    """-> (pairs int8 (K, 4) [dx1, dy1, dx2, dy2], radii uint8 (K,), thresholds float32 (K,))."""
    ln = _lines(path)
    if not ln or ln[0] != "BADMODEL v1":
        raise ValueError(f"{path}: first line must be 'BADMODEL v1'")
    head = ln[1].split()
    if len(head) != 2 or head[0] != "K":
        raise ValueError(f"{path}: second line must be 'K <int>'")
    K = int(head[1])
    if K < 1 or len(ln) != 2 + K:
        raise ValueError(f"{path}: K = {K} but {len(ln) - 2} feature lines")
    pairs = np.zeros((K, 4), dtype=np.int8)
    radii = np.zeros(K, dtype=np.uint8)
    thr = np.zeros(K, dtype=np.float32)
    for k, row in enumerate(ln[2:]):
        f = row.split()
        if len(f) != 6:
            raise ValueError(f"{path}: feature {k}: expected 'x1 y1 x2 y2 s theta'")
        x1, y1, x2, y2, s = (int(v) for v in f[:5])
        if not all(0 <= v <= 31 for v in (x1, y1, x2, y2)):
            raise ValueError(f"{path}: feature {k}: centre outside the 32x32 patch")
        if s < 1 or s % 2 == 0 or s > 15:
            raise ValueError(f"{path}: feature {k}: box side {s} is not an odd 1..15 (side 2r+1, r <= 7)")
        pairs[k] = (x1 - _CENTRE, y1 - _CENTRE, x2 - _CENTRE, y2 - _CENTRE)
        radii[k] = (s - 1) // 2
        thr[k] = float(f[5])
    return pairs, radii, thr


def write_bad_model(path, pairs, radii, thresholds):
    pairs = np.asarray(pairs).reshape(-1, 4)
    radii = np.asarray(radii).reshape(-1)
    thr = np.asarray(thresholds, dtype=np.float64).reshape(-1)
    with open(path, "w", encoding="utf-8") as f:
        f.write(f"BADMODEL v1\nK {len(radii)}\n")
        for (dx1, dy1, dx2, dy2), r, t in zip(pairs.tolist(), radii.tolist(), thr.tolist()):
            f.write(f"{dx1 + _CENTRE} {dy1 + _CENTRE} {dx2 + _CENTRE} {dy2 + _CENTRE} {2 * r + 1} {t:.9g}\n")


def read_hashsift_model(path):
    """-> (B float32 (K, 129), rootsift bool)."""
    ln = _lines(path)
    if not ln or ln[0] != "HASHSIFT v1":
        raise ValueError(f"{path}: first line must be 'HASHSIFT v1'")
    head = ln[1].split()
    if len(head) != 4 or head[0] != "K" or head[2] != "rootsift" or head[3] not in ("0", "1"):
        raise ValueError(f"{path}: second line must be 'K <int> rootsift <0|1>'")
    K = int(head[1])
    if K < 1 or len(ln) != 2 + K:
        raise ValueError(f"{path}: K = {K} but {len(ln) - 2} rows")
    B = np.array([[float(v) for v in row.split()] for row in ln[2:]], dtype=np.float64)
    if B.shape != (K, 129):
        raise ValueError(f"{path}: rows must hold 129 values")
    return B.astype(np.float32), head[3] == "1"


def write_hashsift_model(path, B, rootsift=False):
    B = np.asarray(B, dtype=np.float64)
    with open(path, "w", encoding="utf-8") as f:
        f.write(f"HASHSIFT v1\nK {B.shape[0]} rootsift {1 if rootsift else 0}\n")
        for row in B:
            f.write(" ".join(f"{v:.9g}" for v in row) + "\n")


def write_descriptors(path, words, K):
    """words: (n, K/32) uint32/int32 as the kernels write them (R16)."""
    b = np.ascontiguousarray(words).view(np.uint32).astype("<u4").view(np.uint8).reshape(len(words), -1)
    with open(path, "w", encoding="utf-8") as f:
        f.write(f"DESC v1 bits={K} count={len(b)}\n")
        for row in b[:, : (K + 7) // 8]:
            f.write(row.tobytes().hex() + "\n")


def read_descriptors(path):
    """-> (words uint32 (n, ceil(K/32)), K)."""
    ln = _lines(path)
    head = ln[0].split() if ln else []
    if len(head) != 4 or head[:2] != ["DESC", "v1"] or not head[2].startswith("bits=") or not head[3].startswith("count="):
        raise ValueError(f"{path}: first line must be 'DESC v1 bits=<K> count=<n>'")
    K, n = int(head[2][5:]), int(head[3][6:])
    if len(ln) != 1 + n:
        raise ValueError(f"{path}: count = {n} but {len(ln) - 1} rows")
    nbytes, nwords = (K + 7) // 8, (K + 31) // 32
    out = np.zeros((n, nwords * 4), dtype=np.uint8)
    for i, row in enumerate(ln[1:]):
        raw = bytes.fromhex(row)
        if len(raw) != nbytes:
            raise ValueError(f"{path}: row {i} holds {len(raw)} bytes, expected {nbytes}")
        out[i, :nbytes] = np.frombuffer(raw, dtype=np.uint8)
    return out.view("<u4").astype(np.uint32), K
