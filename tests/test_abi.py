"""Host-only checks of the C-ABI library (no GPU needed): it loads on a CPU-only host,
exports every entry point include/bindesc.h declares, and rejects bad arguments with
BD_EINVAL before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2108_08380_b200 as bd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "bindesc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:BD_API\s+)?(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**([a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_expected_entry_points():
    names = header_functions()
    assert set(names) == set(bd.EXPORTS), names


def test_library_exports_every_header_symbol():
    L = bd.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    # and only C symbols: no C++ mangled export leaks across the boundary
    out = os.popen(f"nm -D --defined-only {bd.library_path()}").read()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for name in header_functions():
        assert name in exported
    assert not [s for s in exported if s.startswith("_Z")], "C++ symbols exported"


def test_debug_library_exports_the_same_abi():
    """libbindesc_debug.so (BINDESC_DEBUG=1: device bounds checks, poisoned shared memory,
    mbarrier watchdogs) is a drop-in build of the same ABI."""
    dbg = os.path.join(os.path.dirname(bd.library_path()), "libbindesc_debug.so")
    assert os.path.exists(dbg)
    L = ctypes.CDLL(dbg)
    for name in header_functions():
        assert hasattr(L, name), name
    L.bd_version.restype = ctypes.c_int
    assert L.bd_version() == bd.lib().bd_version()


def test_version_and_error_string():
    assert bd.lib().bd_version() >= 100
    assert isinstance(bd.lib().bd_last_error(), bytes)


def _create(pairs, radii, thr, K):
    h = ctypes.c_void_p()
    pairs = np.ascontiguousarray(pairs, np.int8)
    radii = np.ascontiguousarray(radii, np.uint8)
    thr = np.ascontiguousarray(thr, np.float32)
    rc = bd.lib().bad_create(pairs.ctypes.data, radii.ctypes.data, thr.ctypes.data, K, ctypes.byref(h))
    return rc, h


@pytest.mark.parametrize("K", [0, 12, 31, 544, -32])
def test_bad_create_rejects_bad_K(K):
    n = max(K, 1)
    rc, h = _create(np.zeros((n, 4)), np.ones(n), np.zeros(n), K)
    assert rc == bd.BD_EINVAL and not h.value
    assert b"K=" in bd.lib().bd_last_error()


def test_bad_create_rejects_bad_tables():
    p = np.zeros((32, 4)); r = np.ones(32); t = np.zeros(32)
    p2 = p.copy(); p2[3, 1] = 16
    assert _create(p2, r, t, 32)[0] == bd.BD_EINVAL
    p2 = p.copy(); p2[3, 2] = -17
    assert _create(p2, r, t, 32)[0] == bd.BD_EINVAL
    r2 = r.copy(); r2[5] = 8
    assert _create(p, r2, t, 32)[0] == bd.BD_EINVAL
    t2 = t.copy(); t2[7] = np.nan
    assert _create(p, r, t2, 32)[0] == bd.BD_EINVAL
    h = ctypes.c_void_p()
    assert bd.lib().bad_create(None, None, None, 32, ctypes.byref(h)) == bd.BD_EINVAL
    assert bd.lib().bad_create(None, None, None, 32, None) == bd.BD_EINVAL


def test_hashsift_create_rejects():
    h = ctypes.c_void_p()
    B = np.zeros((40, 129), np.float32)
    assert bd.lib().hashsift_create(B.ctypes.data, 40, ctypes.byref(h)) == bd.BD_EINVAL
    B = np.zeros((32, 129), np.float32); B[2, 5] = np.inf
    assert bd.lib().hashsift_create(B.ctypes.data, 32, ctypes.byref(h)) == bd.BD_EINVAL


def test_compute_rejects_null_model_and_args():
    L = bd.lib()
    assert L.bad_compute(None, None, 1, 10, 10, 10, None, None, 5, None, None, None) == bd.BD_EINVAL
    assert L.bad_compute_patches(None, None, 5, None, None) == bd.BD_EINVAL
    assert L.hashsift_compute_patches(None, None, 5, None, None, None) == bd.BD_EINVAL
    assert L.bd_describe_warped(None, None, None, 1, 10, 10, 10, None, None, 5, None, None, None, None) == bd.BD_EINVAL
    assert L.bd_warp_patches(None, 1, 10, 10, 10, None, None, -1, None, None, None) == bd.BD_EINVAL
    # pitch < W, bad sizes
    assert L.bd_integral_image(ctypes.c_void_p(16), 1, 10, 20, 10, ctypes.c_void_p(16), None) == bd.BD_EINVAL
    assert L.bd_integral_image(ctypes.c_void_p(16), 1, 0, 20, 20, ctypes.c_void_p(16), None) == bd.BD_EINVAL
    assert L.bd_integral_image(ctypes.c_void_p(16), 1, 5000, 5000, 5000, ctypes.c_void_p(16), None) == bd.BD_EINVAL
    assert L.bd_warp_patches(ctypes.c_void_p(16), 1, 10, 10, 10, ctypes.c_void_p(8), None, 3,
                             ctypes.c_void_p(16), None, None) == bd.BD_EINVAL  # misaligned kps


def test_product_path_does_not_import_oracle():
    import ast
    pkg = os.path.join(ROOT, "paper_2108_08380_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, (ast.Import, ast.ImportFrom)):
                        mods = [a.name for a in node.names] if isinstance(node, ast.Import) else [node.module or ""]
                        assert not any(m.split(".")[0] in ("oracle", "synth") for m in mods), (p, mods)
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "oracle" not in open(p).read().lower().replace("no oracle", ""), p


def test_match_hamming_rejects():
    L = bd.lib()
    off = np.array([0, 4], np.int64)
    bad = np.array([0, 0], np.int64)
    P = ctypes.c_void_p
    dummy = P(1024)  # never dereferenced: every call below fails validation first
    assert L.bd_match_hamming(None, off.ctypes.data, dummy, off.ctypes.data, 1, 256, dummy, None, None, None, None,
                              None) == bd.BD_EINVAL
    assert L.bd_match_hamming(dummy, off.ctypes.data, dummy, off.ctypes.data, 1, 100, dummy, None, None, None, None,
                              None) == bd.BD_EINVAL
    assert L.bd_match_hamming(dummy, bad.ctypes.data, dummy, off.ctypes.data, 1, 256, dummy, None, None, None, None,
                              None) == bd.BD_EINVAL
    assert L.bd_match_hamming(dummy, off.ctypes.data, dummy, off.ctypes.data, 0, 256, dummy, None, None, None, None,
                              None) == bd.BD_EINVAL
    # mutual without the reverse NN output
    assert L.bd_match_hamming(dummy, off.ctypes.data, dummy, off.ctypes.data, 1, 256, dummy, None, None, None,
                              dummy, None) == bd.BD_EINVAL
    assert b"mutual" in L.bd_last_error()
