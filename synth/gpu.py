"""CUDA twin of the synth generators (libsynth.so) — TEST / BENCH INFRASTRUCTURE.
Generates the BASELINE.json synthetic images / patches directly in device memory,
byte-identical to synth.image() / synth.patches() (tests/test_gpu_synth.py)."""
from __future__ import annotations

import ctypes
import os

import synth

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run paper_2108_08380_b200/build.py")
        L = ctypes.CDLL(_LIB)
        U64, I64, I, LL, P = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p
        L.synth_images.argtypes = [U64, I64, I, I, I, I64, LL, P, P]
        L.synth_patches.argtypes = [U64, I64, I64, LL, P, P]
        _lib = L
    return _lib


def images(seed: int, unit0: int, n: int, H: int, W: int, device="cuda", out=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((n, H, W), dtype=torch.uint8, device=device)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    rc = lib().synth_images(seed, unit0, n, H, W, W, synth.G1, out.data_ptr(), s)
    if rc:
        raise RuntimeError(f"synth_images failed: cuda error {rc}")
    return out


def patches(seed: int, unit0: int, n: int, device="cuda", out=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((n, 32, 32), dtype=torch.uint8, device=device)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    rc = lib().synth_patches(seed, unit0, n, synth.G1, out.data_ptr(), s)
    if rc:
        raise RuntimeError(f"synth_patches failed: cuda error {rc}")
    return out
