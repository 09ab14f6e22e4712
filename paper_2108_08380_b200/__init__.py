"""paper_2108_08380_b200 — B200-native batched BAD / HashSIFT binary descriptors.

Thin Python binding over the C ABI in ``include/bindesc.h`` (``libbindesc.so``, sm_100a).
Argument marshalling only: every step of the path runs in the library's CUDA kernels.
torch supplies device memory and streams.  There is NO CPU fallback: if the shared
library cannot be loaded, or a tensor is not on a CUDA device, the calls raise.

Method: arXiv 2108.08380 — BAD and HashSIFT; see DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import model_files

__all__ = ["BadModel", "HashSiftModel", "bad_compute", "bad_compute_patches", "hashsift_compute",
           "hashsift_compute_patches", "warp_patches", "describe_warped", "integral_image", "match_hamming",
           "library_path", "BindescError"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# BINDESC_DEBUG=1 loads the debug build (device bounds checks, poisoned shared memory,
# mbarrier watchdogs; paper_2108_08380_b200/build.py) — same ABI, same results
_LIB_PATH = os.path.join(_HERE, "libbindesc_debug.so" if os.environ.get("BINDESC_DEBUG") == "1" else "libbindesc.so")

BD_OK, BD_EINVAL, BD_ENOMEM, BD_ECUDA, BD_EUNSUPPORTED = 0, -1, -2, -3, -4

# every entry point include/bindesc.h declares (checked by tests/test_abi.py)
EXPORTS = ["bad_create", "bad_destroy", "bad_num_bits", "bad_compute", "bad_compute_patches",
           "hashsift_create", "hashsift_destroy", "hashsift_num_bits", "hashsift_compute_patches",
           "hashsift_compute", "bd_warp_patches", "bd_describe_warped", "bd_integral_image",
           "bd_last_error", "bd_version", "bd_profile_start", "bd_profile_stop", "bd_profile_query",
           "bd_match_hamming", "bad_create_ex", "hashsift_create_ex", "bd_warp_patches_ex",
           "bd_describe_warped_ex", "bd_select_features", "bd_describe_warped_host"]

BD_BAD_SCALE_RADIUS = 1
BD_HS_ROOTSIFT = 1
WARP_MODES = {"nn": 0, "bilinear": 1}


class BindescError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"bindesc error {code}: {msg}")
        self.code = code


_lib = None


def library_path() -> str:
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    """Load libbindesc.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_2108_08380_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(_LIB_PATH)
        P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        PP = ctypes.POINTER(ctypes.c_void_p)
        sig = {
            "bad_create": ([P, P, P, I, PP], I),
            "bad_destroy": ([P], None),
            "bad_num_bits": ([P], I),
            "bad_compute": ([P, P, I, I, I, I64, P, P, I64, P, P, P], I),
            "bad_compute_patches": ([P, P, I64, P, P], I),
            "hashsift_create": ([P, I, PP], I),
            "hashsift_destroy": ([P], None),
            "hashsift_num_bits": ([P], I),
            "hashsift_compute_patches": ([P, P, I64, P, P, P], I),
            "hashsift_compute": ([P, P, I, I, I, I64, P, P, I64, P, P, P, P], I),
            "bd_warp_patches": ([P, I, I, I, I64, P, P, I64, P, P, P], I),
            "bd_describe_warped": ([P, P, P, I, I, I, I64, P, P, I64, P, P, P, P], I),
            "bd_integral_image": ([P, I, I, I, I64, P, P], I),
            "bd_match_hamming": ([P, P, P, P, I, I, P, P, P, P, P, P], I),
            "bad_create_ex": ([P, P, P, I, I, PP], I),
            "hashsift_create_ex": ([P, I, I, PP], I),
            "bd_warp_patches_ex": ([P, I, I, I, I64, P, P, I64, I, P, P, P], I),
            "bd_describe_warped_ex": ([P, P, P, I, I, I, I64, P, P, I64, I, P, P, P, P], I),
            "bd_select_features": ([P, I, P, I, P, P, I, P, P, I, P, P, P], I),
            "bd_describe_warped_host": ([P, P, P, I, I, I, I64, P, P, I64, I, P, P, P, I], I),
            "bd_last_error": ([], ctypes.c_char_p),
            "bd_version": ([], I),
            "bd_profile_start": ([], I),
            "bd_profile_stop": ([], I),
            "bd_profile_query": ([I, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_double)], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != BD_OK:
        raise BindescError(rc, lib().bd_last_error().decode())


def _torch():
    import torch
    return torch


def _dev_ptr(t, name, dtype=None, shape=None, device=None):
    """data pointer of a contiguous CUDA tensor (None -> NULL), after checking what the C ABI
    cannot check for device buffers: dtype, exact shape (None entries = any) and device.  A
    wrong-sized out / status / kp_image buffer would otherwise be read or written out of bounds
    by the kernels."""
    if t is None:
        return None
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None:
        ok = (t.dtype in dtype) if isinstance(dtype, tuple) else (t.dtype == dtype)
        if not ok:
            raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if shape is not None:
        if t.dim() != len(shape) or any(e is not None and int(d) != int(e) for d, e in zip(t.shape, shape)):
            raise ValueError(f"{name} must have shape {tuple('*' if e is None else e for e in shape)}, "
                             f"got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


_WORDS = None  # filled lazily: (torch.int32, torch.uint32) where available


def _words_dtype():
    global _WORDS
    if _WORDS is None:
        torch = _torch()
        _WORDS = (torch.int32,) + ((torch.uint32,) if hasattr(torch, "uint32") else ())
    return _WORDS


def _kps_args(kps, kp_image, m_dev):
    """validated (kps, kp_image) pointers: kps float32 (m, 4), kp_image int32 (m,) or None."""
    torch = _torch()
    m = kps.shape[0]
    kp = _dev_ptr(kps, "kps", torch.float32, (m, 4), m_dev)
    ki = _dev_ptr(kp_image, "kp_image", torch.int32, (m,), m_dev)
    return kp, ki, m


def _stream(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class BadModel:
    """BAD-K model: K tests (dx1, dy1, dx2, dy2, r, theta)."""

    def __init__(self, pairs, radii, thresholds, scale_radius=False):
        pairs = np.ascontiguousarray(pairs, dtype=np.int8).reshape(-1, 4)
        radii = np.ascontiguousarray(radii, dtype=np.uint8).reshape(-1)
        thr = np.ascontiguousarray(thresholds, dtype=np.float32).reshape(-1)
        K = len(radii)
        if pairs.shape[0] != K or thr.shape[0] != K:
            raise ValueError("pairs / radii / thresholds disagree on K")
        h = ctypes.c_void_p()
        flags = BD_BAD_SCALE_RADIUS if scale_radius else 0
        _check(lib().bad_create_ex(pairs.ctypes.data, radii.ctypes.data, thr.ctypes.data, K, flags, ctypes.byref(h)))
        self._h = h
        self.K = K

    @classmethod
    def from_file(cls, path, scale_radius=False):
        """A `BADMODEL v1` text file (model_files.py)."""
        return cls(*model_files.read_bad_model(path), scale_radius=scale_radius)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.bad_destroy(self._h)
            self._h = None


class HashSiftModel:
    """HashSIFT-N model: B = [W | b], N x 129 float32."""

    def __init__(self, B, rootsift=False):
        B = np.ascontiguousarray(B, dtype=np.float32)
        if B.ndim != 2 or B.shape[1] != 129:
            raise ValueError("B must be N x 129")
        h = ctypes.c_void_p()
        _check(lib().hashsift_create_ex(B.ctypes.data, B.shape[0], BD_HS_ROOTSIFT if rootsift else 0,
                                        ctypes.byref(h)))
        self._h = h
        self.N = B.shape[0]

    @classmethod
    def from_file(cls, path):
        """A `HASHSIFT v1` text file (model_files.py)."""
        B, rootsift = model_files.read_hashsift_model(path)
        return cls(B, rootsift=rootsift)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hashsift_destroy(self._h)
            self._h = None


def _images_args(images):
    """images uint8 (n, H, W) or (H, W) on a CUDA device; rows may be strided (a view of a
    pitched buffer, e.g. buf[:, :, :W]): stride(2) == 1, stride(1) = pitch >= W and
    stride(0) == H * pitch (the C ABI's n x H rows of `pitch` bytes)."""
    torch = _torch()
    if not isinstance(images, torch.Tensor) or not images.is_cuda:
        raise TypeError("images must be a CUDA tensor (no CPU fallback)")
    if images.dtype != torch.uint8:
        raise TypeError(f"images must be torch.uint8, got {images.dtype}")
    if images.dim() == 2:
        images = images.unsqueeze(0)
    if images.dim() != 3:
        raise ValueError(f"images must be (n, H, W), got {tuple(images.shape)}")
    n, H, W = images.shape
    pitch = images.stride(1) if H > 1 else max(W, images.stride(1))
    if W > 1 and images.stride(2) != 1:
        raise ValueError("image rows must be contiguous (stride(2) == 1)")
    if pitch < W or (n > 1 and images.stride(0) != H * pitch):
        raise ValueError(f"images must be n x H rows of a common pitch >= W (strides {images.stride()})")
    return images.data_ptr(), n, H, W, pitch


def bad_compute(model: BadModel, images, kps, kp_image=None, out=None, status=None, stream=None):
    """images uint8 (n, H, W) CUDA; kps float32 (m, 4) [x, y, angle, scale]; kp_image int32 (m,).
    -> out uint32 (m, K/32) [, status uint8 (m,)]"""
    torch = _torch()
    ip, n, H, W, pitch = _images_args(images)
    dev = images.device
    kp, ki, m = _kps_args(kps, kp_image, dev)
    if out is None:
        out = torch.empty((m, model.K // 32), dtype=torch.int32, device=dev)
    _check(lib().bad_compute(model.handle, ip, n, H, W, pitch, kp, ki, m,
                             _dev_ptr(out, "out", _words_dtype(), (m, model.K // 32), dev),
                             _dev_ptr(status, "status", torch.uint8, (m,), dev), _stream(stream)))
    return out


def bad_compute_patches(model: BadModel, patches, out=None, stream=None):
    torch = _torch()
    n = patches.shape[0]
    dev = patches.device
    pp = _dev_ptr(patches, "patches", torch.uint8, (n, 32, 32) if patches.dim() == 3 else (n, 1024), dev)
    if out is None:
        out = torch.empty((n, model.K // 32), dtype=torch.int32, device=dev)
    _check(lib().bad_compute_patches(model.handle, pp, n, _dev_ptr(out, "out", _words_dtype(), (n, model.K // 32), dev),
                                     _stream(stream)))
    return out


def hashsift_compute_patches(model: HashSiftModel, patches, out=None, sift=None, want_sift=False, stream=None):
    torch = _torch()
    n = patches.shape[0]
    dev = patches.device
    pp = _dev_ptr(patches, "patches", torch.uint8, (n, 32, 32) if patches.dim() == 3 else (n, 1024), dev)
    if out is None:
        out = torch.empty((n, model.N // 32), dtype=torch.int32, device=dev)
    if want_sift and sift is None:
        sift = torch.empty((n, 128), dtype=torch.float32, device=dev)
    _check(lib().hashsift_compute_patches(model.handle, pp, n,
                                          _dev_ptr(out, "out", _words_dtype(), (n, model.N // 32), dev),
                                          _dev_ptr(sift, "sift", torch.float32, (n, 128), dev),
                                          _stream(stream)))
    return (out, sift) if want_sift else out


def hashsift_compute(model: HashSiftModel, images, kps, kp_image=None, out=None, sift=None, status=None,
                     stream=None):
    torch = _torch()
    ip, n, H, W, pitch = _images_args(images)
    dev = images.device
    kp, ki, m = _kps_args(kps, kp_image, dev)
    if out is None:
        out = torch.empty((m, model.N // 32), dtype=torch.int32, device=dev)
    _check(lib().hashsift_compute(model.handle, ip, n, H, W, pitch, kp, ki, m,
                                  _dev_ptr(out, "out", _words_dtype(), (m, model.N // 32), dev),
                                  _dev_ptr(sift, "sift", torch.float32, (m, 128), dev),
                                  _dev_ptr(status, "status", torch.uint8, (m,), dev), _stream(stream)))
    return out


def warp_patches(images, kps, kp_image=None, out=None, status=None, stream=None, mode="nn"):
    torch = _torch()
    ip, n, H, W, pitch = _images_args(images)
    dev = images.device
    kp, ki, m = _kps_args(kps, kp_image, dev)
    if out is None:
        out = torch.empty((m, 32, 32), dtype=torch.uint8, device=dev)
    _check(lib().bd_warp_patches_ex(ip, n, H, W, pitch, kp, ki, m, WARP_MODES[mode],
                                    _dev_ptr(out, "out", torch.uint8, (m, 32, 32), dev),
                                    _dev_ptr(status, "status", torch.uint8, (m,), dev), _stream(stream)))
    return out


def describe_warped(bad: BadModel | None, hs: HashSiftModel | None, images, kps, kp_image=None, out_bad=None,
                    out_hs=None, status=None, stream=None, mode="nn"):
    """configs[4] step: NN warp once, BAD-K and HashSIFT-N on the warped patch."""
    torch = _torch()
    ip, n, H, W, pitch = _images_args(images)
    dev = images.device
    kp, ki, m = _kps_args(kps, kp_image, dev)
    if bad is not None and out_bad is None:
        out_bad = torch.empty((m, bad.K // 32), dtype=torch.int32, device=dev)
    if hs is not None and out_hs is None:
        out_hs = torch.empty((m, hs.N // 32), dtype=torch.int32, device=dev)
    ob = _dev_ptr(out_bad, "out_bad", _words_dtype(), (m, bad.K // 32), dev) if bad is not None else None
    oh = _dev_ptr(out_hs, "out_hs", _words_dtype(), (m, hs.N // 32), dev) if hs is not None else None
    _check(lib().bd_describe_warped_ex(bad.handle if bad is not None else None,
                                       hs.handle if hs is not None else None, ip, n, H, W, pitch, kp, ki,
                                       m, WARP_MODES[mode], ob, oh,
                                       _dev_ptr(status, "status", torch.uint8, (m,), dev), _stream(stream)))
    return out_bad, out_hs


def _host_ptr(t, name, dtype, shape=None):
    """data pointer of a contiguous CPU tensor of the given dtype and shape (None -> NULL)."""
    if t is None:
        return None
    torch = _torch()
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a CPU tensor (pinned for copy/compute overlap)")
    ok = (t.dtype in dtype) if isinstance(dtype, tuple) else (t.dtype == dtype)
    if not ok:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if shape is not None and (t.dim() != len(shape) or any(int(d) != int(e) for d, e in zip(t.shape, shape))):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def describe_warped_host(bad: BadModel | None, hs: HashSiftModel | None, images, kps, kp_image, out_bad=None,
                         out_hs=None, status=None, mode="nn", chunk_images=0):
    """End-to-end describe_warped from HOST tensors (bd_describe_warped_host): synchronous,
    host->device copies overlapped with the kernels chunk by chunk.  images uint8 (n, H, W),
    kps float32 (m, 4), kp_image int32 (m,) non-decreasing; outputs are CPU int32 tensors
    (pinned when allocated here)."""
    torch = _torch()
    if images.dim() == 2:
        images = images.unsqueeze(0)
    n, H, W = images.shape
    m = kps.shape[0]
    pin = images.is_pinned()
    if bad is not None and out_bad is None:
        out_bad = torch.empty((m, bad.K // 32), dtype=torch.int32, pin_memory=pin)
    if hs is not None and out_hs is None:
        out_hs = torch.empty((m, hs.N // 32), dtype=torch.int32, pin_memory=pin)
    _check(lib().bd_describe_warped_host(bad.handle if bad is not None else None,
                                         hs.handle if hs is not None else None,
                                         _host_ptr(images, "images", torch.uint8), n, H, W, images.stride(1),
                                         _host_ptr(kps, "kps", torch.float32, (m, 4)),
                                         _host_ptr(kp_image, "kp_image", torch.int32, (m,)), m, WARP_MODES[mode],
                                         _host_ptr(out_bad, "out_bad", _words_dtype(), (m, bad.K // 32))
                                         if bad is not None else None,
                                         _host_ptr(out_hs, "out_hs", _words_dtype(), (m, hs.N // 32))
                                         if hs is not None else None,
                                         _host_ptr(status, "status", torch.uint8, (m,)), int(chunk_images)))
    return out_bad, out_hs


def integral_image(images, out=None, stream=None):
    torch = _torch()
    ip, n, H, W, pitch = _images_args(images)
    if out is None:
        out = torch.empty((n, H + 1, W + 1), dtype=torch.int32, device=images.device)
    _check(lib().bd_integral_image(ip, n, H, W, pitch,
                                   _dev_ptr(out, "out", _words_dtype(), (n, H + 1, W + 1), images.device),
                                   _stream(stream)))
    return out


def match_hamming(a, b, a_off=None, b_off=None, K=None, mutual=True, stream=None):
    """NEXT-1: brute-force Hamming NN + mutual NN on the tensor cores.
    a, b: int32/uint32 CUDA tensors (rows, K/32) of packed descriptors; a_off / b_off: host
    sequences of n_pairs + 1 row offsets (default: one pair = all rows).
    -> dict(nn_ab, dist_ab, nn_ba, dist_ba, mutual) of CUDA tensors (nn pair-relative)."""
    torch = _torch()
    K = K or a.shape[1] * 32
    a_off = np.ascontiguousarray([0, a.shape[0]] if a_off is None else a_off, dtype=np.int64)
    b_off = np.ascontiguousarray([0, b.shape[0]] if b_off is None else b_off, dtype=np.int64)
    n_a, n_b = int(a_off[-1]), int(b_off[-1])
    dev = a.device
    r = {"nn_ab": torch.empty(n_a, dtype=torch.int32, device=dev),
         "dist_ab": torch.empty(n_a, dtype=torch.int32, device=dev)}
    if mutual:
        r["nn_ba"] = torch.empty(n_b, dtype=torch.int32, device=dev)
        r["dist_ba"] = torch.empty(n_b, dtype=torch.int32, device=dev)
        r["mutual"] = torch.empty(n_a, dtype=torch.uint8, device=dev)
    if K % 32 or a.dim() != 2 or b.dim() != 2 or a.shape[1] != K // 32 or b.shape[1] != K // 32:
        raise ValueError(f"a, b must be (rows, K/32) packed words with K % 32 == 0 (K={K}, a {tuple(a.shape)}, "
                         f"b {tuple(b.shape)})")
    if n_a > a.shape[0] or n_b > b.shape[0] or (np.diff(a_off) < 0).any() or (np.diff(b_off) < 0).any():
        raise ValueError("row offsets must be non-decreasing and within a / b")
    _check(lib().bd_match_hamming(_dev_ptr(a, "a", _words_dtype(), None, dev), a_off.ctypes.data,
                                  _dev_ptr(b, "b", _words_dtype(), None, dev), b_off.ctypes.data,
                                  len(a_off) - 1, K, _dev_ptr(r["nn_ab"], "nn_ab"), _dev_ptr(r["dist_ab"], "dist"),
                                  _dev_ptr(r.get("nn_ba"), "nn_ba"), _dev_ptr(r.get("dist_ba"), "dist_ba"),
                                  _dev_ptr(r.get("mutual"), "mutual"), _stream(stream)))
    return r


def select_features(patches, triplets, s_ap, s_an, tau, cand_pairs, cand_radii, stream=None):
    """NEXT-4: one feature-selection iteration (Alg. 1 lines 4-12 + Alg. 2 integer sort).
    patches uint8 (M, 32, 32), triplets int32 (N, 3), s_ap / s_an int32 (N,) CUDA tensors;
    cand_pairs (J, 4) int8 / cand_radii (J,) uint8 host arrays.
    -> (loss int64 (J,), bucket int32 (J,)) CUDA tensors (bucket -1 = theta -inf)."""
    torch = _torch()
    cp = np.ascontiguousarray(cand_pairs, dtype=np.int8).reshape(-1, 4)
    cr = np.ascontiguousarray(cand_radii, dtype=np.uint8).reshape(-1)
    J = len(cr)
    dev = patches.device
    loss = torch.empty(J, dtype=torch.int64, device=dev)
    bucket = torch.empty(J, dtype=torch.int32, device=dev)
    M, Nt = patches.shape[0], triplets.shape[0]
    if cp.shape[0] != J:
        raise ValueError("cand_pairs / cand_radii disagree on J")
    _check(lib().bd_select_features(_dev_ptr(patches, "patches", torch.uint8, (M, 32, 32), dev), M,
                                    _dev_ptr(triplets, "triplets", torch.int32, (Nt, 3), dev), Nt,
                                    _dev_ptr(s_ap, "s_ap", torch.int32, (Nt,), dev),
                                    _dev_ptr(s_an, "s_an", torch.int32, (Nt,), dev), int(tau),
                                    cp.ctypes.data, cr.ctypes.data, J, _dev_ptr(loss, "loss"), _dev_ptr(bucket, "bucket"),
                                    _stream(stream)))
    return loss, bucket


def bits_to_bytes(words) -> np.ndarray:
    """uint32 words (n, K/32) (torch or numpy) -> LSB-first bytes (n, K/8) as the oracle packs."""
    if hasattr(words, "cpu"):
        words = words.cpu().numpy()
    w = np.ascontiguousarray(words).view(np.uint32)
    return w.astype("<u4").view(np.uint8).reshape(w.shape[0], -1)


def profile_start() -> None:
    """Start kernel-level tracing (CUDA events around every library kernel launch)."""
    _check(lib().bd_profile_start())


def profile_stop() -> dict:
    """Stop tracing; -> {kernel name: (launches, total device ms)} (waits for the events)."""
    L = lib()
    _check(L.bd_profile_stop())
    out = {}
    i = 0
    name, n, ms = ctypes.c_char_p(), ctypes.c_int64(), ctypes.c_double()
    while L.bd_profile_query(i, ctypes.byref(name), ctypes.byref(n), ctypes.byref(ms)) == BD_OK:
        out[name.value.decode()] = (int(n.value), float(ms.value))
        i += 1
    return out
