"""Build the sm_100a shared libraries in-tree (they travel to the GPU box with the repo).

  paper_2108_08380_b200/libbindesc.so   the product: kernels + C ABI (include/bindesc.h)
  synth/libsynth.so                     test/bench input generator (CUDA twin of synth/)

nvcc cross-compiles for sm_100a without a GPU; cudart is linked statically so the library
loads (and exports its symbols) on a CPU-only host.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2108_08380_b200")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libbindesc.so")
# debug build of the same sources (-DBD_DEBUG_CHECKS: device bounds checks, shared memory
# poisoned before use, mbarrier watchdogs — internal.cuh); loaded with BINDESC_DEBUG=1
DEBUG_LIB = os.path.join(PKG, "libbindesc_debug.so")
SYNTH_SRC = os.path.join(ROOT, "synth", "synth.cu")
SYNTH_LIB = os.path.join(ROOT, "synth", "libsynth.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]
# per-file extra flags: the sample-point rule R6 is evaluated in fp32 with no
# fused multiply-add; warp.cu uses packed f32x2 arithmetic that ptxas would otherwise contract
FILE_FLAGS = {"warp.cu": ["-fmad=false"]}  # R6 fp32 rule: no contraction at all in this file


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str], log: str) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... (see {log})")


def _build_lib(lib: str, bdir: str, defines: list[str], force: bool) -> None:
    from concurrent.futures import ThreadPoolExecutor
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "bindesc.h")]
    os.makedirs(bdir, exist_ok=True)
    if not (force or _stale(lib, srcs + hdrs)):
        return
    objs = [os.path.join(bdir, os.path.basename(s) + ".o") for s in srcs]

    def compile_one(so):
        src, obj = so
        if force or _stale(obj, [src] + hdrs):
            _run([NVCC, *ARCH, *FLAGS, *FILE_FLAGS.get(os.path.basename(src), []), "-DBINDESC_BUILD", *defines, "-c",
                  src, "-o", obj], obj + ".log")

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(compile_one, zip(srcs, objs)))
    with open(os.path.join(bdir, "libbindesc.log"), "w") as f:
        for o in objs:
            f.write(open(o + ".log").read() if os.path.exists(o + ".log") else "")
    tmp = lib + f".tmp{os.getpid()}"
    _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", tmp], os.path.join(bdir, "link.log"))
    os.replace(tmp, lib)


def build(force: bool = False, verbose: bool = False, debug: bool = True) -> None:
    bdir = os.path.join(ROOT, "build")
    _build_lib(LIB, bdir, [], force)
    if debug:
        _build_lib(DEBUG_LIB, os.path.join(bdir, "debug"), ["-DBD_DEBUG_CHECKS"], force)
    if force or _stale(SYNTH_LIB, [SYNTH_SRC]):
        tmp = SYNTH_LIB + f".tmp{os.getpid()}"
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC", SYNTH_SRC, "-o", tmp],
             os.path.join(ROOT, "build", "libsynth.log"))
        os.replace(tmp, SYNTH_LIB)
    if verbose:
        print(open(os.path.join(ROOT, "build", "libbindesc.log")).read())


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
