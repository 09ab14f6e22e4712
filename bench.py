#!/usr/bin/env python
"""bench.py — B200 throughput of the batched BAD / HashSIFT extraction path.

Default workload (one "step" = one pass of the whole hot path):
BASELINE.json configs[4] — 8192 seeded 3840x2160 smoothed-noise images (67.9 GB), 4000
keypoints each (scale log-U[1,6], angle U[0,2pi)); every keypoint gets a nearest-neighbour
32x32 patch (a5, with the a2 sample-point rule), BAD-512 on the warped patch (a1 on-chip
integral, a3, a4) and HashSIFT-256 (a6-a9), through the C ABI call bd_describe_warped.
Images are sharded evenly across ranks (total work fixed -> "scaling": "strong"); there is
no collective in the data path (NCCL only for the barrier, the max-over-ranks timing and the
per-image digest check).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 0..4] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

--config selects the workload of the main line (default 4).  configs[1..3] shard their units
(images / patches) across ranks like configs[4]; configs[0] (one image) runs as N replicas.

Prints ONE JSON line (rank 0).  `value` = Mdescriptors/s over the whole job (configs[4]: one
descriptor = one keypoint's BAD-512 + HashSIFT-256 pair, R25).  `roofline` is the dominant
kernel's algorithmic bytes / its CUDA-event duration against the measured HBM copy bandwidth
(MEASURED_PEAKS.json) — the metric's "% of HBM roofline"; `roofline.issue_view` adds the
issue-slot view (ncu warp instructions per unit) for kernels bound on chip.  `per_config`
(N = 1) times configs[0..3] through their own C-ABI calls: median and best of >= 10
individually event-timed calls, Mdesc/s, HBM fraction of SURVEY §8(d)'s algorithmic bytes and
the SM clocks sampled during those calls.  `cpu_baseline` is the CPU oracle (oracle/) timed on a
bounded sample on the host cores (rank 0); `e2e` repeats the metric through the host-buffer C
ABI call bd_describe_warped_host (configs[4]) or with pinned-host copies around the device
call (configs[0..3]); `sharding` compares per-image SHA-256 digests of the descriptors
gathered from all ranks with a single-image recomputation of sampled images on rank 0.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "Mdescriptors/s per GPU (BAD-256, HashSIFT-256) and % of HBM roofline, 1/2/4/8 B200"
DTYPE = ("u8 pixels, u32/u16 integer box sums and exact compares (BAD); f32 SIFT; "
         "TF32 tensor-core operands with f32 accumulate (HashSIFT projection)")


# algorithmic bytes per unit per kernel: what the kernel must
# read and write in HBM by definition of its step, not what it happens to move.
def kernel_bytes(name: str, K: int = 512, N: int = 256) -> float:
    return {
        "warp_nn": 1024 + 1024 + 16 + 4 + 1,   # sampled image bytes + patch out + kp + kp_image + status
        "bad_patch": 1024 + K / 8,              # patch in, bits out
        "sift": 1024 + 512,                     # patch in, 128 fp32 out
        "project": 512 + N / 8,                 # 128 fp32 in, bits out
        "zero_invalid": 1 + 4,                  # status + a word (upper bound)
        "integral": 1 + 2,                      # per pixel: u8 in, u16 (mod 2^16) integral out
        "bad_image": K / 8 + 16,                # per keypoint: bits out + keypoint in (gathers: on chip)
    }.get(name, 0.0)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), "measured"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv, self.err = None, str(e)
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- dist
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            # communicator init lines (ranks, transport) to stderr, so the log shows the NCCL
            # communicator spans all ranks; stdout keeps the one JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=world)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _reduce(x: float, world: int, op: str) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def allreduce_max(x: float, world: int) -> float:
    return _reduce(x, world, "max")


def allreduce_sum(x: float, world: int) -> float:
    return _reduce(x, world, "sum")


def shard(n: int, rank: int, world: int):
    return (n * rank) // world, (n * (rank + 1)) // world


# ----------------------------------------------------------------------------- digests
def words_to_bytes(words) -> np.ndarray:
    """uint32 words (m, K/32) (numpy int32/uint32) -> LSB-first bytes (m, K/8) (R16)."""
    w = np.ascontiguousarray(words).view(np.uint32).astype("<u4")
    return w.view(np.uint8).reshape(w.shape[0], -1)


def image_digests(bad_words, hs_words, per: int) -> list:
    """SHA-256 per image of its keypoints' descriptor rows (BAD bytes then HashSIFT bytes,
    LSB-first, SURVEY §8(c) parity report: 'per-image SHA-256 agreement across P')."""
    b = words_to_bytes(bad_words) if bad_words is not None else None
    h = words_to_bytes(hs_words) if hs_words is not None else None
    m = (b if b is not None else h).shape[0]
    out = []
    for i in range(m // per):
        s = hashlib.sha256()
        if b is not None:
            s.update(b[i * per:(i + 1) * per].tobytes())
        if h is not None:
            s.update(h[i * per:(i + 1) * per].tobytes())
        out.append(s.hexdigest())
    return out


def gather_digests(local: list, i0: int, world: int) -> list:
    """all ranks' (first image, digests) -> the digests of all images in image order."""
    if world == 1:
        return list(local)
    import torch.distributed as dist
    got = [None] * world
    dist.all_gather_object(got, (i0, list(local)))
    got.sort(key=lambda t: t[0])
    return [d for _, ds in got for d in ds]


def check_sharding(all_digests: list, recompute, sample: list) -> dict:
    """compare the gathered digests of the sampled images with a P = 1 single-image
    recomputation (recompute(i) -> digest) on this rank."""
    mism = [i for i in sample if recompute(i) != all_digests[i]]
    return {"images": len(all_digests), "checked": len(sample), "mismatches": len(mism),
            "mismatch_images": mism[:8],
            "digest": hashlib.sha256("".join(all_digests).encode()).hexdigest()}


def sample_images(n_img: int, world: int, k: int = 4) -> list:
    """first and last image of every rank's shard plus a few evenly spaced ones"""
    s = set()
    for r in range(world):
        a, b = shard(n_img, r, world)
        if b > a:
            s.update((a, b - 1))
    s.update(np.linspace(0, n_img - 1, k).astype(int).tolist())
    return sorted(s)


# ----------------------------------------------------------------------------- oracle leg
def oracle_c4_rate(budget_s: float, seed: int = 4):
    """The CPU oracle, as it stands, on a bounded sample of configs[4]: image 0 and its first
    n keypoints (n calibrated so the timed run takes ~budget_s).  -> (Mdesc/s, cores, n)."""
    import oracle
    c = synth.CONFIGS[4]
    img = synth.image(seed, 0, c["H"], c["W"])
    kp_all = synth.keypoints_random_batch(seed, [0], c["kp_per_image"], c["H"], c["W"], c["margin"],
                                          c["scale_max"])
    pairs, radii, thr = synth.bad_tests(seed, c["K"])
    B = synth.hashsift_matrix(seed, c["N"])

    def run(n):
        t = time.perf_counter()
        P = oracle.warp_nn(img, kp_all[:n])
        oracle.bad_patches(P, pairs, radii, thr)
        oracle.hashsift_patches(P, B)
        return time.perf_counter() - t

    t0 = run(256)
    n = int(min(c["kp_per_image"], max(256, 256 * budget_s / max(t0, 1e-6))))
    reps = max(1, int(budget_s / max(t0 * n / 256, 1e-6)))
    reps = min(reps, 8)
    dt = sum(run(n) for _ in range(reps))
    return n * reps / dt / 1e6, oracle.max_threads(), n, reps


def oracle_rate(cfg: int, budget_s: float):
    """the oracle on a bounded sample of configs[cfg] -> (Mdesc/s, cores, sample text)"""
    if cfg == 4:
        t = time.perf_counter()
        r, cores, n, reps = oracle_c4_rate(budget_s)
        return (r, cores, f"configs[4] image 0, first {n} keypoints x {reps} (NN warp + BAD-512 + HashSIFT-256, fp64)",
                time.perf_counter() - t)
    import oracle
    c = synth.CONFIGS[cfg]
    if cfg in (0, 1):
        img = synth.image(cfg, 0, c["H"], c["W"])
        kp = synth.keypoints_as_array(synth.config_keypoints(cfg, 0))
        pairs, radii, thr = synth.bad_tests(cfg, c["K"])
        f = lambda n: oracle.bad_image(img, kp[:n], pairs, radii, thr)  # noqa: E731
        unit, nmax = "keypoints of image 0", len(kp)
    else:
        P = synth.patches(cfg, range(65536))
        if cfg == 2:
            pairs, radii, thr = synth.bad_tests(cfg, c["K"])
            f = lambda n: oracle.bad_patches(P[:n], pairs, radii, thr)  # noqa: E731
        else:
            B = synth.hashsift_matrix(cfg, c["N"])
            f = lambda n: oracle.hashsift_patches(P[:n], B)  # noqa: E731
        unit, nmax = "patches", len(P)
    t = time.perf_counter()
    f(min(64, nmax))
    t0 = max(time.perf_counter() - t, 1e-6)
    n = int(min(nmax, max(64, 64 * budget_s / t0)))
    t = time.perf_counter()
    reps = 0
    while True:
        f(n)
        reps += 1
        if time.perf_counter() - t > budget_s or reps >= 20:
            break
    dt = time.perf_counter() - t
    return n * reps / dt / 1e6, oracle.max_threads(), f"configs[{cfg}] first {n} {unit} x {reps} (fp64)", dt


def reference_main(args, rank, world):
    """--impl reference: the CPU oracle is this tier's reference arm."""
    if rank != 0:
        return
    per_step_budget = max(1.0, 150.0 / (args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_rate(args.config, per_step_budget / 4)
    rates, secs = [], []
    for _ in range(args.steps):
        r, cores, sample, dt = oracle_rate(args.config, per_step_budget)
        rates.append(r)
        secs.append(dt)
    value = float(np.median(rates))
    c = synth.CONFIGS[args.config]
    wl = WORKLOAD_INFO[args.config]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Mdesc/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(secs)) * 1e3,
            "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": c["name"], **wl["config"]},
            "cpu_baseline": {"value": value, "unit": "Mdesc/s", "cores": cores, "kind": "oracle",
                             "sample": sample + " per step"},
            "e2e": {"value": value, "unit": "Mdesc/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- workloads
def _c(i):
    return synth.CONFIGS[i]


WORKLOAD_INFO = {
    0: {"units": _c(0)["kp_per_image"], "scaling": "weak",
        "config": {"images": 1, "H": _c(0)["H"], "W": _c(0)["W"], "keypoints": _c(0)["kp_per_image"], "K": 256,
                   "descriptor": "one keypoint's BAD-256", "parallelism": "replicas (one image per rank)"}},
    1: {"units": _c(1)["n_images"] * _c(1)["kp_per_image"], "scaling": "strong",
        "config": {"images": _c(1)["n_images"], "H": _c(1)["H"], "W": _c(1)["W"],
                   "keypoints": _c(1)["n_images"] * _c(1)["kp_per_image"], "K": 512,
                   "descriptor": "one keypoint's BAD-512"}},
    2: {"units": _c(2)["n_patches"], "scaling": "strong",
        "config": {"patches": _c(2)["n_patches"], "K": 256, "descriptor": "one patch's BAD-256"}},
    3: {"units": _c(3)["n_patches"], "scaling": "strong",
        "config": {"patches": _c(3)["n_patches"], "N": 256, "descriptor": "one patch's HashSIFT-256"}},
    4: {"units": _c(4)["n_images"] * _c(4)["kp_per_image"], "scaling": "strong",
        "config": {"images": _c(4)["n_images"], "H": _c(4)["H"], "W": _c(4)["W"], "kp_per_image": _c(4)["kp_per_image"],
                   "keypoints": _c(4)["n_images"] * _c(4)["kp_per_image"], "K": 512, "N": 256,
                   "descriptor": "one keypoint's BAD-512 + HashSIFT-256 pair"}},
}


class Workload:
    """one BASELINE.json config on this rank's shard: device-resident inputs, the step (one
    C-ABI call over the shard), per-kernel units for the roofline, the pinned-host e2e step and
    per-image digests for the sharding check."""

    def __init__(self, cfg, rank, world, bd, sg, torch, n_override=None):
        self.cfg, self.bd, self.sg, self.torch = cfg, bd, sg, torch
        c = dict(synth.CONFIGS[cfg])
        self.c = c
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.K, self.N = c.get("K"), c.get("N")
        if cfg == 0:
            self.n_total, self.i0, self.i1 = 1, 0, 1
            img = synth.image(0, 0, c["H"], c["W"])
            self.imgs = torch.from_numpy(img).to(dev)
            self.kp_np = synth.keypoints_as_array(synth.config_keypoints(0, 0))
            self.kps = torch.from_numpy(self.kp_np).to(dev)
            self.kpi = None
            self.m = len(self.kp_np)
            self.mb = bd.BadModel(*synth.bad_tests(0, 256))
            self.out = torch.empty((self.m, 8), dtype=torch.int32, device=dev)
            self.alg_bytes = self.m * 646
            self.kunits = {"integral": c["H"] * c["W"], "bad_image": self.m}
            self.per = self.m
        elif cfg in (1, 4):
            self.n_total = n_override or c["n_images"]
            self.i0, self.i1 = shard(self.n_total, rank, world)
            nl = self.i1 - self.i0
            H, W, per = c["H"], c["W"], c["kp_per_image"]
            self.per = per
            self.imgs = sg.images(cfg, self.i0, nl, H, W)
            self.kp_np = synth.keypoints_random_batch(cfg, range(self.i0, self.i1), per, H, W, c["margin"],
                                                      c["scale_max"])
            self.kpi_np = np.repeat(np.arange(nl, dtype=np.int32), per)
            self.kps = torch.from_numpy(self.kp_np).to(dev)
            self.kpi = torch.from_numpy(self.kpi_np).to(dev)
            self.m = nl * per
            self.status = torch.empty(self.m, dtype=torch.uint8, device=dev)
            if cfg == 1:
                self.mb = bd.BadModel(*synth.bad_tests(1, 512))
                self.out = torch.empty((self.m, 16), dtype=torch.int32, device=dev)
                self.alg_bytes = nl * H * W + self.m * 64
                self.kunits = {"integral": nl * H * W, "bad_image": self.m}
            else:
                self.mb = bd.BadModel(*synth.bad_tests(4, self.K))
                self.mh = bd.HashSiftModel(synth.hashsift_matrix(4, self.N))
                self.out_bad = torch.empty((self.m, self.K // 32), dtype=torch.int32, device=dev)
                self.out_hs = torch.empty((self.m, self.N // 32), dtype=torch.int32, device=dev)
                self.alg_bytes = nl * H * W + self.m * (self.K + self.N) // 8
                self.kunits = {k: self.m for k in ("warp_nn", "bad_patch", "sift", "project", "zero_invalid")}
        else:
            self.n_total = n_override or c["n_patches"]
            self.i0, self.i1 = shard(self.n_total, rank, world)
            self.m = self.i1 - self.i0
            # digest unit: blocks of 1000 patches when every shard boundary is a multiple of it
            self.per = 1000 if all(shard(self.n_total, r, world)[0] % 1000 == 0 for r in range(world + 1)) \
                and self.n_total % 1000 == 0 else 1
            self.P = sg.patches(cfg, self.i0, self.m)
            if cfg == 2:
                self.mb = bd.BadModel(*synth.bad_tests(2, 256))
                self.out = torch.empty((self.m, 8), dtype=torch.int32, device=dev)
                self.kunits = {"bad_patch": self.m}
            else:
                self.mh = bd.HashSiftModel(synth.hashsift_matrix(3, 256))
                self.out = torch.empty((self.m, 8), dtype=torch.int32, device=dev)
                self.kunits = {"sift": self.m, "project": self.m}
            self.alg_bytes = self.m * (1024 + 32)
        torch.cuda.synchronize()

    def kbytes(self, name):
        if self.cfg == 4:
            return kernel_bytes(name, self.K, self.N)
        if self.cfg in (0, 1):
            return kernel_bytes(name, self.K)
        return kernel_bytes(name, 256, 256)

    def step(self):
        bd, cfg = self.bd, self.cfg
        if cfg in (0, 1):
            bd.bad_compute(self.mb, self.imgs, self.kps, self.kpi, out=self.out)
        elif cfg == 2:
            bd.bad_compute_patches(self.mb, self.P, out=self.out)
        elif cfg == 3:
            bd.hashsift_compute_patches(self.mh, self.P, out=self.out)
        else:
            bd.describe_warped(self.mb, self.mh, self.imgs, self.kps, self.kpi, out_bad=self.out_bad,
                               out_hs=self.out_hs, status=self.status)

    # ---- e2e: host buffers, copies inside the timed region ----
    def e2e_setup(self, n_images, chunk):
        torch = self.torch
        self.e2e_chunk = chunk
        if self.cfg == 4:
            ne = min(n_images, self.i1 - self.i0)
            per = self.per
            self.h_imgs = self.imgs[:ne].cpu().pin_memory()
            self.h_kps = torch.from_numpy(self.kp_np[:ne * per]).pin_memory()
            self.h_kpi = torch.from_numpy(self.kpi_np[:ne * per]).pin_memory()
            me = ne * per
            self.h_ob = torch.empty((me, self.K // 32), dtype=torch.int32).pin_memory()
            self.h_oh = torch.empty((me, self.N // 32), dtype=torch.int32).pin_memory()
            self.h_st = torch.empty(me, dtype=torch.uint8).pin_memory()
            self.e2e_units = me
            self.h2d = ne * self.c["H"] * self.c["W"] + me * 20
            self.d2h = me * (self.K + self.N) // 8
            self.e2e_sample = (f"{ne} images/rank/step from pinned host memory through bd_describe_warped_host "
                               f"(chunks of {chunk or -(-ne // 8)} images, copies overlapped with kernels)")
            return
        # configs[0..3]: the whole shard's inputs from pinned host memory, the device call,
        # the descriptors back to pinned host memory
        if self.cfg in (0, 1):
            self.h_in = [self.imgs.cpu().pin_memory(), self.kps.cpu().pin_memory()]
            self.d_in = [self.imgs, self.kps]
            if self.kpi is not None:
                self.h_in.append(self.kpi.cpu().pin_memory())
                self.d_in.append(self.kpi)
        else:
            self.h_in, self.d_in = [self.P.cpu().pin_memory()], [self.P]
        self.h_out = self.out.cpu().pin_memory()
        self.e2e_units = self.m
        self.h2d = sum(t.numel() * t.element_size() for t in self.h_in)
        self.d2h = self.h_out.numel() * 4
        self.e2e_sample = "the rank's whole shard: pinned H2D of the inputs, the C-ABI call, D2H of the descriptors"

    def e2e_step(self):
        if self.cfg == 4:
            self.bd.describe_warped_host(self.mb, self.mh, self.h_imgs, self.h_kps, self.h_kpi, out_bad=self.h_ob,
                                         out_hs=self.h_oh, status=self.h_st, chunk_images=self.e2e_chunk)
            return
        for d, h in zip(self.d_in, self.h_in):
            d.copy_(h, non_blocking=True)
        self.step()
        self.h_out.copy_(self.out, non_blocking=True)
        self.torch.cuda.current_stream().synchronize()

    # ---- per-image digests (sharding check) ----
    def digests(self):
        """per digest unit (an image; for patch workloads a block of `per` patches)"""
        if self.cfg == 4:
            return image_digests(self.out_bad.cpu().numpy(), self.out_hs.cpu().numpy(), self.per)
        return image_digests(self.out.cpu().numpy(), None, self.per)

    @property
    def digest_units(self):
        return self.n_total // self.per if self.cfg in (2, 3) else self.n_total

    def recompute_digest(self, i):
        """image/patch i alone through the same C-ABI call (a P = 1, single-unit batch)"""
        bd, sg, torch, c, dev = self.bd, self.sg, self.torch, self.c, self.dev
        if self.cfg in (1, 4):
            H, W, per = c["H"], c["W"], c["kp_per_image"]
            img = sg.images(self.cfg, i, 1, H, W)
            kp = torch.from_numpy(synth.keypoints_random_batch(self.cfg, [i], per, H, W, c["margin"],
                                                               c["scale_max"])).to(dev)
            if self.cfg == 4:
                ob, oh = bd.describe_warped(self.mb, self.mh, img, kp)
                return image_digests(ob.cpu().numpy(), oh.cpu().numpy(), per)[0]
            return image_digests(bd.bad_compute(self.mb, img, kp).cpu().numpy(), None, per)[0]
        if self.cfg == 0:
            return image_digests(bd.bad_compute(self.mb, self.imgs, self.kps).cpu().numpy(), None, self.per)[0]
        P = sg.patches(self.cfg, i * self.per, self.per)
        if self.cfg == 2:
            return image_digests(bd.bad_compute_patches(self.mb, P).cpu().numpy(), None, self.per)[0]
        return image_digests(bd.hashsift_compute_patches(self.mh, P).cpu().numpy(), None, self.per)[0]


def time_calls(fn, reps, torch):
    """3 warm-ups, `reps` back-to-back calls between two events (mean), then each call
    bracketed by its own events (median, best) — SURVEY §8(d) timing protocol."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    mean = e0.elapsed_time(e1) / reps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    each = sorted(a.elapsed_time(b) for a, b in ev)
    return mean, each[len(each) // 2], each[0]


def per_config(bd, sg, torch, hbm, reps, which=(0, 1, 2, 3)):
    """configs[0..3] on this GPU through their own C-ABI calls, each with its SM clocks."""
    res = {}
    for cfg in which:
        w = Workload(cfg, 0, 1, bd, sg, torch)
        # enough calls for >= ~0.4 s under the clock sampler (at least `reps`)
        _, t1, _ = time_calls(w.step, 3, torch)
        n = int(min(4000, max(reps, 0.2 / max(t1 / 1e3, 1e-6))))
        with ClockSampler(torch.cuda.current_device()) as clk:
            bd.profile_start()
            mean, med, best = time_calls(w.step, n, torch)
            prof = bd.profile_stop()
        calls = 3 + 2 * n
        r = {"workload": w.c["name"], "reps": n, "ms_median": round(med, 5), "ms_best": round(best, 5),
             "ms_mean_back_to_back": round(mean, 5), "Mdesc_s": round(w.m / med / 1e3, 2),
             "alg_bytes": int(w.alg_bytes), "hbm_frac": round(w.alg_bytes / (med / 1e3) / 1e9 / hbm, 4),
             "hbm_frac_best": round(w.alg_bytes / (best / 1e3) / 1e9 / hbm, 4),
             "kernels_ms": {k: round(v[1] / calls, 5) for k, v in prof.items()},
             "clocks": clk.summary()}
        if cfg == 0:  # a latency workload: one call's device time, direct and graph
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    w.step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                w.step()
            torch.cuda.synchronize()
            _, gmed, gbest = time_calls(g.replay, reps, torch)
            r.update({"latency_us": round(med * 1e3, 2), "graph_latency_us": round(gmed * 1e3, 2),
                      "note": "latency workload: 500 descriptors per call; report latency, not roofline %"})
        res[f"c{cfg}"] = r
        del w
        torch.cuda.empty_cache()
    return res


def issue_view(name, units_per_launch, ms_per_launch, sm_mhz, sms):
    """issue-slot view of a kernel bound on chip: ncu warp instructions per unit (profiles/
    ncu_traffic.json `inst_per_unit`, from smsp__inst_executed.sum) x units / duration against
    SMs x 4 SMSPs x 1 warp instruction per clock."""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(tp):
        return None
    t = json.load(open(tp)).get(name)
    if not t or "inst_per_unit" not in t:
        return None
    achieved = t["inst_per_unit"] * units_per_launch / (ms_per_launch / 1e3) / 1e9
    peak = sms * 4 * sm_mhz * 1e6 / 1e9
    return {"achieved": round(achieved, 1), "peak": round(peak, 1), "unit": "G warp-inst/s",
            "frac": round(achieved / peak, 4), "inst_per_unit": t["inst_per_unit"],
            "l1_data_pipe_frac": round(t.get("l1_data_pipe_pct", 0.0) / 100, 4),
            "source": f"ncu --set full, profiles/{t['tag']}_full.md; peak = SMs x 4 x {sm_mhz:.0f} MHz"}


# ----------------------------------------------------------------------------- main leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, choices=[0, 1, 2, 3, 4], default=4,
                    help="BASELINE.json config of the main line (default 4)")
    ap.add_argument("--images", type=int, default=None, help="override the image / patch count (debug)")
    ap.add_argument("--e2e-images", type=int, default=64, help="configs[4]: images per rank per e2e step")
    ap.add_argument("--e2e-chunk", type=int, default=0, help="images per pipeline chunk in the e2e call (0: n/8)")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--per-config-reps", type=int, default=20)
    ap.add_argument("--no-per-config", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        reference_main(args, rank, world)
        return

    import torch

    import paper_2108_08380_b200 as bd
    import synth.gpu as sg

    cfg = args.config
    w = Workload(cfg, rank, world, bd, sg, torch, n_override=args.images)
    info = WORKLOAD_INFO[cfg]

    for _ in range(args.warmup):
        w.step()
    torch.cuda.synchronize()
    barrier(world)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier(world)
        torch.cuda.synchronize()
        bd.profile_start()
        e0.record(stream)
        for _ in range(args.steps):
            w.step()
        e1.record(stream)
        torch.cuda.synchronize()
        prof = bd.profile_stop()
        barrier(world)
    ms_local = e0.elapsed_time(e1)
    ms = allreduce_max(ms_local, world)
    total_units = allreduce_sum(float(w.m), world)
    value = total_units * args.steps / (ms / 1e3) / 1e6
    if cfg == 4:
        assert int(w.status.sum().item()) == 0, "synthetic keypoints must all be valid"

    # ---- roofline of the dominant kernel (CUDA-event durations on the launching stream) ----
    hbm, _bf16, peak_src = load_peaks()
    sm_max = float(clk.max_mhz or 1965.0)
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    kernels = {}
    for name, (launches, kms) in prof.items():
        units = w.kunits.get(name, w.m) * args.steps
        per_launch_units = units / max(launches, 1)
        k = {"launches": launches, "ms_total": round(kms, 4), "ms_per_launch": kms / max(launches, 1),
             "share": kms / ms_local if ms_local > 0 else None,
             "units_per_launch": per_launch_units, "alg_bytes_per_launch": per_launch_units * w.kbytes(name)}
        k["alg_GBps"] = k["alg_bytes_per_launch"] / (k["ms_per_launch"] / 1e3) / 1e9
        k["hbm_frac"] = k["alg_GBps"] / hbm
        kernels[name] = k
    dom = max(kernels, key=lambda k: kernels[k]["ms_total"])
    d = kernels[dom]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        t = json.load(open(tp)).get(dom)
        if t:
            traffic = t["dram_bytes_per_unit"] * d["units_per_launch"]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(d["alg_GBps"], 1), "peak": hbm, "unit": "GB/s",
                "frac": round(d["hbm_frac"], 4), "traffic": traffic, "peak_source": peak_src,
                "alg_bytes_per_launch": d["alg_bytes_per_launch"],
                "step_frac": round(w.alg_bytes * args.steps / (ms_local / 1e3) / 1e9 / hbm, 4),
                "step_alg_bytes": int(w.alg_bytes)}
    iv = issue_view(dom, d["units_per_launch"], d["ms_per_launch"], clk.summary()["sm_mhz"] or sm_max, sms)
    if iv:
        roofline["issue_view"] = iv
    gpu_launches = int(allreduce_sum(float(sum(v["launches"] for v in kernels.values())), world))

    # ---- sharding check: per-image digests gathered from all ranks vs P = 1 recomputation ----
    dig = gather_digests(w.digests(), w.i0, world)
    sharding = None
    if rank == 0 and cfg != 0:
        sharding = check_sharding(dig, w.recompute_digest, sample_images(w.digest_units, world))
        sharding.update({"ranks": world, "unit": "image" if cfg in (1, 4) else f"block of {w.per} patches"})
    barrier(world)

    # ---- e2e through the public API with host buffers ----
    w.e2e_setup(args.e2e_images, args.e2e_chunk)
    for _ in range(args.warmup):
        w.e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        w.e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ems = allreduce_max(e0.elapsed_time(e1), world)
    e2e_val = allreduce_sum(float(w.e2e_units), world) * args.steps / (ems / 1e3) / 1e6
    e2e = {"value": round(e2e_val, 3), "unit": "Mdesc/s", "h2d_bytes_per_step": int(w.h2d * world),
           "d2h_bytes_per_step": int(w.d2h * world), "h2d_GBps": round(w.h2d * args.steps / (ems / 1e3) / 1e9, 2),
           "sample": w.e2e_sample}
    if cfg == 4:  # the e2e bound: a plain pinned host->device copy of the same image bytes (PCIe)
        d_scratch = torch.empty_like(w.h_imgs, device=w.dev)
        d_scratch.copy_(w.h_imgs, non_blocking=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            d_scratch.copy_(w.h_imgs, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        h2d_gbps = 3 * w.h_imgs.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
        del d_scratch
        e2e.update({"pcie_h2d_copy_GBps": round(h2d_gbps, 2), "frac_of_h2d_copy": round(e2e["h2d_GBps"] / h2d_gbps, 3)})

    # ---- CPU baseline: the oracle on the host cores (rank 0) ----
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        r, cores, sample, _ = oracle_rate(cfg, args.cpu_budget)
        cpu = {"value": r, "unit": "Mdesc/s", "cores": cores, "kind": "oracle", "sample": sample}

    # ---- configs[0..3] through their own calls, with clocks (N = 1 only) ----
    pc = None
    if rank == 0 and world == 1 and not args.no_per_config:
        del w
        torch.cuda.empty_cache()
        pc = per_config(bd, sg, torch, hbm, max(10, args.per_config_reps),
                        which=tuple(c for c in (0, 1, 2, 3)))
    barrier(world)

    if rank == 0:
        conf = {"workload": synth.CONFIGS[cfg]["name"] if not args.images else
                f"configs[{cfg}] with {args.images} units", **info["config"]}
        conf["parallelism"] = info["config"].get("parallelism", f"sharded x{world} by contiguous "
                                                 f"{'image' if cfg in (1, 4) else 'patch'} ranges, "
                                                 "no data-path collective")
        conf["l2"] = "inputs larger than L2 (126 MB); no flush needed" if cfg in (1, 2, 3, 4) else \
            "one 0.3 MB image: L2-resident between calls (a latency workload)"
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mdesc/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": info["scaling"], "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": conf, "per_gpu": round(value / world, 3),
            "roofline": roofline,
            "kernels": {k: {kk: (round(vv, 5) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                        for k, v in kernels.items()},
            "per_config": pc,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "sharding": sharding,
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
