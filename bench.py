#!/usr/bin/env python
"""bench.py — B200 throughput of the batched BAD / HashSIFT extraction path.

Default workload (one "step" = one pass of the whole hot path):
BASELINE.json configs[4] — 8192 seeded 3840x2160 smoothed-noise images (67.9 GB), 4000
keypoints each (scale log-U[1,6], angle U[0,2pi)); every keypoint gets a nearest-neighbour
32x32 patch (a5, with the a2 sample-point rule), BAD-512 on the warped patch (a1 on-chip
integral, a3, a4) and HashSIFT-256 (a6-a9), through the C ABI call bd_describe_warped.
Images are sharded evenly across ranks (total work fixed -> "scaling": "strong"); there is
no collective in the data path (NCCL only for the barrier and the max-over-ranks timing).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 0..4] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line (rank 0).  `value` = Mdescriptors/s over the whole job where one
descriptor = one keypoint's BAD-512 + HashSIFT-256 pair (configs[4]); `roofline` is the
dominant kernel's algorithmic bytes / its CUDA-event duration against the measured HBM
copy bandwidth (MEASURED_PEAKS.json); `cpu_baseline` is the CPU oracle (oracle/) timed on
a bounded sample on the host cores; `e2e` repeats the metric through the host-buffer C ABI
call bd_describe_warped_host with pinned host buffers (H2D of images+keypoints and D2H of the
descriptors inside the timed region, overlapped with the kernels chunk by chunk) on a
per-step sample of images.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "Mdescriptors/s per GPU (BAD-256, HashSIFT-256) and % of HBM roofline, 1/2/4/8 B200"

# algorithmic bytes per unit per kernel: what the kernel must
# read and write in HBM by definition of its step, not what it happens to move.
def kernel_bytes(name: str, K: int = 512, N: int = 256) -> float:
    return {
        "warp_nn": 1024 + 1024 + 16 + 4 + 1,   # sampled image bytes + patch out + kp + kp_image + status
        "bad_patch": 1024 + K / 8,              # patch in, bits out
        "sift": 1024 + 512,                     # patch in, 128 fp32 out
        "project": 512 + N / 8,                 # 128 fp32 in, bits out
        "zero_invalid": 1 + 4,                  # status + a word (upper bound)
        "integral": 1 + 4 + 4 + 4,              # per pixel: u8 in, u32 out, column pass r+w
        "bad_image": 1037 + K / 8,              # per keypoint
    }.get(name, 0.0)


# algorithmic ALU operations per unit for the kernels bound by arithmetic issue rather than
# HBM: SIFT = SURVEY §8(d)'s "per pixel ~ 40 flops + 1 sqrt + 1 atan2 +
# 1 exp" over 1024 pixels, plus ~4 ops per entry for normalise / clip / renormalise.
def kernel_ops(name: str) -> float:
    return {"sift": 1024 * 43 + 4 * 128}.get(name, 0.0)


def alu_peak(sm_mhz: float):
    """FP32 lane-operations per second: 148 SMs x 4 SMSPs x 32 lanes x one instruction per
    clock (B200_PROFILING.md: 148 SMs, clocks.max.sm 1965 MHz)."""
    try:
        import torch
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    except Exception:  # pragma: no cover
        sms = 148
    return sms * 128 * sm_mhz * 1e6


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
            self._stop.wait(0.05)

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
            torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=world)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def shard(n: int, rank: int, world: int):
    return (n * rank) // world, (n * (rank + 1)) // world


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


def reference_main(args, rank, world):
    """--impl reference: the CPU oracle is this tier's reference arm."""
    if rank != 0:
        return
    per_step_budget = max(1.0, 150.0 / (args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_c4_rate(per_step_budget / 4)
    rates, ms = [], []
    for _ in range(args.steps):
        r, cores, n, reps = oracle_c4_rate(per_step_budget)
        rates.append(r)
        ms.append(n * reps / (r * 1e6) * 1e3)
    value = float(np.median(rates))
    c = synth.CONFIGS[4]
    sample = f"configs[4] image 0, first {n} keypoints x {reps} reps per step (warp+BAD-512+HashSIFT-256)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Mdesc/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(ms)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": c["name"], "images": c["n_images"], "H": c["H"],
                                             "W": c["W"], "kp_per_image": c["kp_per_image"], "K": c["K"],
                                             "N": c["N"]},
            "cpu_baseline": {"value": value, "unit": "Mdesc/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "Mdesc/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- main leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--images", type=int, default=None, help="override configs[4] image count (debug)")
    ap.add_argument("--e2e-images", type=int, default=64, help="images per rank per e2e step")
    ap.add_argument("--e2e-chunk", type=int, default=0, help="images per pipeline chunk in the e2e call (0: n/8)")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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

    c = dict(synth.CONFIGS[4])
    n_img = args.images or c["n_images"]
    H, W, per, K, N = c["H"], c["W"], c["kp_per_image"], c["K"], c["N"]
    i0, i1 = shard(n_img, rank, world)
    nl = i1 - i0
    dev = torch.device("cuda", torch.cuda.current_device())

    # ---- inputs resident in HBM before the timed region (generation is not timed) ----
    imgs = sg.images(4, i0, nl, H, W)
    kp_np = synth.keypoints_random_batch(4, range(i0, i1), per, H, W, c["margin"], c["scale_max"])
    kpi_np = np.repeat(np.arange(nl, dtype=np.int32), per)
    kps = torch.from_numpy(kp_np).to(dev)
    kpi = torch.from_numpy(kpi_np).to(dev)
    pairs, radii, thr = synth.bad_tests(4, K)
    mb, mh = bd.BadModel(pairs, radii, thr), bd.HashSiftModel(synth.hashsift_matrix(4, N))
    m = nl * per
    out_bad = torch.empty((m, K // 32), dtype=torch.int32, device=dev)
    out_hs = torch.empty((m, N // 32), dtype=torch.int32, device=dev)
    status = torch.empty(m, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def step():
        bd.describe_warped(mb, mh, imgs, kps, kpi, out_bad=out_bad, out_hs=out_hs, status=status)

    for _ in range(args.warmup):
        step()
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
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        prof = bd.profile_stop()
        barrier(world)
    ms_local = e0.elapsed_time(e1)
    ms = allreduce_max(ms_local, world)
    total_kp = allreduce_sum(float(m), world)
    value = total_kp * args.steps / (ms / 1e3) / 1e6
    assert int(status.sum().item()) == 0, "synthetic keypoints must all be valid"

    # ---- roofline of the dominant kernel (CUDA-event durations on the launching stream) ----
    hbm, _bf16, peak_src = load_peaks()
    sm_max = float(clk.max_mhz or 1965.0)
    kernels = {}
    for name, (launches, kms) in prof.items():
        units = m * args.steps  # every kernel of the warped path runs once per keypoint
        per_launch_units = units / max(launches, 1)
        kernels[name] = {"launches": launches, "ms_total": round(kms, 4), "ms_per_launch": kms / max(launches, 1),
                         "share": kms / ms_local if ms_local > 0 else None,
                         "alg_bytes_per_launch": per_launch_units * kernel_bytes(name, K, N)}
        kernels[name]["alg_GBps"] = kernels[name]["alg_bytes_per_launch"] / (kernels[name]["ms_per_launch"] / 1e3) / 1e9
        kernels[name]["hbm_frac"] = kernels[name]["alg_GBps"] / hbm
    dom = max(kernels, key=lambda k: kernels[k]["ms_total"])
    d = kernels[dom]
    achieved = d["alg_bytes_per_launch"] / (d["ms_per_launch"] / 1e3) / 1e9   # GB/s
    traffic = None
    ncu_view = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        t = json.load(open(tp)).get(dom)
        if t:
            traffic = t["dram_bytes_per_unit"] * d["alg_bytes_per_launch"] / kernel_bytes(dom, K, N)
            if "l1_data_pipe_pct" in t:  # the unit that binds these kernels
                ncu_view = {"l1_data_pipe_frac": round(t["l1_data_pipe_pct"] / 100, 4),
                            "issue_frac": round(t.get("issue_pct", 0.0) / 100, 4),
                            "source": f"ncu --set full, profiles/{t['tag']}_full.md"}
    step_bytes = m * (2074 + K / 8 + N / 8)   # image bytes per kp + bits written
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic, "peak_source": peak_src,
                "step_frac": round(step_bytes * args.steps / (ms_local / 1e3) / 1e9 / hbm, 4)}
    if ncu_view:
        roofline["ncu_view"] = ncu_view
    if kernel_ops(dom):  # issue-bound kernel: report against the ALU peak
        units_per_launch = m * args.steps / max(d["launches"], 1)
        ops = units_per_launch * kernel_ops(dom) / (d["ms_per_launch"] / 1e3) / 1e9
        peak_ops = alu_peak(sm_max) / 1e9
        roofline.update({"bound": "alu", "achieved": round(ops, 1), "peak": round(peak_ops, 1), "unit": "Gop/s",
                         "frac": round(ops / peak_ops, 4),
                         "peak_source": f"derived: SMs x 128 FP32 lanes x {sm_max:.0f} MHz (DESIGN.md §6)",
                         "hbm_view": {"achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                                      "frac": round(achieved / hbm, 4), "peak_source": peak_src}})
    gpu_launches = int(allreduce_sum(float(sum(v["launches"] for v in kernels.values())), world))

    # ---- e2e: the host-buffer C ABI call (bd_describe_warped_host), pinned host buffers,
    # host<->device copies inside the timed region, overlapped with the kernels per chunk ----
    ne = min(args.e2e_images, nl)
    h_imgs = imgs[:ne].cpu().pin_memory()
    h_kps = torch.from_numpy(kp_np[:ne * per]).pin_memory()
    h_kpi = torch.from_numpy(kpi_np[:ne * per]).pin_memory()
    me = ne * per
    h_ob = torch.empty((me, K // 32), dtype=torch.int32).pin_memory()
    h_oh = torch.empty((me, N // 32), dtype=torch.int32).pin_memory()
    h_st = torch.empty(me, dtype=torch.uint8).pin_memory()

    def e2e_step():
        bd.describe_warped_host(mb, mh, h_imgs, h_kps, h_kpi, out_bad=h_ob, out_hs=h_oh, status=h_st,
                                chunk_images=args.e2e_chunk)

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ems = allreduce_max(e0.elapsed_time(e1), world)
    e2e_val = allreduce_sum(float(me), world) * args.steps / (ems / 1e3) / 1e6
    h2d = ne * H * W + me * 20
    d2h = me * (K + N) // 8
    # the e2e bound: a plain pinned host->device copy of the same image bytes (PCIe)
    d_scratch = torch.empty_like(h_imgs, device=dev)
    d_scratch.copy_(h_imgs, non_blocking=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(3):
        d_scratch.copy_(h_imgs, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    h2d_gbps = 3 * h_imgs.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
    del d_scratch
    e2e_gbps = h2d * args.steps / (ems / 1e3) / 1e9

    # ---- CPU baseline: the oracle on the host cores (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r, cores, n_s, reps = oracle_c4_rate(args.cpu_budget)
        cpu = {"value": r, "unit": "Mdesc/s", "cores": cores, "kind": "oracle",
               "sample": f"configs[4] image 0, first {n_s} keypoints x {reps} (NN warp + BAD-512 + HashSIFT-256, fp64)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mdesc/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "u8/u32 integer (BAD), f32 (SIFT, projection)", "data": "synthetic",
            "config": {"workload": c["name"] if n_img == c["n_images"] else f"configs[4] with {n_img} images",
                       "images": n_img, "H": H, "W": W, "kp_per_image": per, "keypoints": int(total_kp),
                       "K": K, "N": N, "descriptor": "one keypoint's BAD-512 + HashSIFT-256 pair",
                       "parallelism": f"image-sharded x{world}, no data-path collective",
                       "l2": "inputs (67.9 GB of images) larger than L2; no flush needed"},
            "per_gpu": round(value / world, 3),
            "roofline": roofline,
            "kernels": {k: {kk: (round(vv, 5) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                        for k, v in kernels.items()},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_val, 3), "unit": "Mdesc/s", "h2d_bytes_per_step": int(h2d * world),
                    "d2h_bytes_per_step": int(d2h * world),
                    "h2d_GBps": round(e2e_gbps, 2), "pcie_h2d_copy_GBps": round(h2d_gbps, 2),
                    "frac_of_h2d_copy": round(e2e_gbps / h2d_gbps, 3),
                    "sample": f"{ne} images/rank/step from pinned host memory through bd_describe_warped_host "
                              f"(chunks of {args.e2e_chunk or -(-ne // 8)} images, copies overlapped with kernels)"},
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
