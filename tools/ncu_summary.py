#!/usr/bin/env python
"""Summarise ncu output into tracked files under profiles/.

  python tools/ncu_summary.py --tag r01 --launches gpurun_out/launches_r01.csv \
      --rep gpurun_out/prof_r01.ncu-rep --units 256000

* launches CSV (``ncu --metrics gpu__time_duration.sum --csv``): per-kernel launch count,
  total device time and SHARE of the profiled program (cold-cache, serialised: compare
  shares, not absolutes) -> profiles/<tag>_launches.md
* full capture (``ncu --set full``): per kernel duration, DRAM bytes read/written, DRAM and SM
  throughput, issue activity, occupancy, shared-memory wavefronts and bank conflicts,
  tensor-pipe activity -> profiles/<tag>_full.md; DRAM bytes per unit (keypoint/patch) ->
  profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp inst"),
]


def short(name: str) -> str:
    n = name.split("(")[0]
    n = n.replace("<unnamed>::", "").replace("void ", "")
    return n.split("::")[-1].split("<")[0]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + float(r[vi].replace(",", "")))
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[label] = (r[i], units[i])
        res.append(d)
    return res


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--units", type=float, default=None, help="units (keypoints/patches) per profiled launch")
    ap.add_argument("--cmd", default="", help="command line that was profiled (recorded)")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.launches:
        agg = launches(a.launches)
        tot = sum(t for _, t in agg.values())
        lines = [f"# ncu launch list — {a.tag}", "", f"command: `{a.cmd}`", "",
                 "ncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares).", "",
                 "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| {k} | {n} | {t / 1e6:.3f} | {t / tot:.3f} |")
        open(os.path.join(ROOT, "profiles", f"{a.tag}_launches.md"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    if a.rep:
        res = full(a.rep)
        labels = [l for _, l in METRICS]
        lines = [f"# ncu --set full — {a.tag}", "", f"command: `{a.cmd}`", "",
                 f"units per launch: {a.units}", "",
                 "| kernel | " + " | ".join(labels) + " |", "|---|" + "---|" * len(labels)]
        traffic = {}
        for d in res:
            cells = []
            for l in labels:
                v = d.get(l)
                cells.append(f"{v[0]} {v[1]}".strip() if v else "")
            lines.append(f"| {d['kernel']} | " + " | ".join(cells) + " |")
            if a.units and "dram read" in d:
                b = to_bytes(*d["dram read"]) + to_bytes(*d["dram write"])
                ent = {"dram_bytes_per_launch": b, "dram_bytes_per_unit": b / a.units, "tag": a.tag}
                if d.get("L1 data-pipe %"):
                    ent["l1_data_pipe_pct"] = float(d["L1 data-pipe %"][0])
                if d.get("issue %"):
                    ent["issue_pct"] = float(d["issue %"][0])
                if d.get("warp inst"):
                    ent["inst_per_unit"] = round(float(d["warp inst"][0].replace(",", "")) / a.units, 2)
                traffic[d["kernel"].replace("_kernel", "").replace("_tc", "")] = ent
        open(os.path.join(ROOT, "profiles", f"{a.tag}_full.md"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
        if traffic:
            p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
            old = json.load(open(p)) if os.path.exists(p) else {}
            old.update(traffic)
            json.dump(old, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
