#!/usr/bin/env python
"""Summarise warp-stall samples of an ncu report by SASS instruction (run here, not on the box).

  python tools/ncu_hot.py gpurun_out/x.ncu-rep [top] [kernel-index]
Prints the total, barrier/sync instructions with the stall samples of the instruction after
them (ncu attributes a barrier wait to the next instruction), and the top-N instructions."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows, hdr = [], None
for x in csv.reader(out.splitlines()):
    if "Address" in x and "Source" in x:
        hdr = x
        continue
    if hdr and len(x) == len(hdr):
        rows.append(dict(zip(hdr, x)))
k = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[k] or 0) for r in rows)
print("total samples", tot, "instructions", len(rows))
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(int(r[h] or 0) for r in rows) for h in stall_cols}
print("by reason:", ", ".join(f"{h[6:]} {100 * v / tot:.1f}%" for h, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
for i, r in enumerate(rows):
    s = r["Source"].strip()
    if any(t in s for t in ("BAR.", "SYNCS.PHASECHK", "WARPSYNC")) and i + 1 < len(rows):
        n = int(rows[i + 1][k] or 0)
        print(f"  sync {i:5d} exec {r['Instructions Executed']:>9} next-stall {n:7d} ({100 * n / tot:4.1f}%)  {s[:60]}")
print("top instructions:")
for i, r in sorted(enumerate(rows), key=lambda t: -int(t[1][k] or 0))[:top]:
    s = int(r[k] or 0)
    print(f"  {i:5d} {s:7d} {100 * s / tot:4.1f}%  exec {r['Instructions Executed']:>9}  {r['Source'].strip()[:70]}")
