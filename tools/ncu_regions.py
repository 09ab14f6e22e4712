#!/usr/bin/env python
"""Stall-sample share per SASS region of one kernel in an ncu report (source page), split at
barrier / TMEM / mbarrier instructions:  python tools/ncu_regions.py REP [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks = txt.split('"Kernel Name",')[1:]
for b in blocks:
    name = b.split("\n", 1)[0]
    if want not in name:
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr, data = rows[0], rows[1:]
    iS, iN, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[iN]) for r in data if r[iN].isdigit())
    print(name[:90], "samples", tot)
    acc, start, region = 0, 0, {}
    for k, r in enumerate(data):
        n = int(r[iN]) if r[iN].isdigit() else 0
        acc += n
        for h in stalls:
            v = r[hdr.index(h)]
            if v.isdigit():
                region[h] = region.get(h, 0) + int(v)
        s = r[iS].strip()
        if any(t in s for t in ("BAR.SYNC", "BAR.ARV", "SYNCS.PHASECHK", "EXIT")) or k == len(data) - 1:
            top = sorted(region.items(), key=lambda t: -t[1])[:4]
            seg = sum(region.values())
            if seg:
                print(f"  [{start:5d}-{k:5d}] {seg / tot * 100:5.1f}%  end: {s[:48]:48s} " +
                      " ".join(f"{h[6:]}={v / seg * 100:.0f}%" for h, v in top))
            start, region = k + 1, {}
