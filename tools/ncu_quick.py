#!/usr/bin/env python
"""Print the ncu_summary metric set for every kernel of a report (no files written).

  python tools/ncu_quick.py gpurun_out/x.ncu-rep"""
import csv
import io
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import METRICS, short  # noqa: E402

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(short(d["Kernel Name"]))
    for m, name in METRICS:
        if m in d:
            print(f"  {name:16s} {d[m]}")
