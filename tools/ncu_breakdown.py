#!/usr/bin/env python
"""Per-kernel L1 data-pipe breakdown of an ncu --set full report (per unit of work):
  python tools/ncu_breakdown.py gpurun_out/ncu_c2_r02b.ncu-rep [units_per_launch] [unit_name]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
uname = sys.argv[3] if len(sys.argv) > 3 else "unit"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
M = {
    "time_us": "gpu__time_duration.sum",
    "inst": "smsp__inst_executed.sum",
    "shared_wf": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "shared_ld_wf": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "shared_st_wf": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "ld_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "st_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "lgds_wf_per_sm": "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg",
    "pipe_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "tmem_ld": "smsp__sass_inst_executed_op_tmem_ldt.sum",
    "shfl": "smsp__sass_inst_executed_op_shfl.sum",
    "gst": "smsp__sass_inst_executed_op_global_st.sum",
    "gld": "smsp__sass_inst_executed_op_global_ld.sum",
    "sms": "device__attribute_multiprocessor_count",
}
idx = {k: (hdr.index(v) if v in hdr else None) for k, v in M.items()}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0]
    g = {k: (float(r[i].replace(",", "")) if i is not None and r[i] not in ("", "n/a") else None) for k, i in idx.items()}
    if g["time_us"] and g["time_us"] > 1e4:  # ns units
        pass
    out = {"kernel": name}
    for k, v in g.items():
        if v is None:
            continue
        if k in ("pipe_pct", "issue_pct", "sms", "time_us"):
            out[k] = v
        elif k == "lgds_wf_per_sm":
            out["lgds_wf_per_" + uname] = round(v * (g["sms"] or 148) / units, 2)
        else:
            out[k + "_per_" + uname] = round(v / units, 2)
    print(out)
