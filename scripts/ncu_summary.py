#!/usr/bin/env python
"""Summarise an ncu report: per kernel duration, IPC, occupancy, pipe use, DRAM, stalls.
usage: python scripts/ncu_summary.py gpurun_out/<tag>.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
want = {
    "dur_us": "gpu__time_duration.sum",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "fmaheavy_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smem_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "warp_inst": "smsp__inst_executed.sum",
}
stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if pat and not pat.search(name):
        continue
    vals = {k: r[col[v]] for k, v in want.items() if v in col}
    # ncu prints each metric in its own unit (row 1 of the CSV): bring bytes to MB and times to us
    units = rows[1]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
    tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
    for k in ("dram_rd_MB", "dram_wr_MB"):
        if k in vals:
            vals[k] = f"{float(vals[k].replace(',', '')) * scale.get(units[col[want[k]]], 1.0):.1f}"
    if "dur_us" in vals:
        vals["dur_us"] = f"{float(vals['dur_us'].replace(',', '')) * tscale.get(units[col[want['dur_us']]], 1.0):.1f}"
    st = sorted(((float(r[col[h]] or 0), h.split("stalled_")[1].split("_per")[0]) for h in stall), reverse=True)[:5]
    print(name[:60])
    print("   " + "  ".join(f"{k}={v}" for k, v in vals.items()))
    print("   stalls/issue: " + "  ".join(f"{n}={v:.2f}" for v, n in st))
