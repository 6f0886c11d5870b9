#!/usr/bin/env python3
"""Summarise an ncu report: key throughput metrics, stall reasons, hottest SASS.
usage: python profiles/ncu_summary.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Active Warps Per SM",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Executed Instructions",
        "Compute (SM) Throughput", "L1/TEX Hit Rate"]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, vals = rows[0], rows[1], rows[2]
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"):
    if k in h:
        i = h.index(k)
        print(f"{k:60s} {vals[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = rows[2:]
ix = {k: i for i, k in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[ix[S]] or 0) for r in data)
print("stall samples", tot)
reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(float(r[ix[k]] or 0) for r in data) for k in reasons}
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]:
    print(f"  {k:28s} {100 * v / max(tot, 1):5.1f}%")
for r in sorted(data, key=lambda r: -int(r[ix[S]] or 0))[:top]:
    print(f"{int(r[ix[S]] or 0) * 100 / max(tot, 1):5.1f}% exec={r[ix['Instructions Executed']]:>12s}  "
          f"{r[ix['Source']][:80]}")
