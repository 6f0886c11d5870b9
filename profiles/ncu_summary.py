#!/usr/bin/env python3
"""Summarise an ncu report: key throughput metrics, stall reasons, hottest SASS.
usage: python profiles/ncu_summary.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

import gzip
import os

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def page(name, *extra):
    """From a .ncu-rep, or from the CSVs profiles/ncu_export.sh wrote (prefix)."""
    if rep.endswith(".ncu-rep"):
        return subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra],
                              capture_output=True, text=True).stdout
    key = {"details": "details.csv", "raw": "raw.csv"}.get(name)
    if key is None:
        key = "cudasass.csv.gz" if "cuda,sass" in extra else "sass.csv.gz"
    path = f"{rep}.{key}"
    if path.endswith(".gz"):
        return gzip.open(path, "rt").read()
    return open(path).read()


raw = page("details")
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
raw = page("raw")
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
src = page("source", "--print-source", "sass")
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

# per source line (cuda,sass view)
try:
    src = page("source", "--print-source", "cuda,sass")
    rows = list(csv.reader(io.StringIO(src)))
    cur, line, agg = None, None, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0]:
            line = (cur, r[0], r[1][:80])
            continue
        try:
            s_ = int(r[4] or 0)
        except (ValueError, IndexError):
            continue
        agg[line] = agg.get(line, 0) + s_
    tot = max(sum(agg.values()), 1)
    print("--- hottest source lines")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]} {k[2]}")
except Exception as ex:  # noqa
    print("no cuda,sass view:", ex)
