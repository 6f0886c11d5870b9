#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel count, mean and total time, and each kernel's share of the total.
usage: python profiles/launch_summary.py launches.csv [skip_first_n]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = collections.defaultdict(list)
for r in rows[1 + skip:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    t = float(d["Metric Value"]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                     "msecond": 1e3, "nsecond": 1e-3}.get(d["Metric Unit"], 1e-3)
    agg[d["Kernel Name"].split("(")[0][:70]].append(t)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'n':>5s} {'mean us':>10s} {'total us':>11s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} {len(v):5d} {sum(v) / len(v):10.1f} {sum(v):11.1f} {100 * sum(v) / tot:5.1f}%")
