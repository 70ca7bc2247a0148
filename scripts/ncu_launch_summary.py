#!/usr/bin/env python
"""Per-kernel totals and shares from an ncu --metrics gpu__time_duration.sum launch list (CSV).
usage: python scripts/ncu_launch_summary.py <launches.csv> [answers-in-run]"""
import collections
import csv
import sys

path = sys.argv[1]
answers = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = []
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
rd = csv.reader(lines)
hdr = next(rd)
c = {h: i for i, h in enumerate(hdr)}
tot = collections.Counter()
cnt = collections.Counter()
unit = None
for r in rd:
    if r[c["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[c["Kernel Name"]].split("(")[0].replace("void ", "").replace("cwgpu::", "")
    v = float(r[c["Metric Value"]].replace(",", ""))
    unit = r[c["Metric Unit"]]
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':40s} {'launches':>9s} {'total ms':>10s} {'ms/answer':>10s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k[:40]:40s} {cnt[k]:9d} {v:10.2f} {v / answers:10.2f} {100 * v / T:6.1f}%")
print(f"{'all':40s} {sum(cnt.values()):9d} {T:10.2f} {T / answers:10.2f}")
