#!/usr/bin/env python
"""Per-opcode warp-stall attribution from an ncu report's source page (SASS view).
usage: python scripts/ncu_stalls.py <rep> <kernel-regex> [top-lines]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern,
                      "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[start]
c = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
n = collections.Counter()
lines = []
for r in rows[start + 1:]:
    if len(r) < len(hdr) or r[0] == "Address":
        continue
    src = r[c["Source"]].strip()
    parts = src.split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    op = op.split(".")[0]
    ex = float(r[c["Instructions Executed"]] or 0)
    n[op] += ex
    s_line = 0.0
    for s in stalls:
        v = float(r[c[s]] or 0)
        tot[s] += v
        byop[op][s] += v
        s_line += v
    lines.append((s_line, r[0], src, {s: float(r[c[s]] or 0) for s in stalls}))
T = sum(tot.values()) or 1
print("total samples", T)
for s, v in tot.most_common(12):
    print(f"{s:28s} {100 * v / T:5.1f}%")
E = sum(n.values()) or 1
print("--- by opcode: share of stall samples / share of executed warp-instructions [top stalls]")
for o in sorted(byop, key=lambda o: -sum(byop[o].values()))[:14]:
    sv = sum(byop[o].values())
    tops = ", ".join(f"{k[6:]} {100 * v / T:.1f}" for k, v in byop[o].most_common(4))
    print(f"{o:10s} {100 * sv / T:5.1f}%  inst {100 * n[o] / E:5.1f}%  [{tops}]")
if top:
    print("--- hottest instructions")
    for s_line, addr, src, d in sorted(lines, reverse=True)[:top]:
        tops = ", ".join(f"{k[6:]} {100 * v / T:.1f}" for k, v in collections.Counter(d).most_common(2))
        print(f"{100 * s_line / T:5.1f}%  {addr}  {src[:70]:70s} [{tops}]")
