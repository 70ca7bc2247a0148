#!/usr/bin/env python
"""profiles/<tag>_ncu_traffic_<cfg>.json from an ncu --set full capture of bench.py.

For the first captured launch of each hot kernel: dram read + write bytes, duration, and the
algorithmic units of that launch (the same units cwg_kernel_units counts), so bench.py can
report `traffic` per launch of any size.
usage: python scripts/ncu_traffic.py <rep> <config> <out.json>"""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2202_07569_b200 import configs  # noqa: E402

rep, cname, out = sys.argv[1], sys.argv[2], sys.argv[3]
cfg = configs.config(cname)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = {x: i for i, x in enumerate(rows[0])}
units_row = rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
         "ns": 1e-3, "nsecond": 1e-3, "": 1}


def num(r, k):
    return float(r[h[k]].replace(",", "")) * SCALE.get(units_row[h[k]], 1)


first = {}
for r in rows[2:]:
    name = r[h["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").replace("cwgpu::", "").strip()
    first.setdefault(name, r)
# the aux / MAC basis of this configuration, from the library itself (no stale labels)
from paper_2202_07569_b200 import Context  # noqa: E402

_info = Context(cfg.N, cfg.primes, cfg.t)
_info.load_db(configs.perfect_map(range(2), cfg.m, cfg.k), None, n_total=cfg.n, m=cfg.m)
J, Mm = _info.info().J, _info.info().Mm
res = {"source": rep.split("/")[-1], "config": cname, "J": J, "Mm": Mm}
P = None
if "k_tensor_intt_r" in first:
    P = num(first["k_tensor_intt_r"], "launch__grid_size") / (3 * J)
for name, r in first.items():
    dram = num(r, "dram__bytes_read.sum") + num(r, "dram__bytes_write.sum")
    grid = num(r, "launch__grid_size")
    if name == "k_tensor_intt_r":
        key, units = "k_tensor_intt", grid
    elif name == "k_ntt32r_sel3":
        key, units = name, grid
    elif name.startswith("k_round") and P:
        key, units = "k_round_tma", P * 3 * cfg.N
    elif name.startswith("k_mac2") and P:
        key, units = "k_mac", P * (cfg.s + 3) * Mm * cfg.N * 4
    elif name.startswith("k_ntt_mac"):
        # units = selection polynomials transformed (rows x components x MAC primes); the grid
        # covers chunks of rows, so take the tile's P from the tensor launch
        if not P:
            continue
        key, units = "k_ntt_mac", P * 3 * Mm
    else:
        continue
    res[key] = {"dram_bytes_per_launch": dram, "units_per_launch": units, "dram_bytes_per_unit": dram / units,
                "duration_us": num(r, "gpu__time_duration.sum")}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
