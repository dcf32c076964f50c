"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel launch:
python tools/launch_table.py launches.csv"""
import csv
import sys
from collections import OrderedDict

rows = OrderedDict()
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    key = (r["ID"], r["Kernel Name"])
    d = rows.setdefault(key, {})
    v = float(r["Metric Value"].replace(",", ""))
    d[r["Metric Name"]] = v
tot = 0.0
for (i, name), d in rows.items():
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    rd, wr = d.get("dram__bytes_read.sum", 0) / 1e6, d.get("dram__bytes_write.sum", 0) / 1e6
    print(f"{i:>4} {t:8.1f} us  rd {rd:8.1f} MB  wr {wr:8.1f} MB  {(rd + wr) / max(t, 1e-9):6.2f} TB/s  {name[:90]}")
print(f"total {tot:.1f} us over {len(rows)} launches")
