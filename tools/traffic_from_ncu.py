"""Join ncu per-launch DRAM counters with tools/bench_layers_once.py's launch order ->
profiles/dominant_kernel_traffic.json (list of {variant, problem, dram_bytes_per_launch})."""
import csv
import json
import sys

log, csvpath, out = sys.argv[1:4]
order = json.loads(next(l for l in open(log) if l.startswith("ORDER "))[6:])
rows = [r for r in csv.reader(l for l in open(csvpath) if l.startswith('"'))]
hdr = rows[0]
ii, ki, mi, ui, vi = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
per = {}
for r in rows[1:]:
    if not any(s in r[ki] for s in ("f1_kernel", "f0_kernel", "tc_gemm")):
        continue
    d = per.setdefault(int(r[ii]), {"kernel": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
launches = [per[i] for i in sorted(per)]
assert len(launches) == len(order), (len(launches), len(order))
recs = []
for o, l in zip(order, launches):
    o = dict(o)
    o["dram_bytes_per_launch"] = l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
    o["kernel"] = l["kernel"][:80]
    recs.append(o)
json.dump({"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (one launch per unique "
                     "(variant, problem) of bench.py's step, tools/bench_layers_once.py)", "launches": recs},
          open(out, "w"), indent=1)
print(json.dumps(recs, indent=1)[:2000])
