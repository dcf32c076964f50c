"""Summarise ncu outputs into profiles/: a launch list (per-kernel count, time, share)
and the dominant kernel's counters (dram bytes -> bench.py's roofline.traffic).

usage: python tools/summarize_ncu.py launches.csv dominant.ncu-rep FAM R A C WR WC M K N BATCH OUT_PREFIX
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path


def launches(path):
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as fh:
        rows = [r for r in csv.reader(l for l in fh if l.startswith('"'))]
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:90]
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[ui], 1e-6)
        per[name][0] += 1
        per[name][1] += float(r[vi].replace(",", "")) * scale
    return per


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def main():
    lpath, rep, fam, *nums, prefix = sys.argv[1:]
    cfg, prob = [int(x) for x in nums[:5]], [int(x) for x in nums[5:9]]
    per = launches(lpath)
    total = sum(t for _, t in per.values())
    ours = {k: v for k, v in per.items() if any(s in k for s in ("f1_kernel", "f0_kernel", "tc_gemm", "im2col", "maxpool"))}
    lines = ["| kernel | launches | total ms (ncu, serialised) | share of all launches |", "|---|---|---|---|"]
    for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.3f} | {t / total:.3f} |")
    m = raw_metrics(rep)
    get = lambda k: m.get(k, ("", "n/a"))  # noqa: E731
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = sum(float(get(k)[1]) * scale.get(get(k)[0], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    M, K, N, Bt = prob
    es = 2 if fam == "bf16" else 4
    algo = Bt * (M * K * es + K * N * es + M * N * 4)
    rec = {"variant": cfg, "family": fam, "problem": prob, "dram_bytes_per_launch": dram,
           "algorithmic_bytes_per_launch": algo, "kernel": get("Kernel Name")[1],
           "ncu_duration": get("gpu__time_duration.sum"),
           "fma_pipe_pct": get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active")[1],
           "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active")[1],
           "registers": get("launch__registers_per_thread")[1],
           "smem_bank_conflicts_ld": get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum")[1]}
    Path(prefix + "_dominant.json").write_text(json.dumps(rec, indent=1) + "\n")
    Path(prefix + "_launches.md").write_text("\n".join(lines) + "\n")
    print(json.dumps(rec, indent=1))
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()
