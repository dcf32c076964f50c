"""Digest of one `ncu --set full` capture (exported on the GPU box as `--page raw --csv`
and `--page source --csv`, gzip'd): the counters the DESIGN/profiles tables cite, the
top warp-stall reasons and the SASS opcode mix (executed and sampled).
usage: python tools/ncu_digest.py NAME_raw.csv [NAME_src.csv.gz] > digest.json"""
import collections
import csv
import gzip
import json
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_inst_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block_dynamic",
    "occupancy_limit_smem": "launch__occupancy_limit_shared_mem",
    "occupancy_limit_regs": "launch__occupancy_limit_registers",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "cluster": "launch__cluster_size",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smem_ld_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smem_ld_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "inst_executed": "smsp__inst_executed.sum",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3,
         "us": 1, "ns": 1e-3, "ms": 1e3}


def raw(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {k: (uu, vv) for k, uu, vv in zip(h, u, v)}
    out = {"kernel": d.get("Kernel Name", ("", ""))[1]}
    for name, key in KEYS.items():
        if key not in d or d[key][1] in ("", "n/a"):
            continue
        unit, val = d[key]
        try:
            x = float(val.replace(",", ""))
        except ValueError:
            continue
        if name.startswith("dram_r") or name.startswith("dram_w"):
            x *= SCALE.get(unit, 1)
        elif name == "duration_us":
            x *= SCALE.get(unit, 1)
        out[name] = x
    stalls = {}
    for k, (_, val) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(val)
            except ValueError:
                pass
    out["stalls_per_issue_top"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    return out


def source(path):
    rows = list(csv.reader(gzip.open(path, "rt")))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    ex, smp = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) < len(h) or not r[ix["Source"]].strip():
            continue
        toks = r[ix["Source"]].split()
        op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
        ex[op] += int(r[ix["Instructions Executed"]] or 0)
        smp[op] += int(r[ix["# Samples"]] or 0)
    te, ts = sum(ex.values()) or 1, sum(smp.values()) or 1
    return {"executed_mix": {k: round(v / te, 4) for k, v in ex.most_common(8)},
            "sampled_mix": {k: round(v / ts, 4) for k, v in smp.most_common(8)}}


if __name__ == "__main__":
    rec = raw(sys.argv[1])
    if len(sys.argv) > 2:
        rec.update(source(sys.argv[2]))
    print(json.dumps(rec, indent=1))
