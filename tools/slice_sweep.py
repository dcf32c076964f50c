"""Forced k-slice sweep (planner re-fit data): for every S in a list, a fresh process with
KPGEMM_FORCE_SLICES=S times (config, problem) cells with the sweep protocol
(CudaEventTimer); S=0 is the planner's own choice.  Prints one JSON line per cell.
usage: python tools/slice_sweep.py [S list, e.g. 0,1,2,3,4,5,6,8,12,16] [min_ms]"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SIMT_CFGS = [(8, 8, 8, 16, 8), (8, 8, 8, 16, 16), (4, 2, 8, 16, 8), (8, 1, 8, 8, 16), (8, 4, 4, 8, 16),
             (4, 8, 8, 8, 8), (4, 8, 8, 16, 8), (8, 1, 2, 1, 64), (8, 4, 2, 1, 64), (4, 4, 2, 1, 64),
             (2, 4, 8, 8, 8), (8, 4, 4, 8, 32), (4, 1, 2, 8, 8), (1, 4, 1, 1, 64)]


def problems():
    sys.path.insert(0, str(ROOT))
    from paper_2008_13145_b200 import shapes
    rows = shapes.network_problems("vgg16")
    # under-filled / few-wave rows: everything below ~6 waves of 128x64 tiles
    return [p for p in rows if (p.m + 127) // 128 * ((p.n + 63) // 64) < 3 * 148 * 4 and p.k >= 512]


def child(S, min_ms):
    sys.path.insert(0, str(ROOT))
    from paper_2008_13145_b200 import gemm
    from paper_2008_13145_b200.dataset import KernelConfig
    from paper_2008_13145_b200.sweep import CudaEventTimer
    probs = problems()
    timer = CudaEventTimer("simt", probs, min_ms=min_ms)
    idx = {c.as_tuple(): i for i, c in enumerate(timer.configs)}
    for p in probs:
        for c in SIMT_CFGS:
            try:
                g, ms, _ = timer(p, idx[c])
            except Exception as e:  # a forced cluster size the device cannot schedule
                print(json.dumps({"S": S, "problem": [p.m, p.k, p.n], "config": c, "error": str(e)[:120]}))
                continue
            plan = gemm.k_slice_plan(KernelConfig(*c), p)
            print(json.dumps({"S": S, "problem": [p.m, p.k, p.n], "config": c, "gflops": round(g, 1),
                              "planner": plan}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(int(sys.argv[2]), float(sys.argv[3]))
        raise SystemExit(0)
    Ss = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4,5,6,8,12,16").split(",")]
    min_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 6.0
    for S in Ss:
        env = dict(os.environ)
        if S > 0:
            env["KPGEMM_FORCE_SLICES"] = str(S)
        subprocess.run([sys.executable, __file__, "--child", str(S), str(min_ms)], env=env, check=False)
