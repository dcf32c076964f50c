"""A/B of two SIMT library builds (KPGEMM_LIB) on the configs a build change touches:
sweep-protocol GFLOP/s (CudaEventTimer) per (config, shape).
usage: KPGEMM_LIB=... python tools/occ_ab.py TAG [wg filter, e.g. 64 for 64-thread work groups]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_13145_b200.dataset import ProblemSize  # noqa: E402
from paper_2008_13145_b200.sweep import CudaEventTimer  # noqa: E402

tag = sys.argv[1]
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 64
SHAPES = [(16, 25088, 4096), (16, 4096, 4096), (32, 25088, 4096), (64, 4096, 4096), (3136, 4608, 512),
          (12544, 4608, 512), (802816, 576, 64), (802816, 27, 64), (50176, 1152, 256), (784, 4608, 512),
          (4096, 4096, 4096)]
probs = [ProblemSize(m, k, n, 1) for m, k, n in SHAPES]
timer = CudaEventTimer("simt", probs, min_ms=4.0)
for p in probs:
    for ci, c in enumerate(timer.configs):
        if c.wg_rows * c.wg_cols != nt:
            continue
        g, ms, _ = timer(p, ci)
        print(json.dumps({"tag": tag, "problem": [p.m, p.k, p.n], "config": c.as_tuple(), "gflops": round(g, 1)}),
              flush=True)
