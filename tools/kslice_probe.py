"""SIMT family A/B probe: GFLOP/s per (problem, config) with k-slicing off (cap 1) and
at the default cap (8), for mid-size VGG16 rows, fc rows and a large square.
Usage: python tools/kslice_probe.py [caps, e.g. 1,8]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig, ProblemSize  # noqa: E402

CAPS = tuple(int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "1,8").split(","))
PROBS = [(196, 4608, 512), (392, 4608, 512), (32, 25088, 4096), (32, 4096, 4096), (8, 25088, 4096),
         (3136, 2304, 256), (1568, 4608, 512), (1, 25088, 4096), (1, 4096, 1000), (12544, 4608, 512),
         (100352, 576, 64), (8192, 8192, 8192)]
CFGS = [(8, 8, 8, 16, 8), (1, 4, 4, 8, 8), (4, 1, 8, 16, 8), (4, 8, 8, 16, 8), (8, 8, 4, 8, 16), (4, 2, 8, 16, 8),
        (4, 8, 8, 8, 8), (8, 8, 8, 16, 16), (1, 8, 1, 1, 64)]
dev = torch.device("cuda", 0)
for m, k, n in PROBS:
    A = torch.rand(m, k, device=dev) * 2 - 1
    B = torch.rand(k, n, device=dev) * 2 - 1
    for c in CFGS:
        cfg = KernelConfig(*c)
        p = ProblemSize(m, k, n, 1)
        row = {"problem": [m, k, n], "config": c}
        for cap in CAPS:
            gemm.set_max_k_slices(cap)
            ops = gemm.GemmOperands(A, B, None, torch.float32)
            ms, it = gemm.bench(gemm.variant_id(cfg, "simt"), ops, warmup=2, min_ms=5.0)
            row[f"gflops_cap{cap}"] = round(2.0 * m * k * n / (ms * 1e6), 1)
            row[f"plan_cap{cap}"] = gemm.k_slice_plan(cfg, p)
        print(json.dumps(row), flush=True)
