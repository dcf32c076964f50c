"""Planner-model data (dev tool): TFLOP/s of SIMT configs on every VGG16 / ResNet-50
GEMM shape whose grid is under 3 waves, for a forced slice count (KPGEMM_FORCE_SLICES;
0 = planner).  One JSON line per (shape, config)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm, shapes  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig  # noqa: E402

CFGS = [(8, 8, 8, 16, 8), (8, 1, 8, 8, 16), (8, 2, 4, 8, 16), (4, 2, 8, 16, 8), (8, 8, 8, 16, 16), (4, 8, 8, 8, 8)]
probs = shapes.network_problems("vgg16") + shapes.network_problems("resnet50")
dev = torch.device("cuda")
forced = int(os.environ.get("KPGEMM_FORCE_SLICES", 0))
seen = set()
for p in probs:
    if p.k < 512 or p.m * p.n < 20000:
        continue
    key = (p.m, p.k, p.n)
    if key in seen:
        continue
    seen.add(key)
    A = torch.rand(p.m, p.k, device=dev)
    B = torch.rand(p.k, p.n, device=dev)
    ops = gemm.GemmOperands(A, B, None, torch.float32)
    for c in CFGS:
        bm, bn = c[0] * c[3], c[2] * c[4]
        tiles = -(-p.m // bm) * -(-p.n // bn)
        occ = max(1, 512 // (c[3] * c[4]))
        if tiles >= 3 * 148 * occ:
            continue
        ms, _ = gemm.bench(gemm.variant_id(KernelConfig(*c), "simt"), ops, warmup=2, min_ms=8)
        print(json.dumps({"shape": list(key), "config": c, "tiles": tiles, "occ": occ, "forced": forced,
                          "plan": gemm.k_slice_plan(KernelConfig(*c), p),
                          "tflops": round(2.0 * p.m * p.k * p.n / (ms * 1e-3) / 1e12, 2)}), flush=True)
