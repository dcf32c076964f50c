"""Tail-tile probe (dev tool): GFLOP/s of large-tile configs on shapes whose m or n is far
below the CTA tile (fc layers at small batch, n = 64 conv layers)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig  # noqa: E402

SHAPES = [(32, 25088, 4096), (32, 4096, 4096), (16, 25088, 4096), (64, 4096, 4096), (802816, 576, 64),
          (200704, 576, 64), (1568, 4608, 512)]
CFGS = [(8, 8, 8, 16, 8), (8, 8, 8, 16, 16), (4, 2, 8, 16, 8), (8, 8, 4, 8, 16), (4, 8, 8, 8, 8), (8, 1, 8, 16, 16)]
dev = torch.device("cuda")
for (m, k, n) in SHAPES:
    A = torch.rand(m, k, device=dev)
    B = torch.rand(k, n, device=dev)
    ops = gemm.GemmOperands(A, B, None, torch.float32)
    row = {}
    for c in CFGS:
        ms, _ = gemm.bench(gemm.variant_id(KernelConfig(*c), "simt"), ops, warmup=2, min_ms=10)
        row[str(c)] = round(2.0 * m * k * n / (ms * 1e-3) / 1e12, 2)
    print(json.dumps({"shape": [m, k, n], "tflops": row}), flush=True)
