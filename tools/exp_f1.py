"""F1 variant experiment: TF/s of selected configs on selected shapes with the library
named by KPGEMM_LIB (dev tool)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig  # noqa: E402

CFGS = [(8, 1, 8, 16, 16), (8, 2, 8, 16, 16), (8, 4, 8, 16, 16), (8, 8, 8, 16, 16), (8, 4, 8, 8, 16),
        (8, 2, 8, 8, 16), (4, 8, 8, 16, 8), (8, 8, 4, 8, 16), (4, 2, 8, 16, 8), (4, 1, 2, 8, 8), (1, 1, 1, 8, 8),
        (8, 4, 8, 16, 8), (8, 8, 4, 16, 16), (8, 8, 8, 16, 8)]
SHAPES = [(8192, 8192, 8192), (4096, 4096, 4096), (12544, 4608, 512), (802816, 576, 64), (196, 4608, 512),
          (50176, 1152, 256)]
dev = torch.device("cuda")
res = {}
for (m, k, n) in SHAPES:
    A = torch.rand(m, k, device=dev)
    B = torch.rand(k, n, device=dev)
    ops = gemm.GemmOperands(A, B, None, torch.float32)
    for c in CFGS:
        vid = gemm.variant_id(KernelConfig(*c), "simt")
        ms, _ = gemm.bench(vid, ops, warmup=2, min_ms=30)
        res[f"{c}@{m}x{k}x{n}"] = 2.0 * m * k * n / (ms * 1e-3) / 1e12
lib = os.environ.get("KPGEMM_LIB", "default")
print(json.dumps({"lib": lib, "tflops": res}))
