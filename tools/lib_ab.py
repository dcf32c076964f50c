"""TF/s of selected SIMT configs on the bench's layer shapes with the library named by
KPGEMM_LIB (dev tool: compare builds, e.g. occupancy targets).  usage: lib_ab.py TAG"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig  # noqa: E402

CFGS = [(8, 1, 8, 8, 16), (8, 8, 8, 16, 8), (4, 2, 8, 16, 8), (8, 1, 8, 16, 16), (8, 8, 8, 16, 16),
        (8, 2, 4, 8, 16), (8, 4, 4, 8, 16), (2, 1, 8, 8, 8), (1, 8, 8, 8, 8), (8, 2, 8, 16, 8), (4, 4, 8, 8, 16),
        (8, 8, 8, 8, 8), (4, 8, 8, 16, 16)]
SHAPES = [(12544, 4608, 512), (3136, 4608, 512), (50176, 2304, 256), (200704, 1152, 128), (802816, 576, 64),
          (16, 25088, 4096), (8192, 8192, 8192)]
dev = torch.device("cuda")
res = {}
for (m, k, n) in SHAPES:
    A = torch.rand(m, k, device=dev)
    B = torch.rand(k, n, device=dev)
    ops = gemm.GemmOperands(A, B, None, torch.float32)
    for c in CFGS:
        vid = gemm.variant_id(KernelConfig(*c), "simt")
        best = 0.0
        for _ in range(2):
            ms, _ = gemm.bench(vid, ops, warmup=2, min_ms=25)
            best = max(best, 2.0 * m * k * n / (ms * 1e-3) / 1e12)
        res[f"{c}@{m}x{k}x{n}"] = best
    del A, B, ops
    torch.cuda.empty_cache()
print(json.dumps({"tag": sys.argv[1] if len(sys.argv) > 1 else "", "lib": os.environ.get("KPGEMM_LIB", "default"),
                  "tflops": res}))
