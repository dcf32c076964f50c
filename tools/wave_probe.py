"""Planner experiment (dev tool): GFLOP/s of a config on a shape for forced slice counts
S = 1..8 (KPGEMM_FORCE_SLICES, one process per S).  Prints one JSON line per run."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig  # noqa: E402

fam = sys.argv[1]
CASES = {
    "simt": [((12544, 4608, 512), (8, 8, 8, 16, 8)), ((12544, 4608, 512), (8, 8, 8, 16, 16)),
             ((25088, 1152, 256), (8, 8, 8, 16, 8)), ((50176, 576, 64), (4, 2, 8, 16, 8)),
             ((6272, 4608, 512), (4, 2, 8, 16, 8)), ((12544, 2304, 256), (8, 8, 4, 8, 16)),
             ((100352, 576, 64), (8, 8, 8, 16, 8)), ((3136, 4608, 512), (8, 8, 8, 16, 16)),
             ((25088, 2304, 512), (8, 8, 8, 16, 16))],
    "simt_many": [((802816, 576, 64), (8, 8, 8, 16, 8)), ((200704, 1152, 128), (8, 8, 8, 16, 8)),
                  ((50176, 4608, 512), (8, 8, 8, 16, 8)), ((100352, 2304, 256), (8, 8, 8, 16, 16)),
                  ((8192, 8192, 8192), (8, 8, 8, 16, 16)), ((4096, 4096, 4096), (8, 8, 8, 16, 16)),
                  ((401408, 576, 128), (4, 2, 8, 16, 8)), ((50176, 2304, 512), (8, 8, 4, 8, 16)),
                  ((2048, 2048, 2048), (4, 2, 8, 16, 8)), ((25088, 4608, 512), (8, 8, 8, 16, 8))],
    "bf16": [((12544, 4608, 512), (128, 64, 256, 4, 192)), ((6272, 2304, 512), (128, 64, 128, 4, 192)),
             ((3136, 4608, 512), (128, 64, 256, 4, 192)), ((25088, 2304, 256), (128, 64, 128, 6, 192)),
             ((12544, 2304, 512), (128, 64, 192, 4, 192))],
}
dev = torch.device("cuda")
dt = torch.bfloat16 if fam == "bf16" else torch.float32
fam_lib = "simt" if fam.startswith("simt") else fam
for (m, k, n), c in CASES[fam]:
    A = (torch.rand(m, k, device=dev) * 2 - 1).to(dt)
    B = (torch.rand(k, n, device=dev) * 2 - 1).to(dt)
    ops = gemm.GemmOperands(A, B, None, dt)
    ms, _ = gemm.bench(gemm.variant_id(KernelConfig(*c), fam_lib), ops, warmup=3, min_ms=20)
    print(json.dumps({"fam": fam, "shape": [m, k, n], "config": c, "forced": int(os.environ.get("KPGEMM_FORCE_SLICES", 0)),
                      "tflops": round(2.0 * m * k * n / (ms * 1e-3) / 1e12, 2)}), flush=True)
