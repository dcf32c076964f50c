"""TC-family A/B probe (dev tool): TFLOP/s of every tf32/bf16 config on a few shapes with
the library named by KPGEMM_LIB; k-slicing cap from argv[1] (ignored by libraries
without kp_set_max_k_slices)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import _lib, gemm  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 8
lib = _lib.load()
if hasattr(lib, "kp_set_max_k_slices"):
    lib.kp_set_max_k_slices(cap)
SHAPES = [(3211264, 27, 64), (100352, 147, 64), (12544, 4608, 512), (6272, 1152, 256), (784, 512, 256),
          (3136, 576, 64), (1568, 4608, 512), (8192, 8192, 8192), (16384, 64, 16384), (16384, 16384, 64), (4096, 4096, 4096),
          (2560, 4096, 4096), (12544, 2304, 512)]
dev = torch.device("cuda")
res = {}
for fam in ("bf16", "tf32"):
    dt = torch.bfloat16 if fam == "bf16" else torch.float32
    for (m, k, n) in SHAPES:
        A = torch.rand(m, k, device=dev).to(dt)
        B = torch.rand(k, n, device=dev).to(dt)
        ops = gemm.GemmOperands(A, B, None, dt)
        for i, cfg in enumerate(gemm.family_configs(fam)):
            ms, _ = gemm.bench(gemm.variant_id(cfg, fam), ops, warmup=3, min_ms=10)
            res[f"{fam}{i}@{m}x{k}x{n}"] = round(2.0 * m * k * n / (ms * 1e-3) / 1e12, 1)
print(json.dumps({"lib": os.environ.get("KPGEMM_LIB", "default"), "cap": cap, "tflops": res}))
