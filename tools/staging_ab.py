"""A/B of the SIMT family's operand staging (TMA + mbarrier vs per-thread cp.async) on
the bench's layer shapes and large squares: TFLOP/s per (config, shape), interleaved
A/B/A/B so clock drift hits both arms (dev tool; results -> profiles/)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig  # noqa: E402

CFGS = [(8, 1, 8, 8, 16), (8, 8, 8, 16, 8), (4, 2, 8, 16, 8), (8, 1, 8, 16, 16), (8, 8, 8, 16, 16),
        (8, 2, 4, 8, 16), (4, 4, 8, 16, 8), (2, 1, 8, 8, 8), (1, 8, 8, 8, 8), (8, 4, 4, 8, 16), (8, 2, 8, 16, 8)]
SHAPES = [(12544, 4608, 512), (3136, 4608, 512), (50176, 2304, 256), (200704, 1152, 128), (802816, 576, 64),
          (16, 25088, 4096), (16, 4096, 4096), (8192, 8192, 8192), (4096, 4096, 4096)]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    CFGS, SHAPES = CFGS[:3], SHAPES[:2]
dev = torch.device("cuda")
res = {}
for (m, k, n) in SHAPES:
    A = torch.rand(m, k, device=dev)
    B = torch.rand(k, n, device=dev)
    ops = gemm.GemmOperands(A, B, None, torch.float32)
    for c in CFGS:
        vid = gemm.variant_id(KernelConfig(*c), "simt")
        t = {"tma": [], "cp.async": []}
        for rep in range(2):
            for mode in ("cp.async", "tma"):
                gemm.set_simt_staging(mode)
                ms, _ = gemm.bench(vid, ops, warmup=2, min_ms=25)
                t[mode].append(2.0 * m * k * n / (ms * 1e-3) / 1e12)
        gemm.set_simt_staging("tma")
        row = {mode: max(v) for mode, v in t.items()}
        res[f"{c}@{m}x{k}x{n}"] = row
        print(f"{c} {m}x{k}x{n}: cp.async {row['cp.async']:.2f}  tma {row['tma']:.2f}  "
              f"x{row['tma'] / row['cp.async']:.3f}", flush=True)
    del A, B, ops
    torch.cuda.empty_cache()
print(json.dumps({"tflops": res}))
