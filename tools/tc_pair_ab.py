"""Tensor-core families on large squares / conv shapes: every config (1-CTA and CTA-pair)
vs cuBLAS (torch.matmul) in the same process, CUDA-event loops >= 25 ms (dev tool)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm  # noqa: E402

SHAPES = [(8192, 8192, 8192), (4096, 4096, 4096), (2048, 2048, 2048), (12544, 4608, 512), (50176, 2304, 256),
          (16384, 16384, 16384)]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    SHAPES = SHAPES[:3]
dev = torch.device("cuda")
res = {}


def cublas(a, b):
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 1
    while True:
        e0.record()
        for _ in range(reps):
            torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if ms > 25 or reps >= 4096:
            return ms / reps
        reps *= 2


for (m, k, n) in SHAPES:
    for fam in ("bf16", "tf32"):
        dt = gemm.input_dtype(fam)
        A = (torch.rand(m, k, device=dev) - 0.5).to(dt)
        B = (torch.rand(k, n, device=dev) - 0.5).to(dt)
        ops = gemm.GemmOperands(A, B, None, dt)
        row = {}
        for cfg in gemm.family_configs(fam):
            ms, _ = gemm.bench(gemm.variant_id(cfg, fam), ops, warmup=2, min_ms=25)
            row[str(cfg.as_tuple())] = 2.0 * m * k * n / (ms * 1e-3) / 1e12
        torch.backends.cuda.matmul.allow_tf32 = fam == "tf32"
        row["cublas"] = 2.0 * m * k * n / (cublas(A, B) * 1e-3) / 1e12
        res[f"{fam}@{m}x{k}x{n}"] = row
        best = max((v, c) for c, v in row.items() if c != "cublas")
        print(f"{fam} {m}x{k}x{n}: best {best[1]} {best[0]:.0f}  cuBLAS {row['cublas']:.0f}  "
              + " ".join(f"{c}:{v:.0f}" for c, v in row.items() if c != "cublas"), flush=True)
        del A, B, ops
        torch.cuda.empty_cache()
print(json.dumps(res))
