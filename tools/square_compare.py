"""cuBLAS comparison lines (torch.matmul fp32 / tf32 / bf16) for the square/skinny set
(BASELINE configs[5]); GFLOP/s per shape as JSON.  Comparison only -- never on the
product path."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import shapes  # noqa: E402

dev = torch.device("cuda")
out = {}
for p in shapes.square_skinny_problems():
    row = {}
    for name, dt, tf32 in (("cublas_fp32", torch.float32, False), ("cublas_tf32", torch.float32, True),
                           ("cublas_bf16", torch.bfloat16, False)):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        a = torch.rand(p.m, p.k, device=dev).to(dt)
        b = torch.rand(p.k, p.n, device=dev).to(dt)
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
            if ms > 20 or reps >= 4096:
                break
            reps *= 4
        row[name] = p.flops / (ms / reps * 1e-3) / 1e9
    out[f"{p.m},{p.k},{p.n},{p.batch}"] = row
    print(p, {k: round(v) for k, v in row.items()}, file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
