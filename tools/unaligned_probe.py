"""Unaligned operand rows (raw k = 27 / 147, n = 27): GFLOP/s and GB/s of algorithmic
bytes per family's best config, unpitched (lda = k) vs pitched to 16 bytes, with the
library named by KPGEMM_LIB.  usage: python tools/unaligned_probe.py TAG"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig  # noqa: E402

CFG = {"bf16": (128, 64, 64, 4, 192), "tf32": (128, 32, 64, 4, 192), "simt": (8, 8, 4, 8, 16)}
SHAPES = [(802816, 27, 64), (200704, 147, 64), (32, 12321, 27), (12544, 27, 64)]
dev = torch.device("cuda")
for fam, c in CFG.items():
    dt = gemm.input_dtype(fam)
    es = dt.itemsize
    vid = gemm.variant_id(KernelConfig(*c), fam)
    for m, k, n in SHAPES:
        for pitched in (False, True):
            al = 16 // es
            lda = -(-k // al) * al if pitched else k
            ldb = -(-n // al) * al if pitched else n
            A = (torch.rand(m, lda, device=dev) * 2 - 1).to(dt)[:, :k]
            B = (torch.rand(k, ldb, device=dev) * 2 - 1).to(dt)[:, :n]
            ops = gemm.GemmOperands(A, B, None, dt)
            ms, _ = gemm.bench(vid, ops, warmup=3, min_ms=20)
            nbytes = es * (m * k + k * n) + 4 * m * n
            print(json.dumps({"tag": sys.argv[1], "lib": os.environ.get("KPGEMM_LIB", "in-tree"), "family": fam,
                              "config": c, "problem": [m, k, n], "pitched": pitched, "ms": round(ms, 5),
                              "gflops": round(2 * m * k * n / ms / 1e6, 1), "gbs": round(nbytes / ms / 1e6, 1)}),
                  flush=True)
            del A, B, ops
