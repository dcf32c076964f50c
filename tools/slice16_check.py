"""16-CTA k-slice clusters: triage and stress.
usage: python tools/slice16_check.py {sync_cpasync16, sync_tma12, sync_tma9, stress}"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import gemm_oracle as go  # noqa: E402
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig, ProblemSize  # noqa: E402

dev = torch.device("cuda")
what = sys.argv[1]
cfg = KernelConfig(8, 4, 2, 1, 64)
if what == "sync_cpasync16":
    gemm.set_simt_staging("cp.async")
    C = gemm.matmul(torch.rand(8, 4096, device=dev), torch.rand(4096, 1000, device=dev), cfg)
    torch.cuda.synchronize()
    print(what, "ok")
elif what.startswith("sync_tma"):
    # forced slice count through the dev override (read once per process)
    C = gemm.matmul(torch.rand(8, 4096, device=dev), torch.rand(4096, 1000, device=dev), cfg)
    torch.cuda.synchronize()
    print(what, os.environ.get("KPGEMM_FORCE_SLICES"), "ok")
elif what == "stress":
    rng = np.random.default_rng(7)
    bad = 0
    for (m, k, n, c) in ((8, 4096, 1000, cfg), (4, 4096, 1000, KernelConfig(4, 4, 2, 1, 64)),
                         (16, 4096, 1000, KernelConfig(8, 8, 8, 16, 8)), (2, 25088, 4096, KernelConfig(8, 4, 2, 1, 64)),
                         (32, 4096, 1000, KernelConfig(4, 2, 8, 16, 8))):
        p = ProblemSize(m, k, n, 1)
        plan = gemm.k_slice_plan(c, p)
        A = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        B = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        want = go.gemm_sliced(A, B, plan[1])[0].view(np.uint32)
        dA, dB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
        out = torch.empty(m, n, device=dev)
        for it in range(300):
            gemm.matmul(dA, dB, c, "simt", out=out)
            if it % 30 == 0 or it == 299:
                got = out.cpu().numpy().view(np.uint32)
                if not np.array_equal(got, want):
                    bad += 1
        print(p, c.as_tuple(), "plan", plan, "bad checks", bad, flush=True)
    print("stress", "FAIL" if bad else "ok")
