"""One code path per process for compute-sanitizer triage.
usage: python tools/sanitize_focus.py {pair_bf16,pair_tf32,simt_tma,simt_tma_slice8,simt_tma_slice16,tc_bf16}"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import KernelConfig, ProblemSize  # noqa: E402

dev = torch.device("cuda")
what = sys.argv[1]
if what.startswith("pair_"):
    fam = what[5:]
    pair = next(c for c in gemm.family_configs(fam) if c.tile_rows == 256)
    dt = gemm.input_dtype(fam)
    C = gemm.matmul(torch.rand(600, 256, device=dev).to(dt), torch.rand(256, 520, device=dev).to(dt), pair, fam)
elif what == "tc_bf16":
    cfg = gemm.family_configs("bf16")[1]
    C = gemm.matmul(torch.rand(600, 256, device=dev).to(torch.bfloat16),
                    torch.rand(256, 520, device=dev).to(torch.bfloat16), cfg, "bf16")
elif what == "simt_tma":
    C = gemm.matmul(torch.rand(1000, 512, device=dev), torch.rand(512, 512, device=dev), KernelConfig(8, 4, 4, 8, 8))
elif what == "simt_tma_slice8":
    cfg, p = KernelConfig(8, 4, 2, 1, 64), ProblemSize(16, 4096, 4096, 1)
    print("plan", gemm.k_slice_plan(cfg, p))
    C = gemm.matmul(torch.rand(16, 4096, device=dev), torch.rand(4096, 4096, device=dev), cfg)
elif what == "simt_tma_slice16":
    cfg, p = KernelConfig(8, 4, 2, 1, 64), ProblemSize(8, 4096, 1000, 1)
    print("plan", gemm.k_slice_plan(cfg, p))
    C = gemm.matmul(torch.rand(8, 4096, device=dev), torch.rand(4096, 1000, device=dev), cfg)
torch.cuda.synchronize()
print(what, "ok", float(C.sum()))
