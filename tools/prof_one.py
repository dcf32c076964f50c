"""Launch one kernel variant a few times (for ncu captures).
usage: prof_one.py FAMILY R A C WGR WGC M K N [BATCH] [REPS]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm
from paper_2008_13145_b200.dataset import KernelConfig

fam = sys.argv[1]
cfg = KernelConfig(*map(int, sys.argv[2:7]))
m, k, n = map(int, sys.argv[7:10])
batch = int(sys.argv[10]) if len(sys.argv) > 10 else 1
reps = int(sys.argv[11]) if len(sys.argv) > 11 else 3
dt = gemm.input_dtype(fam)
A = torch.rand(batch, m, k, device="cuda").to(dt)
B = torch.rand(batch, k, n, device="cuda").to(dt)
for _ in range(reps):
    gemm.matmul(A, B, cfg, fam)
torch.cuda.synchronize()
print("ok")
