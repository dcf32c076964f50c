"""Diagnose the tcgen05 families on structured inputs (identity / one-hot)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2008_13145_b200 import gemm
from paper_2008_13145_b200.dataset import KernelConfig

dev = torch.device("cuda")
torch.set_printoptions(linewidth=200, precision=2)
for fam in ("tf32", "bf16"):
    cfg = gemm.family_configs(fam)[1 if fam == "tf32" else 0]
    dt = gemm.input_dtype(fam)
    for (m, k, n) in ((128, 32, 64), (128, 64, 64)):
        A = torch.randn(m, k, device=dev).to(dt)
        I = torch.zeros(k, n, device=dev)
        I[torch.arange(min(k, n)), torch.arange(min(k, n))] = 1
        C = gemm.matmul(A, I.to(dt), cfg, fam)
        ref = A.float() @ I
        print(fam, cfg.as_tuple(), (m, k, n), "max err vs A@I:", (C - ref).abs().max().item())
        # which column of ref does each output column match?
        match = []
        for j in range(min(n, 16)):
            d = (C[:, j:j + 1] - ref).abs().max(dim=0).values
            match.append(int(d.argmin()) if d.min() < 1e-2 else -1)
        print("   col j -> matches ref col:", match)
        # B = random, A = one-hot rows: C row i = B row (perm)
        Bm = torch.randn(k, n, device=dev).to(dt)
        E = torch.zeros(m, k, device=dev)
        E[torch.arange(m), torch.arange(m) % k] = 1
        C2 = gemm.matmul(E.to(dt), Bm, cfg, fam)
        ref2 = E @ Bm.float()
        print("   onehot-A max err:", (C2 - ref2).abs().max().item())
        rows = []
        for i in range(min(m, 12)):
            d = (C2[i:i + 1, :] - Bm.float()).abs().max(dim=1).values
            rows.append(int(d.argmin()) if d.min() < 1e-2 else -1)
        print("   row i -> matches B row:", rows)
