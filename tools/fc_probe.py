"""HBM-bound rows probe: every config of a family on the VGG16 fc rows (and conv1_1),
sweep protocol (CudaEventTimer, L2 rotation), top configs with GB/s of algorithmic
bytes.  Usage: python tools/fc_probe.py [family] [batches] [min_ms]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_13145_b200 import gemm  # noqa: E402
from paper_2008_13145_b200.dataset import ProblemSize  # noqa: E402
from paper_2008_13145_b200.sweep import CudaEventTimer  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "simt"
batches = [int(b) for b in (sys.argv[2] if len(sys.argv) > 2 else "1,16,32,64").split(",")]
min_ms = float(sys.argv[3]) if len(sys.argv) > 3 else 6.0
probs = []
for b in batches:
    probs += [ProblemSize(b, 25088, 4096, 1), ProblemSize(b, 4096, 4096, 1), ProblemSize(b, 4096, 1000, 1)]
probs.append(ProblemSize(16 * 224 * 224, 27, 64, 1))
esz = gemm.input_dtype(fam).itemsize
timer = CudaEventTimer(fam, probs, min_ms=min_ms)
cfgs = gemm.family_configs(fam)
for p in probs:
    nbytes = esz * (p.m * p.k + p.k * p.n) + 4 * p.m * p.n
    rows = []
    for ci in range(len(cfgs)):
        g, ms, _ = timer(p, ci)
        rows.append((g, ms, ci))
    rows.sort(reverse=True)
    top = [{"config": list(cfgs[ci].as_tuple()), "gflops": round(g, 1), "gbs": round(nbytes / ms / 1e6, 1),
            "plan": gemm.k_slice_plan(cfgs[ci], p, fam)} for g, ms, ci in rows[:6]]
    print(json.dumps({"problem": [p.m, p.k, p.n], "bytes": nbytes, "top": top}), flush=True)
