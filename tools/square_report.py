"""BASELINE configs[5] report: per square/skinny shape, the best config of each family
(from the measured sweep tables) against the cuBLAS comparison lines."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_13145_b200 import dataset  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
fams = {}
for fam, name in (("paper", "square_paper"), ("simt", "square_simt"), ("tf32", "square16k_tf32"),
                  ("bf16", "square16k_bf16")):
    pm = dataset.parse_benchmark_csv((ROOT / "data" / "sweeps" / f"{name}.csv").read_text())
    fams[fam] = {(p.m, p.k, p.n): (float(pm.values[i].max()), pm.configs[int(pm.values[i].argmax())].as_tuple())
                 for i, p in enumerate(pm.problems)}
cub_path = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "raw" / "r1_square_cublas.json"
cub = json.loads(cub_path.read_text())
print("| m,k,n | paper F0 best | simt F1 best | tf32 best | bf16 best | cuBLAS fp32 | cuBLAS tf32 | cuBLAS bf16 |")
print("|---|---|---|---|---|---|---|---|")
for key, row in cub.items():
    m, k, n, _ = (int(x) for x in key.split(","))
    cells = []
    for fam in ("paper", "simt", "tf32", "bf16"):
        v = fams[fam].get((m, k, n))
        cells.append(f"{v[0] / 1e3:.1f} `{v[1]}`" if v else "-")
    print(f"| {m},{k},{n} | " + " | ".join(cells) + " | " +
          " | ".join(f"{row[c] / 1e3:.1f}" for c in ("cublas_fp32", "cublas_tf32", "cublas_bf16")) + " |")
print("\nTFLOP/s; best config per family from data/sweeps (sweep protocol: median of 3 CUDA-event loops of "
      ">= 20 ms, operands rotated over 2 x L2 for small problems); cuBLAS via torch.matmul, one >= 20 ms loop "
      "after 2 warm-ups (comparison only; shorter sustained load, so less power-capping on the largest GEMMs).")
