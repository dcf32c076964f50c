"""Run-to-run spread of two sweeps of the same table (same library, same protocol):
per-cell relative difference, per-row best changes, and the north-star metric (k-means-4
+ treeA held-out, and the rest of the paper's grid) on each.  Markdown to stdout.
usage: python tools/sweep_spread.py A.csv B.csv"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2008_13145_b200 import dataset  # noqa: E402

a_path, b_path = sys.argv[1:3]
A = dataset.parse_benchmark_csv(Path(a_path).read_text())
B = dataset.parse_benchmark_csv(Path(b_path).read_text())
assert A.problems == B.problems and A.configs == B.configs, "tables differ in rows/columns"
rel = np.abs(B.values - A.values) / A.values
print(f"### sweep spread: `{a_path}` vs `{b_path}` ({A.n_problems} x {A.n_configs} cells)\n")
print("| per-cell abs(B - A) / A | median | p90 | p99 | max |")
print("|---|---|---|---|---|")
q = np.quantile(rel, [0.5, 0.9, 0.99, 1.0])
print("| all cells | " + " | ".join(f"{x * 100:.2f} %" for x in q) + " |")
big = np.array([p.flops >= 10e9 for p in A.problems])
q = np.quantile(rel[big], [0.5, 0.9, 0.99, 1.0])
print("| rows >= 10 GFLOP | " + " | ".join(f"{x * 100:.2f} %" for x in q) + " |")
best_a, best_b = A.values.max(1), B.values.max(1)
same = int((A.values.argmax(1) == B.values.argmax(1)).sum())
print(f"\nper-row best: same winning config in {same} / {A.n_problems} rows; "
      f"row-best value abs diff median {np.median(np.abs(best_b - best_a) / best_a) * 100:.2f} %, "
      f"max {np.max(np.abs(best_b - best_a) / best_a) * 100:.2f} %\n")
print("| table | kmeans4 subset | k_actual | treeA held-out | ceiling | kmeans8 | spectral8 | pca_kmeans8 | tree8 |")
print("|---|---|---|---|---|---|---|---|---|")
for name, path in (("A", a_path), ("B", b_path)):
    pm, subset, tree, rt, ra, _ = bench.train_selector(path, 4, "kmeans", "treeA")
    grid = bench.selection_grid(pm)
    cells = " | ".join(f"{grid[k]['achieved_test']:.3f} ({grid[k]['k_actual']})"
                       for k in ("kmeans8", "spectral8", "pca_kmeans8", "tree8"))
    print(f"| {name} | {[pm.configs[i].as_tuple() for i in subset.config_indices]} | {subset.k_actual} | "
          f"{rt.achieved:.4f} | {rt.ceiling:.4f} | {cells} |")
