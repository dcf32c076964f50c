"""Selection-quality report for a measured benchmark table (the paper's grid,
evaluate.grid_report): methods x k x tree presets on the seeded 80/20 split, plus the
all-rows (deployment) score.  Markdown to stdout.

usage: python tools/selection_report.py data/sweeps/vgg16_simt.csv [--k 4,5,6,7,8]
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_2008_13145_b200 import classify, dataset, evaluate, selection  # noqa: E402
from paper_2008_13145_b200.normalize import NormScheme, normalize  # noqa: E402


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("table")
    ap.add_argument("--k", default="4,8")
    ap.add_argument("--methods", default="kmeans,spectral,pca_kmeans,tree,topn")
    ap.add_argument("--scheme", default="scaled")
    args = ap.parse_args(argv)
    pm = dataset.parse_benchmark_csv(Path(args.table).read_text())
    train, test = dataset.split(pm, dataset.SplitSpec(0.2, 0))
    nm = normalize(train, NormScheme(args.scheme))
    feats = classify.problem_features(train.problems)
    v = pm.values
    print(f"### {args.table}: {pm.n_problems} problems x {pm.n_configs} configs, scheme {args.scheme}\n")
    print(f"max {v.max():.0f} GFLOP/s; per-row best median {np.median(v.max(axis=1)):.0f}; "
          f"{int((np.bincount(v.argmax(axis=1), minlength=pm.n_configs) > 0).sum())} distinct per-row winners\n")
    print("| method | k | k_actual | ceiling (test) | treeA | treeB | treeC | treeA all rows | ceiling all rows |")
    print("|---|---|---|---|---|---|---|---|---|")
    for method in args.methods.split(","):
        for k in (int(x) for x in args.k.split(",")):
            try:
                sub = selection.select_subset(method, nm, k, 0, problems=train.problems)
            except Exception as exc:  # degenerate input for this method
                print(f"| {method} | {k} | - | {type(exc).__name__} | | | | | |")
                continue
            labels = classify.label_best_in_subset(nm, sub)
            ach = []
            for preset in "ABC":
                tree = classify.train_tree(feats, labels, classify.TREE_PRESETS[preset], n_classes=sub.k_actual)
                ach.append(evaluate.classifier_score(test, sub, lambda x, t=tree: classify.predict_tree(t, x)))
                if preset == "A":
                    allrows = evaluate.classifier_score(pm, sub, lambda x, t=tree: classify.predict_tree(t, x))
            print(f"| {method} | {k} | {sub.k_actual} | {ach[0].ceiling:.4f} | {ach[0].achieved:.4f} | "
                  f"{ach[1].achieved:.4f} | {ach[2].achieved:.4f} | {allrows.achieved:.4f} | {allrows.ceiling:.4f} |")


if __name__ == "__main__":
    main()
