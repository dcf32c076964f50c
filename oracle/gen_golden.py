"""Generate tests/golden/*.json by running the REFERENCE package (kernelprune).

TEST INFRASTRUCTURE ONLY.  This script imports the read-only reference from
/root/reference/pkg/src (present only in the build container) and records its
outputs on seeded inputs, so the parity tests can pin the host-side restatement
(selection / classification / scoring / kptree) bit-exactly on machines where the
reference is absent (the GPU box).  Nothing in the product imports this.

    python oracle/gen_golden.py            # rewrites tests/golden/host_parity.json
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF))
    import numpy as np
    import importlib

    classify, codegen, dataset, evaluate, normalize, selection = (
        importlib.import_module(f"kernelprune.{m}")
        for m in ("classify", "codegen", "dataset", "evaluate", "normalize", "selection"))

    gold: dict = {"generator": "oracle/gen_golden.py", "reference": str(REF),
                  "numpy": np.__version__, "cases": {}}

    # --- Appendix A table: synth 40 x 640, noise 0.05, seed 0 (pipeline.py:149-155)
    probs = dataset.synth_problems(40, seed=0)
    pm = dataset.synth_generate(dataset.SynthModel(noise_sigma=0.05, seed=0), probs, dataset.enumerate_configs())
    text = dataset.serialize_benchmark_csv(pm)
    train, test = dataset.split(pm, dataset.SplitSpec(0.2, 0))
    gold["synth40"] = {
        "csv_sha256": hashlib.sha256(text.encode()).hexdigest(),
        "csv_lines": text.count("\n"),
        "problems": [[p.m, p.k, p.n, p.batch] for p in probs],
        "train_problems": [[p.m, p.k, p.n, p.batch] for p in train.problems],
        "test_problems": [[p.m, p.k, p.n, p.batch] for p in test.problems],
        "values_sha256": hashlib.sha256(pm.values.tobytes()).hexdigest(),
    }
    feats = classify.problem_features(train.problems)
    cases = {}
    for scheme in normalize.SCHEME_KINDS:
        nm = normalize.normalize(train, normalize.NormScheme(scheme))
        for method, k in [("kmeans", 4), ("kmeans", 8), ("spectral", 8), ("pca_kmeans", 8),
                          ("tree", 4), ("topn", 4), ("hdbscan", 4), ("spectral", 4), ("kmeans", 12)]:
            try:
                sub = selection.select_subset(method, nm, k, 0, problems=train.problems)
            except Exception as exc:  # record reference errors too
                cases[f"{scheme}/{method}/{k}"] = {"error": type(exc).__name__}
                continue
            labels = classify.label_best_in_subset(nm, sub)
            rec = {"config_indices": list(sub.config_indices), "k_actual": sub.k_actual,
                   "labels": labels.tolist(),
                   "ceiling": repr(evaluate.subset_ceiling(test, sub))}
            for preset in ("A", "B", "C"):
                tree = classify.train_tree(feats, labels, classify.TREE_PRESETS[preset], n_classes=sub.k_actual)
                rep = evaluate.classifier_score(test, sub, lambda x, t=tree: classify.predict_tree(t, x))
                rec[f"tree{preset}"] = {"achieved": repr(rep.achieved),
                                        "kptree": codegen.export_model(tree, sub, pm.configs)}
            cases[f"{scheme}/{method}/{k}"] = rec
    gold["cases"] = cases

    sub = selection.select_subset("kmeans", normalize.normalize(train, normalize.NormScheme()), 4, 0)
    labels = classify.label_best_in_subset(normalize.normalize(train, normalize.NormScheme()), sub)
    tree = classify.train_tree(feats, labels, classify.TREE_PRESETS["A"], n_classes=sub.k_actual)
    gold["kmeans4_treeA_emit"] = codegen.emit_nested_if(tree, sub, pm.configs)

    # --- reduced grid through grid_report (all classifiers incl. knn/forest/oracle)
    reports = evaluate.grid_report(train, test, ("kmeans", "spectral", "topn", "tree"), (4, 6),
                                   normalize.NormScheme("scaled"),
                                   classify.CLASSIFIER_SPECS + (evaluate.ORACLE_SPEC,), seed=0)
    gold["grid_eval_csv"] = evaluate.eval_report_csv(reports)
    gold["grid_per_row_csv_sha256"] = hashlib.sha256(evaluate.per_row_csv(reports).encode()).hexdigest()

    # --- random tables: kmeans/spectral/hdbscan/tree on 3 seeds
    rand = {}
    for seed in (1, 2, 3):
        rng = np.random.default_rng(seed)
        rows = rng.uniform(1.0, 900.0, size=(60, 48))
        rprobs = [dataset.ProblemSize(int(2 ** rng.integers(4, 12)), int(2 ** rng.integers(4, 12)),
                                      int(rng.integers(16, 5000)), int(rng.choice([1, 4, 16]))) for _ in range(60)]
        seen, uniq = set(), []
        for i, p in enumerate(rprobs):
            if p not in seen:
                seen.add(p)
                uniq.append(i)
        cfgs = dataset.enumerate_configs()[:48]
        rpm = dataset.PerfMatrix(tuple(rprobs[i] for i in uniq), tuple(cfgs), rows[uniq])
        nm = normalize.normalize(rpm, normalize.NormScheme("sigmoid"))
        ent = {"problems": [[p.m, p.k, p.n, p.batch] for p in rpm.problems], "values": rpm.values.tolist()}
        for method, k in [("kmeans", 5), ("spectral", 6), ("hdbscan", 5), ("tree", 5), ("pca_kmeans", 5)]:
            sub = selection.select_subset(method, nm, k, seed, problems=rpm.problems)
            ent[f"{method}/{k}"] = list(sub.config_indices)
        rand[str(seed)] = ent
    gold["random_tables"] = rand

    OUT.mkdir(parents=True, exist_ok=True)
    path = OUT / "host_parity.json"
    path.write_text(json.dumps(gold, indent=1, sort_keys=True) + "\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
