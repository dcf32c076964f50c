"""Generate tests/golden/measured_tables.json: the REFERENCE package's selection and
scoring results on every measured B200 table under data/sweeps/.

TEST INFRASTRUCTURE ONLY.  Imports the read-only reference (kernelprune) from
/root/reference/pkg/src (build container only) and records, per table, the
split -> normalize -> select_subset -> label -> train_tree(A/B/C) -> classifier_score
chain that the north-star metric is (evaluate.py:71-101, selection.py:491-521), with
float results as ``repr`` so tests/test_measured_tables.py can require bit-identity on
machines without the reference.  Each table is keyed by the sha256 of its bytes; a
re-swept table needs this script re-run (the test fails on a stale hash).

    python oracle/gen_golden_tables.py
"""

from __future__ import annotations

import hashlib
import importlib
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "measured_tables.json"

# (method, k) cells of the paper's grid recorded per table; scheme "scaled" is the
# pipeline default (cli.py:242), "sigmoid" exercises the other float path.
CELLS = (("kmeans", 4), ("kmeans", 8), ("spectral", 4), ("spectral", 8), ("pca_kmeans", 8), ("tree", 4))
SCHEMES = ("scaled", "sigmoid")


def run_chain(mods, text: str) -> dict:
    """The selection chain on one CSV table with module set ``mods`` (reference or
    this package): every float as repr, every index list as ints."""
    classify, dataset, evaluate, normalize, selection = (mods[m] for m in
                                                          ("classify", "dataset", "evaluate", "normalize", "selection"))
    pm = dataset.parse_benchmark_csv(text)
    train, test = dataset.split(pm, dataset.SplitSpec(0.2, 0))
    feats = classify.problem_features(train.problems)
    out = {"shape": [len(pm.problems), len(pm.configs)],
           "test_rows": [[p.m, p.k, p.n, p.batch] for p in test.problems]}
    for scheme in SCHEMES:
        nm = normalize.normalize(train, normalize.NormScheme(scheme))
        for method, k in CELLS:
            key = f"{scheme}/{method}{k}"
            try:
                sub = selection.select_subset(method, nm, k, 0, problems=train.problems)
            except Exception as exc:  # the reference's errors are part of the contract
                out[key] = {"error": type(exc).__name__}
                continue
            labels = classify.label_best_in_subset(nm, sub)
            rec = {"config_indices": [int(i) for i in sub.config_indices], "k_actual": int(sub.k_actual),
                   "labels": [int(x) for x in labels], "ceiling": repr(evaluate.subset_ceiling(test, sub))}
            for preset in ("A", "B", "C"):
                tree = classify.train_tree(feats, labels, classify.TREE_PRESETS[preset], n_classes=sub.k_actual)
                pred = lambda x, t=tree: classify.predict_tree(t, x)  # noqa: E731
                rep = evaluate.classifier_score(test, sub, pred)
                rep_all = evaluate.classifier_score(pm, sub, pred)
                rec[f"tree{preset}"] = [repr(rep.achieved), repr(rep_all.achieved), int(tree.n_nodes)]
            out[key] = rec
    return out


def reference_modules() -> dict:
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    return {m: importlib.import_module(f"kernelprune.{m}")
            for m in ("classify", "dataset", "evaluate", "normalize", "selection")}


def main() -> None:
    mods = reference_modules()
    gold = {"generator": "oracle/gen_golden_tables.py", "reference": str(REF), "tables": {}}
    for path in sorted((ROOT / "data" / "sweeps").glob("*.csv")):
        data = path.read_bytes()
        rec = run_chain(mods, data.decode())
        rec["sha256"] = hashlib.sha256(data).hexdigest()
        gold["tables"][path.name] = rec
        print(f"{path.name}: {rec['shape']}", flush=True)
    OUT.write_text(json.dumps(gold, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
