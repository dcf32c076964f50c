"""GPU: the CLI's B200 additions -- ``sweep`` measures a benchmark CSV in the reference's
format (dataset.py:36) and ``run`` consumes it unchanged (pipeline.py:128-217), and
``run --sweep-set`` measures the table inside the pipeline."""

import json

import pytest

from paper_2008_13145_b200 import cli, gemm, parse_benchmark_csv
from paper_2008_13145_b200.pipeline import SWEEP_KEYS

pytestmark = pytest.mark.gpu


def test_sweep_then_run(cuda_device, tmp_path, capsys):
    table = tmp_path / "vgg16_bf16_b1.csv"
    assert cli.main(["sweep", "--set", "vgg16", "--batches", "1", "--family", "bf16", "--output", str(table),
                     "--min-ms", "0.5"]) == 0
    pm = parse_benchmark_csv(table.read_text())
    assert (pm.n_problems, pm.n_configs) == (12, len(gemm.family_configs("bf16"))) and (pm.values > 0).all()
    out = tmp_path / "out"
    assert cli.main(["run", "--input", str(table), "--output-dir", str(out), "--scheme", "scaled",
                     "--method", "kmeans,tree", "--k", "2,3", "--classifier", "treeA,oracle"]) == 0
    rows = (out / "eval_report.csv").read_text().splitlines()
    assert rows[0] == "method,k,scheme,classifier,ceiling,achieved" and len(rows) == 1 + 2 * 2 * 2
    assert list((out / "models").glob("*.kptree")) and list((out / "selectors").glob("*.inc"))
    resolved = json.loads((out / "resolved_config.json").read_text())
    assert not set(SWEEP_KEYS) & set(resolved)  # the reference's document for CSV runs


def test_run_with_sweep_set(cuda_device, tmp_path):
    out = tmp_path / "out"
    assert cli.main(["run", "--sweep-set", "square", "--sweep-family", "tf32", "--output-dir", str(out),
                     "--scheme", "scaled", "--method", "kmeans", "--k", "2", "--classifier", "treeA",
                     "--test-fraction", "0.3"]) == 0
    pm = parse_benchmark_csv((out / "dataset.csv").read_text())
    assert pm.n_configs == len(gemm.family_configs("tf32")) and (pm.values > 0).all()
    resolved = json.loads((out / "resolved_config.json").read_text())
    assert resolved["sweep_set"] == "square" and resolved["sweep_family"] == "tf32"
