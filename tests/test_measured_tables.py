"""North-star metric parity on the MEASURED B200 tables (data/sweeps/*.csv): this
package's split -> normalize -> select_subset (kmeans, spectral, pca_kmeans, tree) ->
treeA/B/C -> classifier_score chain must be repr-identical to the reference's
(kernelprune, evaluate.py:71-101, selection.py:491-521).

Two legs: against tests/golden/measured_tables.json (recorded from the reference by
oracle/gen_golden_tables.py; runs everywhere), and live against the imported
reference where /root/reference exists."""

import hashlib
import importlib
import json
from pathlib import Path

import pytest

from conftest import ROOT, reference_available
from oracle.gen_golden_tables import reference_modules, run_chain

GOLD = json.loads((Path(__file__).parent / "golden" / "measured_tables.json").read_text())
TABLES = sorted(p.name for p in (ROOT / "data" / "sweeps").glob("*.csv"))
OURS = {m: importlib.import_module(f"paper_2008_13145_b200.{m}")
        for m in ("classify", "dataset", "evaluate", "normalize", "selection")}


def test_every_table_has_a_golden_record():
    assert TABLES, "no measured tables under data/sweeps"
    assert sorted(GOLD["tables"]) == TABLES


@pytest.mark.parametrize("name", TABLES)
def test_selection_chain_matches_reference_golden(name):
    data = (ROOT / "data" / "sweeps" / name).read_bytes()
    exp = GOLD["tables"][name]
    assert hashlib.sha256(data).hexdigest() == exp["sha256"], \
        f"{name} changed since the golden was recorded: re-run oracle/gen_golden_tables.py"
    got = run_chain(OURS, data.decode())
    got["sha256"] = exp["sha256"]
    for key in exp:
        assert got[key] == exp[key], f"{name}: {key} differs from the reference"


@pytest.mark.skipif(not reference_available(), reason="reference package not present")
@pytest.mark.parametrize("name", ["vgg16_simt.csv", "resnet50_simt+tf32.csv", "vgg16_bf16.csv"])
def test_selection_chain_matches_live_reference(name):
    text = (ROOT / "data" / "sweeps" / name).read_text()
    assert run_chain(OURS, text) == run_chain(reference_modules(), text)
