"""Run the reference package's own unit tests (/root/reference/pkg/tests) against this
package: ``kernelprune`` is aliased to ``paper_2008_13145_b200`` by
tests/ref_alias_plugin.py.  Covers the modules on the host side of the hot path
(dataset, normalize, pca, selection, classify, evaluate, codegen); the CLI/pipeline
suites (test_cli.py, test_acceptance.py) exercise host orchestration that is out of
scope and are not run.  Skipped where the reference is absent."""

import os
import subprocess
import sys

import pytest

from conftest import REFERENCE_TESTS, ROOT, reference_available

SUITES = ("test_dataset.py", "test_normalize.py", "test_pca.py", "test_selection.py",
          "test_classify.py", "test_evaluate.py", "test_codegen.py")


@pytest.mark.skipif(not reference_available(), reason="reference package not present")
@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_passes_against_this_package(suite, tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(ROOT / "tests"), str(REFERENCE_TESTS)])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "ref_alias_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(tmp_path), "-c", os.devnull, str(REFERENCE_TESTS / suite)]
    proc = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0, proc.stdout[-4000:] + proc.stderr[-2000:]
    assert "passed" in proc.stdout
