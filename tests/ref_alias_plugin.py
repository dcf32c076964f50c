"""pytest plugin: make ``import kernelprune[.X]`` resolve to this package so the
REFERENCE's own unit tests (/root/reference/pkg/tests) run against the B200 build's
host-side restatement.  Test infrastructure only."""

import importlib
import sys

MODULES = ("errors", "dataset", "normalize", "pca", "selection", "classify", "evaluate", "codegen", "pipeline",
           "cli")


def pytest_load_initial_conftests(early_config, parser, args):
    pkg = importlib.import_module("paper_2008_13145_b200")
    sys.modules["kernelprune"] = pkg
    for name in MODULES:
        sys.modules[f"kernelprune.{name}"] = importlib.import_module(f"paper_2008_13145_b200.{name}")
