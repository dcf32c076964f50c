import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")
REFERENCE_TESTS = Path("/root/reference/pkg/tests")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libkpgemm.so")


def reference_available() -> bool:
    return (REFERENCE_SRC / "kernelprune" / "__init__.py").exists()


@pytest.fixture(scope="session")
def kernelprune_ref():
    """The read-only reference package, imported from /root/reference (build
    container only); tests using it skip elsewhere."""
    if not reference_available():
        pytest.skip("reference package not present on this machine")
    import importlib
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    mods = {}
    for name in ("dataset", "normalize", "selection", "classify", "evaluate", "codegen", "pca"):
        mods[name] = importlib.import_module(f"kernelprune.{name}")
    return mods


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
