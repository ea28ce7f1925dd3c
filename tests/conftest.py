"""Shared pytest setup: the ``gpu`` marker, import paths, golden fixtures."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")


def pytest_report_header(config):
    from paper_2009_07226_b200 import _lib
    return f"xct library: {_lib.LIB_PATH.name}"


@pytest.fixture(scope="session")
def golden_manifest():
    return json.loads((GOLDEN / "manifest.json").read_text())


def load_golden(name):
    return np.load(GOLDEN / f"{name}.npz")
