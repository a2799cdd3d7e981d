"""Test configuration: the ``gpu`` marker and shared fixtures.

``-m "not gpu"`` runs here (no GPU): oracle vs golden vectors, host logic, the
C-ABI export table, multi-process (gloo) sharding. ``-m gpu`` runs on a B200 and
compares the CUDA path (through the C ABI) with the oracle.
"""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); calls the CUDA kernels")


@pytest.fixture(scope="session")
def ref_vectors():
    return dict(np.load(GOLDEN / "ref_vectors.npz"))


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(20240811)
