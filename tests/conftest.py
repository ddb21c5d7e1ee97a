"""Shared test fixtures.  `-m "not gpu"` runs on CPU (oracle vs golden,
generators, C-ABI surface, gloo sharding); `-m gpu` runs the CUDA parity
suite on a B200 and fails (never skips) if the device or library is missing."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")
GOLDEN_MATS = ("banded24", "banded40", "grid6", "grid10", "fixture11", "dense12")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (sm_100a) and libsfgpu.so")
    config.addinivalue_line("markers", "slow: full-size configurations")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN_PATH))


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


def golden_matrix(golden, name):
    from oracle.oracle import Csc
    cp = golden[f"{name}/colptr"]
    return Csc(len(cp) - 1, cp, golden[f"{name}/rowidx"], golden[f"{name}/values"])
