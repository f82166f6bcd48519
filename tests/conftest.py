from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def golden(name: str):
    path = GOLDEN / f"{name}.npz"
    if not path.exists():
        path = GOLDEN / f"run_{name}.npz"
    return np.load(path, allow_pickle=True)


def toy_dataset(n_cases=24, n_features=3, seed=0):
    """Same construction as the reference fixture (pkg/tests/conftest.py:22-30)."""
    r = np.random.default_rng(seed)
    X = r.uniform(-2.0, 2.0, size=(n_cases, n_features))
    y = X[:, 0] * X[:, 1] - X[:, 2 % n_features] + 0.5
    return X, y


@pytest.fixture(scope="session")
def lib():
    """The CUDA engine; GPU tests fail loudly (not skip) if it cannot load."""
    from paper_2106_04034_b200 import _lib
    return _lib.load()
