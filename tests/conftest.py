"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built native
library; everything else runs on CPU (oracle vs golden vectors, host logic,
library exports, multi-process gloo logic)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built sm_100a library")
    config.addinivalue_line("markers", "slow: longer-running GPU test")


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(GOLDEN / "golden_small.npz"))


@pytest.fixture(scope="session")
def golden_c1():
    return dict(np.load(GOLDEN / "golden_c1.npz"))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


@pytest.fixture(scope="session")
def T(cuda):
    import torch

    return torch
