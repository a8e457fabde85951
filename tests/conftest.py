import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built libhs.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir() -> Path:
    return GOLDEN


@pytest.fixture(scope="session")
def cuda():
    """torch CUDA device for GPU tests (plumbing only: device buffers)."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected but no CUDA device is visible")
    from paper_2603_12831_b200 import _lib

    _lib.load()
    _lib.require_device()
    return torch.device("cuda:0")
