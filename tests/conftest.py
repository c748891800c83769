import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run through gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def dev():
    """CUDA device for -m gpu tests; the CUDA extension must load (no fallback)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu test run without a visible GPU")
    return torch.device("cuda:0")
