import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the libtag C ABI on CUDA)")
    config.addinivalue_line("markers", "slow: long-running (full-size shapes)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def cuda():
    """GPU tests fail loudly (never skip) when CUDA is missing: the driver runs `-m gpu` on a B200."""
    import torch
    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def tag(cuda):
    from paper_2302_06126_b200 import tag as tagmod
    return tagmod
