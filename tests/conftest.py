import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpcdm.so")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle

HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


@pytest.fixture(scope="session")
def gpu():
    """The built library on a CUDA device; GPU tests fail loudly without one."""
    import torch
    from paper_1212_0873_b200 import build, pcdm
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    build.build()
    pcdm.load()
    return torch.device("cuda:0")
