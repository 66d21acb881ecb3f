import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the library's tuning / test knobs (PCDM_LAYOUT, PCDM_HOT_STAGE, ...) are read only when
# PCDM_DEBUG_KNOBS=1 (csrc/internal.h knob()); the tests force layouts and loops with them
os.environ["PCDM_DEBUG_KNOBS"] = "1"
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpcdm.so")
    config.addinivalue_line("markers", "slow: long-running case")
    config.addinivalue_line("markers", "fullrun: full-length oracle parity (oracle runs start with the gpu fixture)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle

HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


@pytest.fixture(scope="session")
def gpu(request):
    """The built library on a CUDA device; GPU tests fail loudly without one.
    When full-length parity tests are selected, their oracle runs (minutes of
    serial CPU work each) are started here in background processes, so they
    overlap the rest of the GPU suite (tests/fullrun_jobs.py)."""
    import torch
    from paper_1212_0873_b200 import build, pcdm
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    build.build()
    pcdm.load()
    dev = torch.device("cuda:0")
    if any(item.get_closest_marker("fullrun") for item in request.session.items):
        import fullrun_jobs
        fullrun_jobs.start(dev)
        request.addfinalizer(fullrun_jobs.cleanup)
    return dev


def pytest_collection_modifyitems(config, items):
    """Full-length parity tests go last: their oracle jobs run in the background meanwhile."""
    items.sort(key=lambda it: 1 if it.get_closest_marker("fullrun") else 0)
