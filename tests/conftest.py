import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libnskb.so; run via gpurun")


@pytest.fixture(scope="session")
def dev():
    """Initialised device context (GPU tests only)."""
    from paper_2409_11600_b200 import _lib

    return _lib.ctx.init(0)


@pytest.fixture
def session(dev):
    from paper_2409_11600_b200.runtime import Session

    return Session(seed=0)
