import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    import port as _port  # oracle/port.py (test infrastructure)

    _port.build()
    return _port


@pytest.fixture(scope="session")
def native():
    from paper_1510_07230_b200 import native as _native

    _native.lib()
    return _native
