import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a) and librocp_b200.so")
    config.addinivalue_line("markers", "slow: long-running (config-size) GPU checks")


@pytest.fixture(scope="session")
def dev():
    import paper_2007_10798_b200 as rocp
    d = rocp.Device(0)
    yield d
    d.close()
