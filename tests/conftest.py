import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as o
    if not o.available("port"):
        o.build()
    return o.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as o
    if not o.available("reference"):
        try:
            o.build()
        except RuntimeError:
            pass
    if not o.available("reference"):
        pytest.skip("reference oracle (oracle/_ref) not built")
    return o.Oracle("reference")
