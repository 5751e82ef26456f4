import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref/librnla_ref.so not built")
    return oracle.Oracle("reference")
