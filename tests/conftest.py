import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running parity sweeps")


@pytest.fixture(scope="session")
def oracle_c():
    from oracle.oracle import Oracle
    return Oracle("c")


@pytest.fixture(scope="session")
def oracle_ref():
    from oracle.oracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("ref")
