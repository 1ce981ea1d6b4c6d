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


# Kernel families selectable per call through the library's environment
# switches (read on every gmd_forward):
#   ffma2   - default: packed-FP32 (FFMA2) conv + backward edge pass
#   ffma    - scalar-FFMA conv + backward edge pass (A/B reference)
#   tcgen05 - backward radial contraction on tcgen05/TMEM (GMD_BWD_TC=1)
KERNELS = {
    "ffma2": {"GMD_BWD_TC": "0", "GMD_CONV_VARIANT": "0", "GMD_BWD_VARIANT": "0"},
    "ffma": {"GMD_BWD_TC": "0", "GMD_CONV_VARIANT": "1", "GMD_BWD_VARIANT": "1"},
    "tcgen05": {"GMD_BWD_TC": "1", "GMD_CONV_VARIANT": "0", "GMD_BWD_VARIANT": "0"},
}


def use_kernels(monkeypatch, name):
    for k, v in KERNELS[name].items():
        monkeypatch.setenv(k, v)
