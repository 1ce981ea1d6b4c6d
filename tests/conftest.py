import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# fp32-vs-fp64 tolerances of every GPU-vs-oracle comparison, calibrated in
# tests/test_gpu_scale.py::test_tolerance_calibration: the fp64 reference run
# on fp32-ROUNDED positions moves per-atom energies by 1.5e-5 eV at C3, above
# SURVEY §8(c)'s proposed 1e-5, so the proposal is widened 2x to sit at that
# floor (the GPU keeps fp64 positions and lands well inside it: 3e-6 eV):
#   per-atom energy |dE_i| <= 2e-5 eV; total |dE|/N <= 2e-6 eV/atom;
#   forces max |dF| <= 2e-4 eV/A and <= 2e-5 x max |F|; stress <= 2e-6 eV/A^3
TOL_EA, TOL_E, TOL_F, TOL_FREL, TOL_S = 2e-5, 2e-6, 2e-4, 2e-5, 2e-6
SURVEY_TOL = dict(dE_i=1e-5, dE_N=1e-6, dF=1e-4, dS=1e-6)  # SURVEY §8(c) proposal


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
