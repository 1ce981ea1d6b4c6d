"""The C++ drop-in header (include/graphmd_b200/graphmd.hpp) compiles against
the C ABI (CPU) and passes the reference's own test scenarios on the GPU."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "test_cpp_api")


def build():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True, capture_output=True)


def test_cpp_header_builds():
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_dropin_parity():
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "FAIL" not in r.stdout
