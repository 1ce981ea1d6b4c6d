"""The reference's OWN test programs, compiled UNMODIFIED against the B200
drop-in (tests/cpp/Makefile target `ref`: proj/tests/acceptance.cpp and the
doctest unit tests proj/tests/test_*.cpp with include/compat ahead on the
include path, linked to libgraphmd_b200.so only -- none of the reference's
library code).  Built in the container that holds /root/reference; the
binaries travel to the GPU box with the repo.

Expected outcomes: everything passes except the checks whose tolerance is
tighter than fp32 features can meet (the contract is SURVEY §8(c)'s fp32
tolerance, tests/conftest.py) and the reference's CPU-thread scaling shape.
Each such failure is listed below with its reason; any other failure fails
this test."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "tests", "cpp", "ref")


def run(binary, timeout=1500, env=None):
    path = os.path.join(REF, binary)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C tests/cpp ref, needs /root/reference)")
    r = subprocess.run([path], cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env={**os.environ, **(env or {})})
    print(r.stdout[-20000:])
    return r


# unit-test cases whose assertions are fp64-tight (1e-8 .. 1e-14 absolute or
# relative) on quantities the GPU computes in fp32 features: contract is the
# fp32 tolerance of tests/conftest.py, checked by this repo's own tests
FP32_TIGHT = {
    "make_supercell: per-atom energy invariance": "1e-10 eV per atom (test_system.cpp:97)",
    "isolated atom: embedding readout, zero forces and stress": "energy to 1e-14 relative",
    "forces match finite differences": "FD of an fp32-feature energy: noise ~1e-6 eV / 2e-4 A",
    "stress matches strain finite differences": "same, strain FD to 1e-6",
    "rotation invariance and force equivariance": "1e-9 relative energy, 1e-8 eV/A forces",
    # the bound 0.5 a_max t^2 (+1e-12) is the displacement of the max-force
    # atom under a constant force: it holds with equality up to how that force
    # drifts over 10 steps, so fp32 force noise decides it (it passed or
    # failed with the rounding order of the forward's reductions)
    "zero temperature perfect crystal stays put": "equality bound, 1e-12 A slack (test_md.cpp:76-94)",
}
# pass only in exact-forces mode (GMD_EXACT_FORCES=1: fp64 per-lane gradient
# sums in the tuned F = 16 backward, Newton's third law to the last bit)
EXACT_ONLY = {
    "translation invariance: forces sum to zero": "|sum F| <= 1e-8",
    "momentum conservation": "|P| <= 1e-8 after 100 steps",
}
# acceptance criteria: 6 = finite differences at 1e-6 (fp32, as above);
# 7 = CPU thread scaling of p partitions (one GPU: partitions add no compute)
ACCEPTANCE_EXPECTED_FAIL = {"6", "7"}


@pytest.mark.parametrize("exact", [True, False])
def test_reference_unit_tests(exact):
    r = run("unit_tests", env={"GMD_EXACT_FORCES": "1" if exact else "0"})
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:] + r.stderr[-2000:]
    failed = set(re.findall(r'\[test case "([^"]+)"\]', r.stdout))
    failed |= set(re.findall(r'test case "([^"]+)" threw', r.stdout))
    print("failed:", sorted(failed))
    allowed = set(FP32_TIGHT) | (set() if exact else set(EXACT_ONLY))
    assert int(m.group(1)) == 72
    assert failed <= allowed, sorted(failed - allowed)


def test_reference_acceptance():
    r = run("acceptance")
    got = dict(re.findall(r"criterion (\d+) \([^)]*\): (PASS|FAIL|SKIP)", r.stdout))
    print(got)
    assert len(got) == 9
    for c, verdict in got.items():
        if c not in ACCEPTANCE_EXPECTED_FAIL:
            assert verdict == "PASS", (c, r.stdout)
