"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/graphmd_b200.h declares, and its host-side helpers (RNG, supercell,
ToyPotentialParams::init) are identical to the oracle's restatement."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "graphmd_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gmd_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = G.lib()
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/graphmd_b200.h but not exported"
    assert sorted(G.EXPORTS) == syms


def test_version_and_sm100a():
    assert b"sm_100a" in G.lib().gmd_version()
    out = os.popen(f"cuobjdump --list-elf {G.LIB_PATH} 2>/dev/null").read()
    if out:
        assert "sm_100a" in out


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = G.lib().gmd_create(0, C.byref(h))
    assert rc != G.GMD_OK and not h.value
    with pytest.raises(G.Error):
        G._Handle(0)


def test_null_handle_is_an_error():
    assert G.lib().gmd_forward(None, None, None, None, None, None, 0) == G.GMD_ERR_ARG
    assert G.lib().gmd_build(None, 1, None, None, None, None, 1.0, 0.0, 0.0, 1, 1, 0) == G.GMD_ERR_ARG


def test_rng_matches_oracle(oracle_c):
    np.testing.assert_array_equal(G.rng_uniform(7, 999, 0.0, 100.0), oracle_c.rng_uniform(7, 999, 0.0, 100.0))
    np.testing.assert_array_equal(G.rng_uniform(123, 10), oracle_c.rng_uniform(123, 10))


@pytest.mark.parametrize("seed,F,K,L,r3", [(12345, 16, 8, 2, 0.0), (7, 16, 8, 3, 3.0), (1, 8, 4, 1, 0.0)])
def test_params_init_matches_oracle(oracle_c, seed, F, K, L, r3):
    p = G.ToyPotentialParams.init(seed, F, K, L, 5.0, r3)
    np.testing.assert_array_equal(p.blob, oracle_c.params_init(seed, F, K, L, 5.0, r3))
    assert len(p.embedding) == 119 * F and len(p.readout) == F


@pytest.mark.parametrize("reps,amp,seed", [((2, 2, 2), 0.05, 9), ((3, 2, 2), 0.05, 6), ((4, 1, 3), 0.0, 0)])
def test_supercell_matches_oracle(oracle_c, reps, amp, seed):
    q = S.fixture("quartz")
    s = G.make_supercell(q, reps, amp, seed)
    op, oz, ol = oracle_c.supercell(q.positions, q.species, q.lattice, reps, amp, seed)
    np.testing.assert_array_equal(s.positions, op)
    np.testing.assert_array_equal(s.species, oz)
    np.testing.assert_array_equal(s.lattice, ol)


def test_params_validation():
    p = G.ToyPotentialParams.init(1)
    p.blob[3] = np.nan
    with pytest.raises(G.Error, match="non-finite"):
        p.validate()
    with pytest.raises(G.Error):
        G.random_perturb(S.quartz((1, 1, 1)), -1.0, 0)


def test_oracle_is_test_only():
    """The product package never links or imports the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2506_02023_b200")
    banned = ("from oracle", "import oracle", "gmd_oracle", "libgraphmd_ref", "orc_", "gref_")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                for b in banned:
                    assert b not in txt, f"{f} references {b}"


def test_no_float_atomics():
    """north_star (3): segment sums without float atomics.  Every per-node sum
    is a fixed-order row reduction written by one thread (plain read-add-write);
    the SASS of the whole library holds no floating-point atomic or reduction
    (integer counters and the order-preserving u64 encodings of doubles used
    for exact min/max are allowed)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", G.LIB_PATH], capture_output=True, text=True).stdout
    ops = set(re.findall(r"\b((?:RED|ATOM)[A-Z]*\.[A-Z0-9_.]+)", sass))
    assert ops, "no atomics at all: SASS listing empty?"
    bad = sorted(o for o in ops if re.search(r"\.(F16|BF16|F32|F64|FADD)\b|\.F32\.|\.F64\.", o))
    assert not bad, bad
