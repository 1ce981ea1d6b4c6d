"""The reference's file formats the drop-in reads and writes: extended XYZ
(system.cpp:95-186; the reference's own tests load their fixtures through it)
and GMPT parameter files (potential.cpp:178-260).  CPU tests pin the Python
readers/writers to the compiled reference: byte-identical files, identical
parse errors."""
import csv
import os
import subprocess

import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CPP = os.path.join(HERE, "cpp", "test_cpp_api")


@pytest.fixture
def quartz_xyz(tmp_path):
    p = str(tmp_path / "quartz.xyz")
    G.save_xyz(S.fixture("quartz"), p)
    return p


# ---------------------------------------------------------------- XYZ (CPU)
SYSTEMS = {
    "quartz": lambda: S.quartz((2, 1, 1)),
    "triclinic": lambda: S.random_gas(40, 3),
    "slab": lambda: G.AtomicSystem(np.array([[0.1, 0.2, 0.3], [1e-17, -2.5, 1e300]]), np.diag([3.0, 4.0, 5.0]),
                                   np.array([1, 118], np.int32), (True, False, True)),
}


@pytest.mark.parametrize("name", list(SYSTEMS))
@pytest.mark.parametrize("comment", ["", "Properties=species:S:1:pos:R:3 step=7"])
def test_xyz_write_byte_identical_and_read_back(oracle_ref, tmp_path, name, comment):
    s = SYSTEMS[name]()
    a, b = str(tmp_path / "a.xyz"), str(tmp_path / "b.xyz")
    G.save_xyz(s, a, comment)
    oracle_ref.save_xyz(s.positions, s.species, s.lattice, [int(x) for x in s.pbc], b, comment)
    assert open(a).read() == open(b).read()
    r = G.load_xyz(b)
    pos, z, lat, pbc = oracle_ref.load_xyz(a)
    np.testing.assert_array_equal(r.positions, pos)
    np.testing.assert_array_equal(r.species, z)
    np.testing.assert_array_equal(r.lattice, lat)
    assert tuple(r.pbc) == tuple(pbc)
    np.testing.assert_array_equal(r.positions, s.positions)  # 17 digits round-trip


BAD = {
    "empty": "",
    "count": "abc\n",
    "no_comment": "1\n",
    "unterminated": '1\nLattice="1 0 0 0 1 0 0 0 1\nH 0 0 0\n',
    "lattice8": '1\nLattice="1 0 0 0 1 0 0 0"\nH 0 0 0\n',
    "pbc2": '1\nLattice="1 0 0 0 1 0 0 0 1" pbc="T F"\nH 0 0 0\n',
    "pbc_no_lattice": '1\npbc="T F F"\nH 0 0 0\n',
    "no_lattice_default_pbc": "1\ncomment\nH 0 0 0\n",
    "symbol": '1\nLattice="1 0 0 0 1 0 0 0 1"\nXx 0 0 0\n',
    "truncated": '2\nLattice="1 0 0 0 1 0 0 0 1"\nH 0 0 0\n',
    "atom_line": '1\nLattice="1 0 0 0 1 0 0 0 1"\nH 0 zero 0\n',
    "singular": '1\nLattice="1 0 0 0 1 0 0 0 0"\nH 0 0 0\n',
}


@pytest.mark.parametrize("case", list(BAD))
def test_xyz_parse_errors_match_reference(oracle_ref, tmp_path, case):
    from oracle.oracle import OracleError
    p = str(tmp_path / f"{case}.xyz")
    with open(p, "w") as f:
        f.write(BAD[case])
    with pytest.raises(OracleError) as ref:
        oracle_ref.load_xyz(p)
    with pytest.raises(G.Error) as mine:
        G.load_xyz(p)
    assert str(mine.value) == str(ref.value)


def test_non_periodic_without_lattice(tmp_path):
    p = str(tmp_path / "m.xyz")
    with open(p, "w") as f:
        f.write('2\npbc="F F F"\nO 0 0 0\nH 0.9 0 0\n')
    s = G.load_xyz(p)
    assert tuple(s.pbc) == (False, False, False)
    np.testing.assert_array_equal(s.lattice, np.eye(3))


# ------------------------------------------------------- CLI config (CPU)
@pytest.mark.parametrize("L,r3", [(2, 0.0), (3, 3.0)])
def test_params_files_byte_identical(oracle_ref, tmp_path, L, r3):
    """ToyPotentialParams::save / load (potential.cpp:178-260): the Python and
    C++ writers produce the reference's bytes; each reader loads the others'."""
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True, capture_output=True)
    p = G.ToyPotentialParams.init(12345, 16, 8, L, 5.0, r3)
    a, b, c, d = (str(tmp_path / f"{k}.gmpt") for k in "abcd")
    p.save(a)
    oracle_ref.params_save(16, 8, L, 5.0, r3, 12345, p.blob, b)
    assert subprocess.run([CPP, "--params-save", c, "12345", str(L), str(r3)]).returncode == 0
    assert open(a, "rb").read() == open(b, "rb").read() == open(c, "rb").read()
    assert subprocess.run([CPP, "--params-copy", b, d]).returncode == 0
    assert open(d, "rb").read() == open(b, "rb").read()
    q = G.ToyPotentialParams.load(b)
    assert (q.feature_width, q.basis_count, q.layers, q.r_atom, q.r_3body, q.seed) == (16, 8, L, 5.0, r3, 12345)
    np.testing.assert_array_equal(q.blob, p.blob)
    F, K, LL, ra, rr, seed, blob = oracle_ref.params_load(a)
    assert (F, K, LL, ra, rr, seed) == (16, 8, L, 5.0, r3, 12345)
    np.testing.assert_array_equal(blob, p.blob)


def _corrupt(good, case):
    import struct
    if case == "magic":
        return b"GMPX" + good[4:]
    if case == "version":
        return good[:4] + struct.pack("<I", 2) + good[8:]
    if case == "truncated":
        return good[:-8]
    if case == "size":  # readout table one entry short, file otherwise consistent
        n = 16
        return good[:-(8 * n + 8)] + struct.pack("<Q", n - 1) + good[-8 * (n - 1):]
    if case == "nonfinite":
        return good[:-8] + struct.pack("<d", float("nan"))
    if case == "cutoff":  # r_3body > r_atom
        return good[:32] + struct.pack("<d", 9.0) + good[40:]
    raise KeyError(case)


@pytest.mark.parametrize("case", ["magic", "version", "truncated", "size", "nonfinite", "cutoff"])
def test_params_file_errors_match_reference(oracle_ref, tmp_path, case):
    from oracle.oracle import OracleError
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True, capture_output=True)
    good = str(tmp_path / "good.gmpt")
    G.ToyPotentialParams.init(7, 16, 8, 2, 5.0, 3.0).save(good)
    bad = str(tmp_path / "bad.gmpt")
    with open(bad, "wb") as f:
        f.write(_corrupt(open(good, "rb").read(), case))
    with pytest.raises(OracleError) as ref:
        oracle_ref.params_load(bad)
    with pytest.raises(G.Error) as mine:
        G.ToyPotentialParams.load(bad)
    assert str(mine.value) == str(ref.value)
    r = subprocess.run([CPP, "--params-copy", bad, str(tmp_path / "x.gmpt")], capture_output=True, text=True)
    assert r.returncode == 3 and r.stdout.strip() == f"error: {ref.value}"
