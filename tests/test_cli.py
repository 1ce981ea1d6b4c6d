"""the reference's command-line driver on the B200 path
(tools/graphmd_cli: audit / bench / md with the reference's flags, CSV schemas
from proj/docs/formats.md and exit codes) and the extended-XYZ fixture I/O
(system.cpp:95-186) it reads and writes.

CPU tests pin the Python and C++ XYZ readers/writers to the compiled
reference (byte-identical files, identical parse errors) and the CLI's
configuration errors (exit code 2, before any GPU work); GPU tests run every
subcommand."""
import csv
import os
import subprocess

import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CLI = os.path.join(ROOT, "tools", "graphmd_cli")


def build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True, capture_output=True)


def cli(*args, timeout=600):
    build()
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)


def read_csv(path):
    with open(path) as f:
        rows = list(csv.reader(f))
    return rows[0], rows[1:]


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
    # the C++ reader behind the CLI: a configuration error with the same text
    r = cli("audit", "--fixture", p)
    assert r.returncode == 2
    assert r.stderr.strip() == f"config error: {ref.value}"


def test_non_periodic_without_lattice(tmp_path):
    p = str(tmp_path / "m.xyz")
    with open(p, "w") as f:
        f.write('2\npbc="F F F"\nO 0 0 0\nH 0.9 0 0\n')
    s = G.load_xyz(p)
    assert tuple(s.pbc) == (False, False, False)
    np.testing.assert_array_equal(s.lattice, np.eye(3))


# ------------------------------------------------------- CLI config (CPU)
@pytest.mark.parametrize("args", [
    [],
    ["frobnicate"],
    ["audit"],                                              # --fixture required
    ["audit", "--fixture", "/nonexistent.xyz"],
    ["bench", "--fixture", "FIX", "--mode", "bogus"],
    ["md", "--fixture", "FIX", "--bogus", "1"],
    ["audit", "--fixture", "FIX", "--reps", "1,2"],
    ["audit", "--fixture", "FIX", "--cutoff", "five"],
    ["md", "--fixture", "FIX", "--dt", "-1"],
    ["md", "--fixture", "FIX", "--steps"],
])
def test_cli_configuration_errors(quartz_xyz, args):
    r = cli(*[quartz_xyz if a == "FIX" else a for a in args])
    assert r.returncode == 2, (r.stdout, r.stderr)


def test_cli_help():
    r = cli("--help")
    assert r.returncode == 0 and "audit" in r.stdout and "bench" in r.stdout and "md" in r.stdout


# ------------------------------------------------------------- CLI on GPU
@pytest.mark.gpu
def test_audit_passes_and_negative_control_fails(quartz_xyz):
    r = cli("audit", "--fixture", quartz_xyz, "--reps", "3,3,6", "--partitions", "1,2,4", "--cutoff", "5")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert [ln.split()[0] for ln in lines] == ["p=1", "p=2", "p=4"]
    # one-partition and partitioned evaluations are bitwise equal here
    assert all("max|dE|/atom=0 max|dF|=0 max|dS|=0" in ln for ln in lines), lines
    # (slabs wider than 2 rc, so the PURE span is non-empty and the wrong span differs)
    bad = cli("audit", "--fixture", quartz_xyz, "--reps", "3,3,6", "--partitions", "2", "--cutoff", "5",
              "--corrupt-plan")
    assert bad.returncode == 1 and "FAIL p=2" in bad.stderr
    tb = cli("audit", "--fixture", quartz_xyz, "--reps", "3,3,3", "--partitions", "1,3", "--cutoff", "5",
             "--threebody-cutoff", "3", "--tol-energy", "1e-6", "--tol-force", "1e-5", "--tol-stress", "1e-6")
    assert tb.returncode == 0, tb.stderr


@pytest.mark.gpu
def test_bench_modes_emit_reference_schemas(quartz_xyz, tmp_path):
    common = ["--fixture", quartz_xyz, "--reps", "3,3,3", "--cutoff", "5", "--repeat", "3", "--keep-last", "2"]
    heads = {
        "strong": "mode,p,threads,atoms,edges,time_s,baseline_s,normalized",
        "weak": "mode,p,threads,atoms,edges,time_s,baseline_s,normalized",
        "breakdown": "p,atoms,graph_creation_s,feature_calculation_s,forward_pass_s,backward_pass_s,total_s",
        "density": "density_factor,atoms,edges,time_s",
        "capacity": "budget_bytes,scale,atoms,estimated_bytes,status,time_s",
    }
    for mode, head in heads.items():
        out = str(tmp_path / f"{mode}.csv")
        r = cli("bench", *common, "--mode", mode, "--partitions", "1,2", "--out", out)
        assert r.returncode == 0, r.stderr
        h, rows = read_csv(out)
        assert ",".join(h) == head
        if mode in ("strong", "weak"):
            assert [int(x[1]) for x in rows] == [1, 2]
            assert int(rows[0][3]) == 243 and int(rows[0][4]) > 0
            if mode == "weak":
                assert int(rows[1][3]) == 2 * 243
            assert all(float(x[5]) > 0 and float(x[7]) > 0 for x in rows)
        elif mode == "breakdown":
            for x in rows:
                parts = [float(v) for v in x[2:6]]
                assert abs(sum(parts) - float(x[6])) < 1e-9 and min(parts) >= 0
        elif mode == "density":
            assert [float(x[0]) for x in rows] == [1.0, 2.0]
            assert int(rows[1][2]) > int(rows[0][2])  # denser -> more edges
        else:
            assert len(rows) == 1 and rows[0][4] == "ok" and int(rows[0][1]) >= 1
    tiny = cli("bench", *common, "--mode", "capacity", "--budget-bytes", "1000")
    assert tiny.returncode == 0
    assert tiny.stdout.strip().splitlines()[1].endswith(",exceeded,0")


@pytest.mark.gpu
def test_md_outputs_snapshots_and_paired_run(quartz_xyz, tmp_path):
    e, t, traj = str(tmp_path / "e.csv"), str(tmp_path / "t.csv"), str(tmp_path / "snap")
    r = cli("md", "--fixture", quartz_xyz, "--reps", "3,3,3", "--cutoff", "5", "--partitions", "2",
            "--steps", "5", "--dt", "0.5", "--temperature", "300", "--out", e, "--timing-out", t,
            "--traj", traj, "--snapshot-every", "2", "--paired", "--pair-tol", "1e-12")
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("steps=5 E_total_final=")
    assert "paired max|dx|=0 (p=2 vs serial)" in r.stdout
    h, rows = read_csv(e)
    assert ",".join(h) == ("step,potential_ev,kinetic_ev,total_ev,max_force_ev_per_a,graph_creation_s,"
                           "feature_calculation_s,forward_pass_s,backward_pass_s")
    assert [int(x[0]) for x in rows] == list(range(6))
    h, trows = read_csv(t)
    assert ",".join(h) == "step,Graph Creation,Feature Calculation,Forward Pass,Backward Pass"
    assert len(trows) == 6
    for k in (0, 2, 4):
        assert os.path.exists(f"{traj}.{k}.xyz")
    assert not os.path.exists(f"{traj}.5.xyz")
    # the Python mirror writes the same trajectory byte for byte
    s = G.make_supercell(G.load_xyz(quartz_xyz), (3, 3, 3))
    prm = G.ToyPotentialParams.init(12345, 16, 8, 2, 5.0, 0.0)
    opts = G.MDOptions(dt=0.5, steps=5, partitions=2, seed=12345, init_temperature=300.0,
                       trajectory_xyz=str(tmp_path / "py"), snapshot_every=2)
    res = G.run_md(s, prm, opts)
    for k in (0, 2, 4):
        assert open(f"{traj}.{k}.xyz").read() == open(f"{tmp_path}/py.{k}.xyz").read()
    np.testing.assert_allclose([x.total for x in res.records], [float(x[3]) for x in rows], rtol=1e-11)


# ------------------------------------------- parameter files (GMPT, CPU)
CPP = os.path.join(HERE, "cpp", "test_cpp_api")


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
