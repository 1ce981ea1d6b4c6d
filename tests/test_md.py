"""On-device molecular dynamics: velocity_verlet_step /
run_md (proj/src/md.cpp:11-160) with positions, velocities and forces resident
in HBM, against the fp64 oracle restatement (oracle/gmd_oracle.c orc_md_run),
which is pinned bit-for-bit to the reference's own run_md (oracle/_ref).

Tolerances: forces are fp32-accurate (tests/test_gpu_model.py), so a
trajectory drifts from the fp64 one by ~|dF| a dt^2 steps^2: over 20 steps of
1 fs the positions stay within 1e-5 A and the velocities within 1e-5 A/fs;
per-step potential energies within 2e-6 eV/atom and kinetic energies within
1e-6 eV/atom; the GPU trajectory conserves the total energy as well as the
oracle's does (|drift difference| <= 2e-5 eV/atom)."""
import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S


def test_atomic_mass_table():
    z = np.array([1, 8, 14, 54, 55, 118], np.int32)
    from oracle.oracle import Oracle
    o = Oracle("c")
    import ctypes as C
    o.lib.orc_atomic_mass.restype = C.c_double
    ref = [o.lib.orc_atomic_mass(int(v)) for v in z]
    np.testing.assert_array_equal(G.atomic_mass(z), ref)
    with pytest.raises(G.Error, match="atomic number out of range"):
        G.atomic_mass([0])


def test_maxwell_boltzmann_matches_oracle(oracle_c):
    """Velocities of init_md_state are the oracle's (same RNG stream, same
    momentum removal), and the total momentum vanishes."""
    s = S.quartz((2, 2, 2))
    v = G.maxwell_boltzmann_velocities(s, 300.0, 7)
    r = oracle_c.md_run(*S.as_args(s), oracle_c.params_init(1, 16, 8, 1, 5.0), 16, 8, 1, 5.0, 0.0,
                        1.0, 0, 300.0, 7)
    np.testing.assert_array_equal(v, r["vel"])
    p = (v * G.atomic_mass(s.species)[:, None]).sum(0)
    assert np.abs(p).max() < 1e-12
    assert not G.maxwell_boltzmann_velocities(s, 0.0, 7).any()


def test_oracle_md_pinned_to_reference(oracle_c, oracle_ref):
    s = S.quartz((2, 2, 2))
    prm = oracle_c.params_init(12345, 16, 8, 2, 5.0)
    a = oracle_c.md_run(*S.as_args(s), prm, 16, 8, 2, 5.0, 0.0, 1.0, 5, 300.0, 3)
    b = oracle_ref.md_run(*S.as_args(s), prm, 16, 8, 2, 5.0, 0.0, 1.0, 5, 300.0, 3)
    np.testing.assert_allclose(a["pos"], b["pos"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(a["vel"], b["vel"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(a["records"], b["records"], rtol=1e-10, atol=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("r3", [0.0, 3.0])
def test_md_trajectory_matches_oracle(oracle_c, r3):
    s = S.quartz((3, 3, 3))
    n = s.size()
    prm = G.ToyPotentialParams.init(12345, 16, 8, 2, 5.0, r3)
    opts = G.MDOptions(dt=1.0, steps=20, partitions=2, allow_narrow=True, seed=11,
                       init_temperature=300.0)
    res = G.run_md(s, prm, opts)
    ref = oracle_c.md_run(*S.as_args(s), prm.blob, 16, 8, 2, 5.0, r3, 1.0, 20, 300.0, 11)
    assert len(res.records) == 21
    rec = np.array([[r.potential, r.kinetic, r.total, r.max_force] for r in res.records])
    assert np.abs(rec[:, 0] - ref["records"][:, 0]).max() / n <= 2e-6
    assert np.abs(rec[:, 1] - ref["records"][:, 1]).max() / n <= 1e-6
    np.testing.assert_allclose(rec[:, 3], ref["records"][:, 3], rtol=0, atol=2e-4)
    drift_gpu = rec[-1, 2] - rec[0, 2]
    drift_ref = ref["records"][-1, 2] - ref["records"][0, 2]
    assert abs(drift_gpu - drift_ref) / n <= 2e-5
    np.testing.assert_allclose(res.state.positions(), ref["pos"], rtol=0, atol=1e-5)
    np.testing.assert_allclose(res.state.velocities(), ref["vel"], rtol=0, atol=1e-5)
    np.testing.assert_allclose(res.state.forces_host(), ref["forces"], rtol=0, atol=2e-4)
    assert res.state.step == 20
    assert all(r.timing.graph_creation > 0 for r in res.records)


@pytest.mark.gpu
def test_md_wrap_and_partition_invariance():
    """Atoms leave the cell and are wrapped back (wrap_positions); the device
    trajectory is bitwise independent of the slab count."""
    s = S.quartz((3, 3, 3))
    prm = G.ToyPotentialParams.init(5, 16, 8, 2, 5.0)
    out = []
    for p in (1, 3):
        opts = G.MDOptions(dt=2.0, steps=6, partitions=p, allow_narrow=True, seed=2,
                           init_temperature=3000.0)
        out.append(G.run_md(s, prm, opts))
    np.testing.assert_array_equal(out[0].state.positions(), out[1].state.positions())
    np.testing.assert_array_equal(out[0].state.velocities(), out[1].state.velocities())
    f = np.linalg.solve(s.lattice.T, out[0].state.positions().T).T
    assert (f >= 0).all() and (f < 1).all()


@pytest.mark.gpu
def test_md_errors_and_csv(tmp_path):
    s = S.quartz((2, 2, 2))
    prm = G.ToyPotentialParams.init(5, 16, 8, 1, 5.0)
    st = G.init_md_state(s, G.MDOptions(seed=1))
    with pytest.raises(G.Error, match="requires forces"):
        G.velocity_verlet_step(st, prm, G.MDOptions())
    opts = G.MDOptions(steps=2, seed=1, energy_csv=str(tmp_path / "e.csv"),
                       timing_csv=str(tmp_path / "t.csv"))
    G.run_md(s, prm, opts)
    lines = open(tmp_path / "e.csv").read().splitlines()
    assert lines[0].startswith("step,potential_ev,kinetic_ev,total_ev,max_force_ev_per_a")
    assert len(lines) == 4
    assert open(tmp_path / "t.csv").read().splitlines()[0] == (
        "step,Graph Creation,Feature Calculation,Forward Pass,Backward Pass")
    bad = G.MDOptions(dt=-1.0)
    st2 = G.init_md_state(s, G.MDOptions(seed=1))
    G.md_evaluate(st2, prm, bad)
    with pytest.raises(G.Error, match="time step"):
        G.velocity_verlet_step(st2, prm, bad)
