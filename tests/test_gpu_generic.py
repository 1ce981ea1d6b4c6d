"""Model widths other than the tuned F = 16, K = 8 (the reference accepts any
ToyPotentialParams widths, potential.hpp:15-41): the width-generic kernels
(gmd_generic.cu) against the fp64 oracle, and partition invariance.

Two-body and three-body (SURVEY §8d's F = 64 "CHGNet-width" variant).
Tolerances as tests/test_gpu_model.py (fp32 compute against fp64): per-atom
energy 2e-5 eV, total energy 2e-6 eV/atom, forces 2e-4 eV/A, stress 2e-6 eV/A^3
-- scaled by sqrt(F / 16) for wider features (longer fp32 sums)."""
import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S
from tests.conftest import TOL_E, TOL_EA, TOL_F, TOL_FREL, TOL_S

pytestmark = pytest.mark.gpu


def run(s, prm, p=1):
    r3 = prm.r_3body if prm.threebody() else None
    d = G.Distributed.create_distributed(s, prm.r_atom, r3, p, 1, True)
    return G.forward_distributed(d, prm)


@pytest.mark.parametrize("F,K,L,r3", [(8, 4, 2, 0.0), (32, 8, 2, 0.0), (64, 12, 3, 0.0), (16, 8, 9, 0.0),
                                      (5, 3, 1, 0.0), (128, 32, 1, 0.0), (32, 8, 2, 3.0), (64, 8, 3, 2.8),
                                      (16, 8, 9, 3.0), (7, 5, 1, 3.0)])
def test_generic_widths_vs_oracle(oracle_c, F, K, L, r3):
    s = S.quartz((3, 3, 3))
    prm = G.ToyPotentialParams.init(17 + F, F, K, L, 5.0, r3)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, F, K, L, 5.0, r3)
    out = run(s, prm)
    sc = max(1.0, np.sqrt(F / 16.0)) * max(1.0, L / 3.0)
    assert np.abs(out.per_atom - ref["per_atom"]).max() <= TOL_EA * sc
    assert abs(out.energy - ref["energy"]) / s.size() <= TOL_E * sc
    fmax = np.abs(ref["forces"]).max()
    assert np.abs(out.forces - ref["forces"]).max() <= min(TOL_F, max(TOL_FREL * fmax, 1e-6)) * sc
    assert np.abs(out.stress - ref["stress"]).max() <= TOL_S * sc


@pytest.mark.parametrize("F,K,r3", [(32, 8, 0.0), (12, 6, 0.0), (64, 8, 3.0)])
def test_generic_partition_invariance(F, K, r3):
    s = S.quartz((3, 3, 6))
    prm = G.ToyPotentialParams.init(5, F, K, 2, 5.0, r3)
    a = run(s, prm, 1)
    for p in (2, 3):
        b = run(s, prm, p)
        np.testing.assert_array_equal(a.per_atom, b.per_atom)
        np.testing.assert_array_equal(a.forces, b.forces)
        assert a.energy == b.energy
        np.testing.assert_array_equal(a.stress, b.stress)


def test_generic_width_md_and_errors():
    s = S.quartz((2, 2, 2))
    prm = G.ToyPotentialParams.init(3, 24, 6, 2, 5.0, 0.0)
    res = G.run_md(s, prm, G.MDOptions(dt=0.5, steps=5, seed=1, allow_narrow=True))
    e = [r.total for r in res.records]
    assert max(abs(x - e[0]) for x in e) / s.size() < 1e-4
    d = G.Distributed.create_distributed(s, 5.0, 3.0, 1, 1, True)
    with pytest.raises(G.Error, match="feature_width <= 128"):
        G.forward_distributed(d, G.ToyPotentialParams.init(3, 200, 6, 1, 5.0, 0.0))


def test_generic_liquid_c4_like(oracle_c):
    """C4-like liquid with three-body terms at F = 64 (SURVEY §8d variant)."""
    s = S.liquid(1500)
    prm = G.ToyPotentialParams.init(9, 64, 8, 3, 5.0, 3.0)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, 64, 8, 3, 5.0, 3.0)
    out = run(s, prm)
    assert abs(out.energy - ref["energy"]) / s.size() <= 4e-6
    fmax = np.abs(ref["forces"]).max()
    assert np.abs(out.forces - ref["forces"]).max() <= max(4e-4, 4e-5 * fmax)
    assert np.abs(out.stress - ref["stress"]).max() <= 4e-6
    np.testing.assert_array_equal(run(s, prm, 4).forces, out.forces)


@pytest.mark.parametrize("r3", [None, 3.0])
def test_generic_rank_group_equals_single_handle(r3):
    """One rank per GPU (in-process group on one GPU) at F = 32: per-atom
    energies and forces bitwise those of the single-handle partitioned run."""
    from tests.test_gpu_multirank import run_group
    s = S.quartz((3, 3, 6))
    prm = G.ToyPotentialParams.init(21, 32, 6, 2, 5.0, r3 or 0.0)
    ref = run(s, prm, 3)
    seen = np.zeros(s.size(), bool)
    for d, out, ids in run_group(s, prm, 3, r3=r3):
        assert not seen[ids].any()
        seen[ids] = True
        np.testing.assert_array_equal(out.per_atom[ids], ref.per_atom[ids])
        np.testing.assert_array_equal(out.forces[ids], ref.forces[ids])
        assert abs(out.energy - ref.energy) <= 1e-9 * abs(ref.energy)
        np.testing.assert_allclose(out.stress, ref.stress, atol=1e-12, rtol=1e-9)
    assert seen.all()


@pytest.mark.parametrize("variant", ["sm8", "ff", "ff16", "tc"])
def test_wide_backward_families_agree(monkeypatch, oracle_c, variant):
    """F = 64 backward edge pass: the default packed-FP32 kernel (partials in
    shared memory) against its other forms (8 rows in flight; register
    partials with a transposed butterfly over 32 / 16-edge chunks; G = X P on
    tcgen05, 3xTF32 in TMEM); every form is checked against the
    oracle and keep exact Newton's third law (test_gpu_physics bound)."""
    s = S.liquid(1500)
    prm = G.ToyPotentialParams.init(9, 64, 8, 2, 5.0, 3.0)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, 64, 8, 2, 5.0, 3.0)
    for k in ("GMD_WIDE_BWD", "GMD_WIDE_TC"):
        monkeypatch.delenv(k, raising=False)
    a = run(s, prm)
    monkeypatch.setenv("GMD_WIDE_BWD", variant)
    b = run(s, prm, 2)
    assert a.energy == b.energy  # the forward is shared
    fmax = np.abs(ref["forces"]).max()
    for out in (a, b):
        assert np.abs(out.forces - ref["forces"]).max() <= max(4e-4, 4e-5 * fmax)
        assert np.abs(out.stress - ref["stress"]).max() <= 4e-6
        assert np.abs(out.forces.sum(axis=0)).max() <= 1e-12 * fmax * s.size()
    np.testing.assert_allclose(b.forces, a.forces, rtol=0, atol=2e-5 * fmax)
