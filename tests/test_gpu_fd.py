"""Finite-difference checks of the hand-written backward on the GPU path
(the reference's test_potential.cpp:67-102 "forces match finite differences"
/ "stress matches strain finite differences", and acceptance criterion 6).

The GPU energy is a fixed-order fp64 sum of fp32-computed per-atom terms, so
a central difference carries rounding noise of ~1e-6 eV / (2 eps) on top of
the O(eps^2) truncation error: the reference's fp64 bound (1e-6 eV/A) cannot
hold.  Measured on the B200: ~1e-5 eV of energy noise over 72 atoms, i.e.
2e-3 eV/A at eps = 2e-3 A and ~1e-3 at 4e-3 (truncation ~1e-4); the bounds
(3e-3 + 3e-4 max|F|) sit at that noise and three orders of magnitude below
the force scale, so a wrong derivative (a missing term, a sign, a factor 2)
fails them."""
import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

pytestmark = pytest.mark.gpu


def _check_forces(s, prm, eps, tol, atoms):
    out = G.forward_serial(s, prm)
    sub = G.AtomicSystem(s.positions, s.lattice, s.species, s.pbc)
    fd = np.zeros((len(atoms), 3))
    for n, i in enumerate(atoms):  # finite_difference_forces restricted to a subset
        for k in range(3):
            x0 = s.positions[i, k]
            sub.positions[i, k] = x0 + eps
            ep = G.forward_serial(sub, prm).energy
            sub.positions[i, k] = x0 - eps
            em = G.forward_serial(sub, prm).energy
            sub.positions[i, k] = x0
            fd[n, k] = -(ep - em) / (2 * eps)
    err = np.abs(out.forces[atoms] - fd).max()
    fmax = np.abs(out.forces[atoms]).max()
    print(f"max|F| {fmax:.3e}  max|F - FD| {err:.3e}")
    assert fmax > 0.1
    assert err <= tol + 3e-4 * fmax


@pytest.mark.parametrize("F,K,L,r3", [(16, 8, 2, 0.0), (16, 8, 2, 2.8), (64, 8, 2, 2.8), (24, 6, 2, 2.8)])
def test_forces_match_finite_differences(F, K, L, r3):
    """Quartz 2x2x2 (atom graph) and a random 24-atom cell with three-body
    terms, as the reference's subcases; also the F = 64 and width-generic
    kernels."""
    prm = G.ToyPotentialParams.init(3 if r3 == 0 else 4, F, K, L, 5.0 if r3 == 0 else 4.0, r3)
    if r3 == 0:
        s = S.quartz((2, 2, 2), 0.05, 1)
        atoms = list(range(0, 72, 7))
    else:
        s = S.random_system(24, (8, 7, 9), 5)
        atoms = list(range(24))
    _check_forces(s, prm, 4e-3, 3e-3, atoms)


def test_full_finite_difference_forces_api():
    """G.finite_difference_forces (the reference's free function) on a small cell."""
    prm = G.ToyPotentialParams.init(4, 16, 8, 2, 4.0, 2.8)
    s = S.random_system(24, (8, 7, 9), 5)
    out = G.forward_serial(s, prm)
    fd = G.finite_difference_forces(s, prm, 4e-3)
    assert np.abs(out.forces - fd).max() <= 3e-3 + 3e-4 * np.abs(out.forces).max()
    with pytest.raises(G.Error, match="finite-difference step"):
        G.finite_difference_forces(s, prm, 1e-1)


@pytest.mark.parametrize("F,r3", [(16, 2.8), (64, 2.8), (16, 0.0)])
def test_stress_matches_strain_finite_differences(F, r3):
    """Quartz 1x1x1 (the reference's case, replicated 2x2x2 here so the cell
    is wider than 2 r_atom on the GPU's bins) under +-eps strain."""
    prm = G.ToyPotentialParams.init(6, F, 8, 2, 4.0, r3)
    s = S.quartz((2, 2, 2), 0.04, 7)
    out = G.forward_serial(s, prm)
    fd = G.finite_difference_stress(s, prm, 5e-4)
    err = np.abs(out.stress - fd).max()
    print(f"max|S| {np.abs(out.stress).max():.3e}  max|S - FD| {err:.3e}")
    assert np.abs(out.stress).max() > 1e-3
    assert err <= 2e-5
    assert np.abs(out.stress - out.stress.T).max() <= 1e-10
