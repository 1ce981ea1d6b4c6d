"""GPU energy / forces / stress vs the fp64 oracle (proj/tests/test_potential.cpp,
acceptance.cpp criterion 1), and partition invariance of the GPU path.

Tolerances (fp32 compute against the fp64 oracle, stated per quantity;
calibrated in tests/test_gpu_scale.py, see tests/conftest.py):
  per-atom energy  |dE_i|          <= 2e-5 eV
  total energy     |dE| / N        <= 2e-6 eV/atom
  forces           max |dF|        <= 2e-4 eV/A   (and <= 2e-5 relative to max |F|)
  stress           max |dS|        <= 2e-6 eV/A^3
"""
import os

import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S
from tests.conftest import KERNELS, TOL_E, TOL_EA, TOL_F, TOL_FREL, TOL_S, use_kernels

pytestmark = pytest.mark.gpu



@pytest.fixture(params=list(KERNELS), autouse=True)
def kernels(request, monkeypatch):
    """Every test runs with every kernel family (environment switches read per call)."""
    use_kernels(monkeypatch, request.param)
    return request.param


def run_gpu(s, params, p=1, r3=None, allow_narrow=True):
    d = G.Distributed.create_distributed(s, params.r_atom, r3, p, 1, allow_narrow)
    return G.forward_distributed(d, params)


def compare(out, ref, n):
    dea = np.abs(out.per_atom - ref["per_atom"]).max()
    de = abs(out.energy - ref["energy"]) / n
    df = np.abs(out.forces - ref["forces"]).max()
    fmax = np.abs(ref["forces"]).max()
    ds = np.abs(out.stress - ref["stress"]).max()
    assert dea <= TOL_EA, f"per-atom energy error {dea:.3e}"
    assert de <= TOL_E, f"energy error per atom {de:.3e}"
    assert df <= TOL_F and df <= max(TOL_FREL * fmax, 1e-6), f"force error {df:.3e} (max |F| {fmax:.3e})"
    assert ds <= TOL_S, f"stress error {ds:.3e}"
    return dea, de, df, ds


def params_for(seed, L, rc, r3=0.0):
    return G.ToyPotentialParams.init(seed, 16, 8, L, rc, r3)


def test_c1_quartz_two_body(oracle_c):
    s = S.quartz((5, 5, 5))
    prm = params_for(12345, 2, 5.0)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, 16, 8, 2, 5.0, 0.0)
    compare(run_gpu(s, prm), ref, s.size())


def test_c2_partitioned_equals_unpartitioned():
    s = S.quartz((5, 5, 5))
    prm = params_for(12345, 2, 5.0)
    a = run_gpu(s, prm, p=1)
    for p in (2, 3, 4, 8):
        b = run_gpu(s, prm, p=p)
        # row-form kernels: identical arithmetic for any partition count
        np.testing.assert_array_equal(a.per_atom, b.per_atom)
        np.testing.assert_array_equal(a.forces, b.forces)
        assert a.energy == b.energy
        np.testing.assert_array_equal(a.stress, b.stress)


@pytest.mark.parametrize("r3", [0.0, 2.4])
@pytest.mark.parametrize("seed", [0, 1, 2, 5, 13])
def test_random_gas(oracle_c, seed, r3):
    s = S.random_gas(10 + seed * 22, seed)
    prm = params_for(s.size(), 2, 4.0, r3)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, 16, 8, 2, 4.0, r3)
    for p in (1, 2, 3):
        if p > s.size():
            continue
        compare(run_gpu(s, prm, p=p, r3=r3 if r3 > 0 else None), ref, s.size())


@pytest.mark.parametrize("L", [1, 3])
def test_three_body_quartz(oracle_c, L):
    s = S.quartz((3, 3, 3))
    prm = params_for(7, L, 5.0, 3.0)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, 16, 8, L, 5.0, 3.0)
    for p in (1, 2, 4):
        compare(run_gpu(s, prm, p=p, r3=3.0), ref, s.size())


def test_three_body_liquid(oracle_c):
    s = S.liquid(1500)
    prm = params_for(3, 3, 5.0, 3.0)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, 16, 8, 3, 5.0, 3.0)
    compare(run_gpu(s, prm, p=1, r3=3.0), ref, s.size())
    compare(run_gpu(s, prm, p=4, r3=3.0), ref, s.size())


def test_isolated_atom_closed_form():
    # proj/tests/test_potential.cpp:31-51
    s = G.AtomicSystem(np.array([[25.0, 25, 25]]), np.eye(3) * 50, np.array([26], np.int32))
    prm = params_for(5, 2, 4.0)
    out = run_gpu(s, prm)
    F = 16
    h = prm.embedding[26 * F:27 * F].copy()
    for l in range(2):
        h = h + np.tanh(prm.layer_b[l * F:(l + 1) * F])
    assert abs(out.energy - float(prm.readout @ h)) <= 1e-5
    assert np.all(out.forces == 0.0)
    assert np.all(out.stress == 0.0)


def test_dimer_symmetry():
    s = G.AtomicSystem(np.array([[14.0, 15, 15], [16.2, 15, 15]]), np.eye(3) * 30, np.array([8, 8], np.int32))
    out = run_gpu(s, params_for(2, 2, 4.0))
    np.testing.assert_allclose(out.forces[0], -out.forces[1], atol=1e-6)
    assert abs(out.forces[0, 1]) < 1e-6 and abs(out.forces[0, 2]) < 1e-6


def test_translation_sum_forces_zero():
    s = S.random_system(80, (9, 9, 9), 4)
    out = run_gpu(s, params_for(3, 2, 4.0, 2.4), r3=2.4)
    assert np.abs(out.forces.sum(axis=0)).max() < 1e-4


def test_cutoff_mismatch_error():
    s = S.quartz((2, 2, 2))
    d = G.Distributed.create_distributed(s, 4.0, None, 1, 1)
    with pytest.raises(G.Error, match="cutoff does not match"):
        G.forward_distributed(d, params_for(1, 2, 5.0))
    with pytest.raises(G.Error, match="require a line graph"):
        G.forward_distributed(d, params_for(1, 2, 4.0, 3.0))


@pytest.mark.parametrize("other", ["tcgen05", "ffma"])
def test_kernel_families_agree(monkeypatch, other):
    """The default packed kernels against the scalar-FFMA and tcgen05 paths."""
    s = S.quartz((4, 4, 4))
    prm = params_for(11, 3, 5.0)
    use_kernels(monkeypatch, "ffma2")
    a = run_gpu(s, prm, p=2)
    use_kernels(monkeypatch, other)
    b = run_gpu(s, prm, p=2)
    if other == "tcgen05":
        assert a.energy == b.energy  # forward is shared
    else:  # same per-feature operations in the same order
        np.testing.assert_array_equal(b.per_atom, a.per_atom)
    np.testing.assert_allclose(b.forces, a.forces, rtol=0, atol=2e-5 * np.abs(a.forces).max())
    np.testing.assert_allclose(b.stress, a.stress, rtol=0, atol=1e-6)


def test_streamed_force_chunks_match_device_output():
    """Host forces in pinned memory: the last edge pass runs in node chunks and
    each chunk's forces are copied out while the next computes; forces and
    per-atom energies are bitwise those of device output, the stress equal up
    to the regrouped fixed-order virial partials."""
    import ctypes as C
    import torch
    s = S.quartz((15, 15, 15))  # 30,375 atoms: large enough for the chunked pass
    prm = params_for(3, 3, 5.0)
    n = s.size()
    L = G.lib()
    h = G._Handle(0)
    h.check(L.gmd_set_params(h.h, 16, 8, 3, 5.0, 0.0, G._p(prm.blob)))
    pbc = np.ones(3, np.uint8)
    h.check(L.gmd_build(h.h, n, G._p(s.positions), G._p(s.species), G._p(s.lattice), G._p(pbc), 5.0,
                        0.0, 0.0, 1, 0, G.GMD_ALLOW_NARROW))
    e1, e2 = C.c_double(), C.c_double()
    st1, st2 = np.zeros(9), np.zeros(9)
    pa_d = torch.empty(n, dtype=torch.float64, device="cuda")
    f_d = torch.empty(3 * n, dtype=torch.float64, device="cuda")
    h.check(L.gmd_forward(h.h, C.byref(e1), C.c_void_p(pa_d.data_ptr()), C.c_void_p(f_d.data_ptr()),
                          G._p(st1), None, G.GMD_OUTPUT_DEVICE))
    pa_h = torch.empty(n, dtype=torch.float64).pin_memory()
    f_h = torch.full((3 * n,), np.nan, dtype=torch.float64).pin_memory()
    h.check(L.gmd_forward(h.h, C.byref(e2), C.c_void_p(pa_h.data_ptr()), C.c_void_p(f_h.data_ptr()),
                          G._p(st2), None, 0))
    np.testing.assert_array_equal(f_h.numpy(), f_d.cpu().numpy())
    np.testing.assert_array_equal(pa_h.numpy(), pa_d.cpu().numpy())
    assert e1.value == e2.value
    np.testing.assert_allclose(st2, st1, rtol=1e-12, atol=1e-18)


@pytest.mark.parametrize("species,F,r3", [((14, 8), 16, 0.0), ((14, 8, 1), 16, 0.0), ((8,), 16, 0.0),
                                          ((14, 8, 1), 16, 3.0), ((14, 8), 64, 3.0), ((14, 8, 1, 6), 64, 3.0)])
def test_layer0_species_forms(oracle_c, species, F, r3):
    """Layer 0 reads h0 = emb[Z]: with <= 2 species present the conv runs in
    the species-sum form and the layer-0 backward takes h0 from the staged
    embedding rows; with more species the same kernels fall back to the
    per-edge form.  Both against the fp64 oracle, one to four species, F =
    16 and 64, with and without the three-body stage; p = 2 bitwise p = 1."""
    s = S.random_system(300, (14.0, 14.0, 14.0), 5, species=species)
    prm = G.ToyPotentialParams.init(17, F, 8, 3, 5.0, r3)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, F, 8, 3, 5.0, r3)
    a = run_gpu(s, prm, r3=r3 if r3 > 0 else None)
    scale = np.sqrt(F / 16)
    dea = np.abs(a.per_atom - ref["per_atom"]).max()
    df = np.abs(a.forces - ref["forces"]).max()
    assert dea <= TOL_EA * scale, dea
    assert df <= TOL_F * scale and df <= max(TOL_FREL * scale * np.abs(ref["forces"]).max(), 1e-6), df
    b = run_gpu(s, prm, p=2, r3=r3 if r3 > 0 else None)
    np.testing.assert_array_equal(b.per_atom, a.per_atom)
    np.testing.assert_array_equal(b.forces, a.forces)
