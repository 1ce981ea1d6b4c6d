"""Model widths other than the tuned F = 16, K = 8 (the reference accepts any
ToyPotentialParams widths, potential.hpp:15-41): the width-generic kernels
(gmd_generic.cu) against the fp64 oracle, and partition invariance.

Tolerances as tests/test_gpu_model.py (fp32 compute against fp64): per-atom
energy 2e-5 eV, total energy 2e-6 eV/atom, forces 2e-4 eV/A, stress 2e-6 eV/A^3
-- scaled by sqrt(F / 16) for wider features (longer fp32 sums)."""
import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

pytestmark = pytest.mark.gpu


def run(s, prm, p=1):
    d = G.Distributed.create_distributed(s, prm.r_atom, None, p, 1, True)
    return G.forward_distributed(d, prm)


@pytest.mark.parametrize("F,K,L", [(8, 4, 2), (32, 8, 2), (64, 12, 3), (16, 8, 9), (5, 3, 1), (128, 32, 1)])
def test_generic_widths_vs_oracle(oracle_c, F, K, L):
    s = S.quartz((3, 3, 3))
    prm = G.ToyPotentialParams.init(17 + F, F, K, L, 5.0, 0.0)
    ref = oracle_c.forward_serial(*S.as_args(s), prm.blob, F, K, L, 5.0, 0.0)
    out = run(s, prm)
    sc = max(1.0, np.sqrt(F / 16.0)) * max(1.0, L / 3.0)
    assert np.abs(out.per_atom - ref["per_atom"]).max() <= 2e-5 * sc
    assert abs(out.energy - ref["energy"]) / s.size() <= 2e-6 * sc
    fmax = np.abs(ref["forces"]).max()
    assert np.abs(out.forces - ref["forces"]).max() <= max(2e-4, 2e-5 * fmax) * sc
    assert np.abs(out.stress - ref["stress"]).max() <= 2e-6 * sc


@pytest.mark.parametrize("F,K", [(32, 8), (12, 6)])
def test_generic_partition_invariance(F, K):
    s = S.quartz((3, 3, 6))
    prm = G.ToyPotentialParams.init(5, F, K, 2, 5.0, 0.0)
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
    with pytest.raises(G.Error, match="three-body parameters need"):
        G.forward_distributed(d, G.ToyPotentialParams.init(3, 24, 6, 2, 5.0, 3.0))
    with pytest.raises(G.Error, match="feature_width <= 128"):
        G.forward_distributed(d, G.ToyPotentialParams.init(3, 200, 6, 1, 5.0, 0.0))
