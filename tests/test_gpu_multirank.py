"""One-rank-per-GPU path exercised as an in-process rank group on
one GPU: W handles, each building only its slab's rows and exchanging halo
rows every layer.  Per-atom energies and forces must equal the single-handle
partitioned result bit for bit (same rows, exact halo copies); energy and
stress up to the order of the cross-rank sum."""
import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S
from tests.conftest import use_kernels

pytestmark = pytest.mark.gpu


def run_group(s, prm, W, r3=None):
    hs = G.local_group(W)

    def rank(r):
        def go():
            d = G.Distributed.create_distributed(s, prm.r_atom, r3, W, 1, True, handle=hs[r])
            out = G.forward_distributed(d, prm)
            return d, out, G.owned_ids(d)
        return go

    return G.run_ranks([rank(r) for r in range(W)])


@pytest.mark.parametrize("kern", ["ffma2", "ffma", "tcgen05"])
@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("which", ["quartz", "gas"])
def test_rank_group_equals_single_handle(W, which, kern, monkeypatch):
    use_kernels(monkeypatch, kern)
    s = S.quartz((4, 4, 4)) if which == "quartz" else S.random_gas(600, 5)
    prm = G.ToyPotentialParams.init(11, 16, 8, 3, 4.0)
    ref_d = G.Distributed.create_distributed(s, 4.0, None, W, 1, True)
    ref = G.forward_distributed(ref_d, prm)
    res = run_group(s, prm, W)
    seen = np.zeros(s.size(), bool)
    g_ref = ref_d.graph()
    for r, (d, out, ids) in enumerate(res):
        assert not seen[ids].any()
        seen[ids] = True
        np.testing.assert_array_equal(out.per_atom[ids], ref.per_atom[ids])
        np.testing.assert_array_equal(out.forces[ids], ref.forces[ids])
        assert abs(out.energy - ref.energy) <= 1e-9 * abs(ref.energy)
        np.testing.assert_allclose(out.stress, ref.stress, atol=1e-12, rtol=1e-9)
        # this rank's rows are exactly the reference rows of its atoms
        g = d.graph()
        mine = np.isin(g_ref.dst, ids)
        np.testing.assert_array_equal(g.src, g_ref.src[mine])
        np.testing.assert_array_equal(g.image_offset, g_ref.image_offset[mine])
        # its layout / halo sets are the reference's partition r
        o = ref_d.atom_parts().parts[r].layout
        L = d.atom_parts().parts[r].layout
        np.testing.assert_array_equal(L.node_array, o.node_array)
        np.testing.assert_array_equal(L.markers, o.markers)
    assert seen.all()


def test_rank_group_rejects_mismatch():
    hs = G.local_group(2)
    s = S.quartz((3, 3, 3))

    def bad(r):
        return lambda: G.Distributed.create_distributed(s, 4.0, None, 3, 1, True, handle=hs[r])

    with pytest.raises(G.Error, match="p == world"):
        G.run_ranks([bad(0), bad(1)])


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("kern", ["ffma2", "ffma"])
@pytest.mark.parametrize("which", ["quartz", "liquid"])
def test_rank_group_three_body(W, which, kern, monkeypatch):
    """Three-body graphs one rank per GPU: t' / v_bar rows of reverse bonds whose
    center lives on a peer travel through the bond halo plan; q_bar halo rows
    through the atom plan.  Owned atoms' energies and forces are bitwise equal
    to the single-handle result."""
    use_kernels(monkeypatch, kern)
    s = S.quartz((4, 4, 4)) if which == "quartz" else S.liquid(1200)
    prm = G.ToyPotentialParams.init(7, 16, 8, 3, 5.0, 3.0)
    ref_d = G.Distributed.create_distributed(s, 5.0, 3.0, W, 1, True)
    ref = G.forward_distributed(ref_d, prm)
    res = run_group(s, prm, W, r3=3.0)
    seen = np.zeros(s.size(), bool)
    for d, out, ids in res:
        seen[ids] = True
        np.testing.assert_array_equal(out.per_atom[ids], ref.per_atom[ids])
        np.testing.assert_array_equal(out.forces[ids], ref.forces[ids])
        assert abs(out.energy - ref.energy) <= 1e-9 * abs(ref.energy)
        np.testing.assert_allclose(out.stress, ref.stress, atol=1e-12, rtol=1e-9)
    assert seen.all()


@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("F,K", [(16, 8), (24, 6), (64, 8)])
@pytest.mark.parametrize("r3", [None, 3.0])
@pytest.mark.parametrize("overlap", ["1", "0"])
def test_rank_group_interior_overlap(W, F, K, r3, overlap, monkeypatch):
    """Slabs thick enough to have interior atoms (no in-edge from a peer):
    those compute while the halo is in flight, the border atoms after it
    landed, in two launches per layer.  Per-atom energies and forces stay
    bitwise equal to the single handle, with and without the split."""
    monkeypatch.setenv("GMD_OVERLAP", overlap)
    s = S.quartz((8, 4, 4))
    prm = G.ToyPotentialParams.init(5, F, K, 3, 5.0, r3 or 0.0)
    ref = G.forward_distributed(G.Distributed.create_distributed(s, 5.0, r3, W, 1, True), prm)
    res = run_group(s, prm, W, r3=r3)
    seen = np.zeros(s.size(), bool)
    for d, out, ids in res:
        seen[ids] = True
        assert 0 < G.num_interior(d) < len(ids)
        np.testing.assert_array_equal(out.per_atom[ids], ref.per_atom[ids])
        np.testing.assert_array_equal(out.forces[ids], ref.forces[ids])
        assert abs(out.energy - ref.energy) <= 1e-9 * abs(ref.energy)
        np.testing.assert_allclose(out.stress, ref.stress, atol=1e-12, rtol=1e-9)
    assert seen.all()
