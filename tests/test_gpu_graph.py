"""GPU neighbour-list parity: bit-exact (src, dst, image) sets and canonical
order vs the fp64 oracle (proj/tests/test_neighborlist.cpp, acceptance.cpp
criterion 5)."""
import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

pytestmark = pytest.mark.gpu


def gpu_graph(sys_, rc):
    return G.build_neighbor_list(sys_, rc)


def assert_same_graph(g, o):
    # canonical order is part of the contract: compare arrays position by position
    assert len(g.src) == len(o["src"])
    np.testing.assert_array_equal(g.src, o["src"])
    np.testing.assert_array_equal(g.dst, o["dst"])
    np.testing.assert_array_equal(g.image_offset, o["off"])
    # fp64 export is recomputed exactly: bitwise equal distances and vectors
    np.testing.assert_array_equal(g.distance, o["dist"])
    np.testing.assert_array_equal(g.vector, o["vec"])


def check_invariants(g):
    assert np.all(g.distance <= g.cutoff)
    assert np.all(g.distance > 0)
    keys = S.edge_keys(g.src, g.dst, g.image_offset)
    rev = S.edge_keys(g.dst, g.src, -g.image_offset)
    np.testing.assert_array_equal(keys, rev)  # reversal closure
    assert np.all(np.diff(g.dst) >= 0)


def test_two_atoms(oracle_c):
    s = S.random_system(0, (100, 100, 100), 0)
    s = G.AtomicSystem(np.array([[50.0, 50, 50], [51.0, 50, 50]]), s.lattice, np.array([1, 1], np.int32))
    g = gpu_graph(s, 2.0)
    assert g.num_edges() == 2
    check_invariants(g)


def test_self_image_cell(oracle_c):
    s = G.AtomicSystem(np.array([[0.3, 0.7, 1.1]]), np.eye(3) * 2.0, np.array([2], np.int32))
    g = gpu_graph(s, 2.5)
    o = oracle_c.neighbor_list(*S.as_args(s), 2.5, brute=True)
    assert g.num_edges() == 6
    assert_same_graph(g, o)


@pytest.mark.parametrize("reps", [(3, 3, 3), (5, 5, 5)])
def test_quartz_vs_oracle(oracle_c, reps):
    s = S.quartz(reps)
    g = gpu_graph(s, 5.0)
    o = oracle_c.neighbor_list(*S.as_args(s), 5.0)
    assert_same_graph(g, o)
    check_invariants(g)


@pytest.mark.parametrize("seed", range(25))
def test_randomized_systems(oracle_c, seed):
    # proj/tests/test_neighborlist.cpp:82-96
    box = 4.0 + (seed % 7)
    n = 5 + seed * 7 % 60
    s = S.random_triclinic(n, box, seed) if seed % 3 == 0 else S.random_system(n, (box, box + 1.0, box - 0.5), seed)
    rc = 2.0 + 0.37 * (seed % 5)
    g = gpu_graph(s, rc)
    assert_same_graph(g, oracle_c.neighbor_list(*S.as_args(s), rc, brute=True))


@pytest.mark.parametrize("seed", range(0, 100, 3))
def test_acceptance_c5_generator(oracle_c, seed):
    # acceptance.cpp:255-279 (includes the 2.1-2.4 A self-image cells)
    if seed % 10 == 0:
        s = S.random_system(1 + seed % 3, (2.1, 2.4, 2.2), seed)
        rc = 2.6
    else:
        s = S.random_gas(10 + seed * 9, seed)
        rc = 2.4 + 0.31 * (seed % 6)
    g = gpu_graph(s, rc)
    assert_same_graph(g, oracle_c.neighbor_list(*S.as_args(s), rc))


def test_non_periodic_padding(oracle_c):
    s = S.random_system(40, (9.0, 8.0, 7.0), 11)
    s.pbc = (True, False, False)
    g = gpu_graph(s, 3.0)
    assert_same_graph(g, oracle_c.neighbor_list(*S.as_args(s), 3.0))


def test_liquid_dense(oracle_c):
    s = S.liquid(3000)
    g = gpu_graph(s, 5.0)
    assert_same_graph(g, oracle_c.neighbor_list(*S.as_args(s), 5.0))


def test_errors():
    s = S.random_system(3, (5, 5, 5), 0)
    with pytest.raises(G.Error):
        gpu_graph(s, 0.0)
    with pytest.raises(G.Error):
        gpu_graph(s, -1.0)
    with pytest.raises(G.Error):
        gpu_graph(G.AtomicSystem(np.zeros((0, 3)), np.eye(3) * 5, np.zeros(0, np.int32)), 2.0)


def test_deterministic_rebuild():
    s = S.random_system(300, (12, 10, 14), 9)
    a = gpu_graph(s, 3.5)
    b = gpu_graph(s, 3.5)
    for x, y in [(a.src, b.src), (a.image_offset, b.image_offset), (a.vector, b.vector)]:
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("rc", [5.0, 3.7])
def test_cutoff_boundary_and_coincident_pairs(oracle_c, rc):
    """Pairs straddling the cutoff within the fp32 fast-accept margin and the
    reference's 1.000001 prefilter band, plus coincident atoms (d2 == 0):
    these take the exact fp64 path and must match the oracle bit for bit."""
    fac = [1 - 1e-4, 1 - 1e-6, 1 - 1e-8, 1.0, 1 + 1e-9, 1 + 1e-7, 1 + 4e-7, 1 + 9e-7,
           1 + 2e-6, 1 + 1e-4]
    pos = []
    for i, f in enumerate(fac):  # pairs along x, far apart from each other
        base = np.array([10.0 + 12.0 * (i % 5), 10.0 + 12.0 * (i // 5), 20.0])
        pos += [base, base + [rc * f, 0.0, 0.0]]
    pos += [[40.0, 40.0, 40.0], [40.0, 40.0, 40.0]]  # coincident pair
    d = rc / np.sqrt(3.0)
    pos += [[50.0, 50.0, 50.0], [50.0 + d, 50.0 + d, 50.0 + d]]  # |v| == rc in fp64 rounding
    s = G.AtomicSystem(np.array(pos), np.diag([80.0, 80.0, 80.0]), np.ones(len(pos), np.int32))
    g = gpu_graph(s, rc)
    o = oracle_c.neighbor_list(*S.as_args(s), rc)
    assert_same_graph(g, o)
    assert len(g.src) > 0


@pytest.mark.parametrize("shift", [3, 1 << 19, (1 << 20) + 5, 5_000_000])
def test_far_images(oracle_c, shift):
    """Atoms many lattice vectors outside the cell (a common shift plus a few
    cells between atoms): large cell_of values, small relative images; the
    graph matches the oracle bit for bit."""
    s = S.random_system(60, (9.0, 8.0, 10.0), 21)
    pos = s.positions + shift * s.lattice[0] - (shift // 2) * s.lattice[2]
    pos[::3] += 3 * s.lattice[1]  # offsets between atoms stay in the packed image range
    pos[1::7] -= 2 * s.lattice[0]
    s = G.AtomicSystem(pos, s.lattice, s.species)
    assert_same_graph(gpu_graph(s, 3.2), oracle_c.neighbor_list(*S.as_args(s), 3.2))


@pytest.mark.parametrize("shift", [0, 1 << 12, 1 << 16, 5_000_000])
def test_far_pairs_at_cutoff(oracle_c, shift):
    """Pairs at rc (1 +- 1e-11 .. 1e-8) placed `shift` cells out: there the
    wrapped and raw fp64 vectors disagree by up to ~1e-8 A, so the fp32 fast
    accept must switch itself off (k_wrap's max |coordinate| vs the host's
    gate) and every survivor take the reference's raw-position test."""
    rc = 5.0
    rng = np.random.default_rng(shift + 1)
    fac = 1.0 + np.concatenate([-np.logspace(-11, -8, 12), np.logspace(-11, -8, 12)])
    lat = np.diag([80.0, 80.0, 80.0])
    pos = []
    for i, f in enumerate(fac):
        base = np.array([6.0 + 13.0 * (i % 5), 6.0 + 13.0 * ((i // 5) % 5), 6.0 + 13.0 * (i // 25)])
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        pos += [base, base + rc * f * u]
    pos = np.array(pos) + shift * lat[0] - (shift // 3) * lat[2]
    s = G.AtomicSystem(pos, lat, np.ones(len(pos), np.int32))
    assert_same_graph(gpu_graph(s, rc), oracle_c.neighbor_list(*S.as_args(s), rc))


def test_slab_capacity_retry_and_growth(oracle_c):
    """The search writes each destination's keys into a fixed-capacity slab
    row sized from a density estimate (first build) or the previous build's
    maximum degree; a row that overflows is detected and the search reruns
    with the exact capacity (gmd_api.cu build_impl).  A dense blob in a dilute
    gas overflows the first estimate; a denser blob on the same handle then
    overflows the carried capacity.  Both graphs are bit-exact."""
    rng = np.random.default_rng(3)
    box = 60.0
    gas = rng.uniform(0, box, (1500, 3))

    def with_blob(k, radius):
        blob = 30.0 + rng.normal(0, radius, (k, 3))
        pos = np.concatenate([gas, blob])
        return G.AtomicSystem(pos, np.eye(3) * box, np.full(len(pos), 8, np.int32))

    h = G._Handle(0)
    for s in (with_blob(150, 1.2), with_blob(400, 1.0)):
        d = G.Distributed.create_distributed(s, 4.0, None, 1, 1, True, handle=h)
        g = d.graph()
        o = oracle_c.neighbor_list(*S.as_args(s), 4.0)
        assert_same_graph(g, o)
        deg = np.bincount(g.dst, minlength=s.size())
        assert deg.max() > 4 * deg.mean()  # well above the density estimate
