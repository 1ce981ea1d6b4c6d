"""GPU partitions, halo sets and line graphs: bit-exact vs the oracle
(proj/tests/test_partitioner.cpp, test_linegraph.cpp, acceptance.cpp
criteria 2-4)."""
import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

pytestmark = pytest.mark.gpu


def build(s, rc, p, r3=None, allow_narrow=True):
    return G.Distributed.create_distributed(s, rc, r3, p, 1, allow_narrow)


def assert_parts_equal(d, o, p, bonds=False):
    ap = d.atom_parts()
    axis, b = o.rule()
    assert ap.rule.axis == axis
    np.testing.assert_array_equal(ap.rule.boundaries, b)
    np.testing.assert_array_equal(ap.owner, o.owner())
    for i in range(p):
        ol = o.layout(i)
        L = ap.parts[i].layout
        np.testing.assert_array_equal(L.node_array, ol["node_array"])
        np.testing.assert_array_equal(L.markers, ol["markers"])
        np.testing.assert_array_equal(L.duplicates.reshape(-1, 2), ol["duplicates"].reshape(-1, 2))
        oe = o.owned_edges(i)
        np.testing.assert_array_equal(ap.parts[i].owned_edges, oe["owned_edges"])
        np.testing.assert_array_equal(ap.parts[i].local_src, oe["local_src"])
        np.testing.assert_array_equal(ap.parts[i].local_dst, oe["local_dst"])
        np.testing.assert_array_equal(ap.parts[i].border_edge_list, oe["border_edge_list"])
    if bonds:
        lp = d.line_parts()
        ob = o.bonds()
        np.testing.assert_array_equal(lp.bonds.edge_of_bond, ob["edge_of_bond"])
        np.testing.assert_array_equal(lp.bond_owner, ob["bond_owner"])
        for i in range(p):
            ol = o.layout(i, bonds=True)
            L = lp.parts[i].layout
            np.testing.assert_array_equal(L.node_array, ol["node_array"])
            np.testing.assert_array_equal(L.markers, ol["markers"])
            np.testing.assert_array_equal(L.duplicates.reshape(-1, 2), ol["duplicates"].reshape(-1, 2))
            np.testing.assert_array_equal(lp.parts[i].line_edges.reshape(-1, 2), o.line_edges(i).reshape(-1, 2))


def test_chain_hand_trace(oracle_c):
    s = S.chain4()
    d = build(s, 1.5, 2)
    ap = d.atom_parts()
    assert d.graph().num_edges() == 6
    assert list(ap.buckets.pure[0]) == [0] and list(ap.buckets.pure[1]) == [3]
    assert list(ap.buckets.to[0][1]) == [1] and list(ap.buckets.to[1][0]) == [2]
    assert list(ap.parts[0].layout.node_array) == [0, 1, 2]
    l0 = ap.parts[0].layout
    assert (l0.pure_span().begin, l0.pure_span().end) == (0, 1)
    assert (l0.to_span(1).begin, l0.to_span(1).end) == (1, 2)
    assert (l0.from_span(1).begin, l0.from_span(1).end) == (2, 3)
    assert l0.owned_end() == 2
    assert len(ap.parts[0].owned_edges) == 3 and len(ap.parts[1].owned_edges) == 3
    assert len(ap.parts[0].border_edge_list) == 1
    assert_parts_equal(d, oracle_c.create(*S.as_args(s), 1.5, p=2, allow_narrow=True), 2)


def test_p1_identity():
    s = S.random_system(30, (7, 7, 7), 5)
    d = build(s, 2.5, 1, allow_narrow=False)
    ap = d.atom_parts()
    assert len(ap.buckets.pure[0]) == 30
    assert ap.parts[0].layout.size() == 30 and ap.parts[0].layout.owned_end() == 30
    np.testing.assert_array_equal(ap.parts[0].owned_edges, np.arange(d.graph().num_edges()))


def test_quantile_balance():
    s = S.random_system(1000, (10, 10, 40), 3)
    d = build(s, 2.0, 4)
    counts = np.bincount(d.atom_parts().owner, minlength=4)
    assert np.all(counts >= 249) and np.all(counts <= 251)
    assert d.atom_parts().rule.axis == 2


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_quartz_partitions(oracle_c, p):
    s = S.quartz((3, 2, 2), 0.05, 6)
    assert_parts_equal(build(s, 4.0, p), oracle_c.create(*S.as_args(s), 4.0, p=p, allow_narrow=True), p)


@pytest.mark.parametrize("seed", range(0, 100, 7))
def test_acceptance_c3_generator(oracle_c, seed):
    # acceptance.cpp:179-220 systems, p in {2,3,4}, plus line graph with r3 2.4
    s = S.random_gas(30 + seed * 14, seed)
    p = 2 + seed % 3
    d = build(s, 3.2, p, r3=2.4)
    o = oracle_c.create(*S.as_args(s), 3.2, r3=2.4, p=p, allow_narrow=True)
    assert_parts_equal(d, o, p, bonds=True)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_c1_partitions_and_linegraph(oracle_c, p):
    s = S.quartz((5, 5, 5))
    d = build(s, 5.0, p, r3=3.0)
    o = oracle_c.create(*S.as_args(s), 5.0, r3=3.0, p=p, allow_narrow=True)
    assert_parts_equal(d, o, p, bonds=True)


def test_zero_redundancy_and_union():
    s = S.random_gas(400, 4)
    d = build(s, 3.4, 4, r3=2.6)
    ap = d.atom_parts()
    allo = np.sort(np.concatenate([pt.owned_edges for pt in ap.parts]))
    np.testing.assert_array_equal(allo, np.arange(d.graph().num_edges()))
    lp = d.line_parts()
    drawn = np.concatenate([lp.bonds.edge_of_bond[pt.layout.node_array[pt.line_edges.reshape(-1, 2)]]
                            for pt in lp.parts])
    order = np.lexsort((drawn[:, 1], drawn[:, 0]))
    drawn = drawn[order]
    assert len(np.unique(drawn, axis=0)) == len(drawn)


def test_narrow_slab_guard():
    s = S.random_system(200, (40, 10, 10), 3)
    with pytest.raises(G.Error, match="partition-width error"):
        build(s, 3.0, 16, allow_narrow=False)
    build(s, 3.0, 16, allow_narrow=True)


def test_partition_errors():
    s = S.random_system(3, (10, 10, 10), 4)
    with pytest.raises(G.Error, match="more partitions than atoms"):
        build(s, 2.0, 5)
    with pytest.raises(G.Error, match="limited to 64"):
        build(S.random_system(100, (10, 10, 10), 4), 2.0, 65)
    with pytest.raises(G.Error, match="cannot exceed the atom graph cutoff"):
        build(S.random_system(20, (8, 8, 8), 2), 3.0, 1, r3=3.5)
