"""GPU feature API: halo transfer, its adjoint, duplicate sync, distribute /
aggregate (proj/tests/test_engine.cpp), compared with reference semantics."""
import numpy as np
import pytest
import torch

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

pytestmark = pytest.mark.gpu


def build(s, rc, p, r3=None):
    return G.Distributed.create_distributed(s, rc, r3, p, 1, True)


def ref_transfer(d, f, bonds=False):
    """engine.cpp:122-143 on host copies of the blocks."""
    parts = d.line_parts().parts if bonds else d.atom_parts().parts
    blocks = [f.block(i).cpu().numpy().copy() for i in range(d.num_partitions())]
    for i, pi in enumerate(parts):
        for j, pj in enumerate(parts):
            if i == j:
                continue
            to, fr = pj.layout.to_span(i), pi.layout.from_span(j)
            assert to.size() == fr.size()
            blocks[i][fr.begin:fr.end] = blocks[j][to.begin:to.end]
    return blocks


def test_p1_empty_plans_and_identity():
    s = S.random_system(25, (8, 8, 8), 1)
    d = build(s, 3.0, 1)
    L = d.atom_parts().parts[0].layout
    assert L.to_span(0).size() == 0 and L.from_span(0).size() == 0
    feats = 0.5 * np.arange(25 * 4, dtype=np.float64)
    f = d.distribute_node_features(feats, 4)
    np.testing.assert_array_equal(d.aggregate(f), feats)


def test_chain_copy_semantics():
    s = S.chain4()
    d = build(s, 1.5, 2)
    f = d.make_atom_features(1)
    for i in range(2):
        L = d.atom_parts().parts[i].layout
        for r in range(L.owned_end()):
            f.block(i)[r, 0] = float(L.node_array[r])
    d.atom_transfer(f)
    for i in range(2):
        L = d.atom_parts().parts[i].layout
        for r in range(L.size()):
            assert f.block(i)[r, 0].item() == float(L.node_array[r])
    before = f.data.clone()
    d.atom_transfer(f)
    assert torch.equal(before, f.data)  # idempotent


@pytest.mark.parametrize("p", [2, 3, 8])
def test_transfer_matches_reference_semantics(p):
    s = S.quartz((3, 3, 2))
    d = build(s, 4.0, p)
    f = d.make_atom_features(5)
    f.data.copy_(torch.randn_like(f.data))
    want = ref_transfer(d, f)
    d.atom_transfer(f)
    for i in range(p):
        np.testing.assert_array_equal(f.block(i).cpu().numpy(), want[i])


@pytest.mark.parametrize("p", [2, 3, 8])
@pytest.mark.parametrize("bonds", [False, True])
def test_transpose_is_adjoint(p, bonds):
    # <T x, y> = <x, T^T y>  (test_engine.cpp:101-147)
    s = S.quartz((3, 3, 2))
    d = build(s, 4.0, p, r3=3.0)
    mk = d.make_bond_features if bonds else d.make_atom_features
    x = mk(3)
    y = mk(3)
    g = torch.Generator(device="cuda").manual_seed(p)
    x.data.copy_(torch.randn(x.data.shape, generator=g, device="cuda", dtype=torch.float64))
    y.data.copy_(torch.randn(y.data.shape, generator=g, device="cuda", dtype=torch.float64))
    # transfer overwrites FROM spans and the transpose folds duplicates, so x
    # needs zero FROM rows and synced duplicates (test_engine.cpp:101-147)
    parts = d.line_parts().parts if bonds else d.atom_parts().parts
    for i, pt in enumerate(parts):
        x.block(i)[pt.layout.owned_end():] = 0.0
    (d.sync_bond_duplicates if bonds else d.sync_atom_duplicates)(x)
    tx = mk(3)
    tx.data.copy_(x.data)
    (d.bond_transfer if bonds else d.atom_transfer)(tx)
    tty = mk(3)
    tty.data.copy_(y.data)
    (d.bond_transfer_transpose if bonds else d.atom_transfer_transpose)(tty)
    lhs = float((tx.data * y.data).sum())
    rhs = float((x.data * tty.data).sum())
    assert abs(lhs - rhs) <= 1e-9 * max(1.0, abs(lhs))


def test_aggregate_ignores_from_rows():
    s = S.chain4()
    d = build(s, 1.5, 2)
    f = d.make_atom_features(1)
    f.data.fill_(7.0)
    for i in range(2):
        L = d.atom_parts().parts[i].layout
        f.block(i)[L.owned_end():] = -1.0
    np.testing.assert_array_equal(d.aggregate(f), np.full(4, 7.0))


def test_duplicates_sync_and_fold():
    s = S.quartz((5, 5, 5))
    d = build(s, 5.0, 8)
    ap = d.atom_parts()
    ndup = sum(len(pt.layout.duplicates) for pt in ap.parts)
    assert ndup > 0  # narrow slabs at p=8 produce duplicated TO rows (SURVEY: 1,831)
    f = d.make_atom_features(2)
    f.data.copy_(torch.randn_like(f.data))
    d.sync_atom_duplicates(f)
    for i, pt in enumerate(ap.parts):
        b = f.block(i)
        for c, u in pt.layout.duplicates:
            assert torch.equal(b[c], b[u])


def test_corrupt_plan_is_detected():
    s = S.chain4()
    d = build(s, 1.5, 2)
    f = d.make_atom_features(1)
    for i in range(2):
        L = d.atom_parts().parts[i].layout
        f.block(i)[:, 0] = torch.tensor(L.node_array, dtype=torch.float64, device="cuda") + 100 * (i + 1)
    good = ref_transfer(d, f)
    d.corrupt_transfer_plan_for_test()
    d.atom_transfer(f)
    bad = [f.block(i).cpu().numpy() for i in range(2)]
    assert any(not np.array_equal(good[i], bad[i]) for i in range(2))


def test_partitioned_model_matches_feature_api():
    """The model's internal exchange equals the public transfer on canonical rows."""
    s = S.quartz((4, 4, 4))
    d = build(s, 4.0, 4)
    feats = np.random.default_rng(0).standard_normal((s.size(), 4))
    f = d.distribute_node_features(feats.ravel(), 4)
    d.atom_transfer(f)
    for i, pt in enumerate(d.atom_parts().parts):
        np.testing.assert_array_equal(f.block(i).cpu().numpy(), feats[pt.layout.node_array])


def test_corrupt_plan_breaks_forward():
    """The hook also corrupts the forward's atom transfers (engine.cpp:136-137:
    forward_distributed goes through transfer_impl), so the CLI's audit
    negative control fails as the reference's does."""
    s = S.quartz((3, 3, 6))
    prm = G.ToyPotentialParams.init(12345, 16, 8, 2, 5.0, 0.0)
    good = G.forward_distributed(G.Distributed.create_distributed(s, 5.0, None, 2, 1), prm)
    d = G.Distributed.create_distributed(s, 5.0, None, 2, 1)
    d.corrupt_transfer_plan_for_test()
    bad = G.forward_distributed(d, prm)
    assert np.abs(bad.forces - good.forces).max() > 1e-6


def _mean_of_neighbors(d):
    def layer(part, f):  # test_engine.cpp:158-169
        ap = d.atom_parts().parts[part]
        rows = d.atom_rows(part)
        x = f.block(part)[:, 0].cpu().numpy()
        s, c = np.zeros(rows), np.zeros(rows, np.int64)
        np.add.at(s, ap.local_dst, x[ap.local_src])
        np.add.at(c, ap.local_dst, 1)
        lay = ap.layout
        for r in range(lay.owned_end()):
            if lay.local_of(lay.node_array[r]) == r and c[r]:
                f.block(part)[r, 0] = s[r] / c[r]
    return layer


def test_run_layered_and_worker_failure():
    """test_engine.cpp:149-203: mean-of-neighbours on the chain equals the
    serial result for p = 1, 2; identity layers leave rows untouched; a worker
    failure names its partition."""
    def run(p):
        d = build(S.chain4(), 1.5, p)
        f = d.distribute_node_features(np.array([1.0, 2.0, 3.0, 4.0]), 1)
        d.run_layered([_mean_of_neighbors(d)], f)
        return d.aggregate(f)
    serial = run(1)
    np.testing.assert_array_equal(serial, [2.0, 2.0, 3.0, 3.0])
    np.testing.assert_array_equal(run(2), serial)
    d = build(S.chain4(), 1.5, 2)
    f = d.distribute_node_features(np.array([5.0, 6, 7, 8]), 1)
    d.run_layered([lambda i, x: None] * 3, f)
    np.testing.assert_array_equal(d.aggregate(f), [5.0, 6, 7, 8])
    d2 = G.Distributed.create_distributed(S.random_system(40, (10, 8, 8), 11), 3.0, None, 2, 2, True)

    def boom(p):
        if p == 1:
            raise G.Error("boom")
    with pytest.raises(G.Error, match="worker for partition 1 failed: boom"):
        d2.parallel_for_partitions(boom)


def test_edge_features_round_trip():
    d = G.Distributed.create_distributed(S.random_system(40, (10, 8, 8), 11), 3.0, None, 3, 1, True)
    ne = d.num_edges()
    ef = 0.25 * np.arange(ne * 3) - 7.0
    eb = d.distribute_edge_features(ef, 3)
    assert eb.data.shape == (ne, 3)
    ap = d.atom_parts()
    for i in range(3):  # block i = its owned edges, in order
        np.testing.assert_array_equal(eb.block(i).cpu().numpy(), ef.reshape(-1, 3)[ap.parts[i].owned_edges])
    np.testing.assert_array_equal(d.aggregate_edges(eb), ef)
    with pytest.raises(G.Error, match="edge feature shape mismatch"):
        d.distribute_edge_features(np.zeros(5), 3)
    with pytest.raises(G.Error):
        d.atom_transfer(eb)
