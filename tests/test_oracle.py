"""Pin the plain-C oracle restatement (oracle/gmd_oracle.c) against golden
vectors produced by the unmodified reference (tests/golden/gen_golden.py) and,
where oracle/_ref is built, against the live reference.  CPU only."""
import hashlib
import os

import numpy as np
import pytest

from tests import systems as S

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def fixture_args(name):
    s = S.fixture(name)
    return s.positions, s.species, s.lattice


def test_rng_streams(oracle_c):
    np.testing.assert_array_equal(oracle_c.rng_normal(3, 1001), GOLD["rng/normal3"])
    np.testing.assert_array_equal(oracle_c.rng_uniform(7, 999, 0.0, 100.0), GOLD["rng/uniform7"])


def test_supercells(oracle_c):
    p, z, l = fixture_args("quartz")
    for tag, reps, seed in [("q333", (3, 3, 3), 1), ("q555", (5, 5, 5), 1), ("q322", (3, 2, 2), 6), ("q222", (2, 2, 2), 9)]:
        pos, _, lat = oracle_c.supercell(p, z, l, reps, 0.05, seed)
        np.testing.assert_array_equal(pos, GOLD[f"{tag}/pos"])
        np.testing.assert_array_equal(lat, GOLD[f"{tag}/lat"])


@pytest.mark.parametrize("name,rc", [("nl_dimer", 2.0), ("nl_selfimage", 2.5)])
def test_nl_known_answers(oracle_c, name, rc):
    cases = {"nl_dimer": (np.array([[50.0, 50, 50], [51.0, 50, 50]]), np.array([1, 1], np.int32), np.eye(3) * 100),
             "nl_selfimage": (np.array([[0.3, 0.7, 1.1]]), np.array([2], np.int32), np.eye(3) * 2.0)}
    g = oracle_c.neighbor_list(*cases[name], None, rc)
    for k in ("src", "dst", "off", "dist", "vec"):
        np.testing.assert_array_equal(g[k], GOLD[f"{name}/{k}"])
    assert len(g["src"]) == {"nl_dimer": 2, "nl_selfimage": 6}[name]
    b = oracle_c.neighbor_list(*cases[name], None, rc, brute=True)
    np.testing.assert_array_equal(b["src"], g["src"])


def test_nl_quartz(oracle_c):
    p, z, l = fixture_args("quartz")
    for tag, reps in [("q333", (3, 3, 3)), ("q555", (5, 5, 5))]:
        pos, zz, lat = oracle_c.supercell(p, z, l, reps, 0.05, 1)
        g = oracle_c.neighbor_list(pos, zz, lat, None, 5.0)
        assert len(g["src"]) == GOLD[f"{tag}/nl/count"][0]
        h = hashlib.sha256()
        for a in (g["src"], g["dst"], g["off"]):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest().encode() == GOLD[f"{tag}/nl/hash"].tobytes()
        if tag == "q333":
            for k in ("src", "dst", "off", "dist", "vec"):
                np.testing.assert_array_equal(g[k], GOLD[f"{tag}/nl/{k}"])
    assert GOLD["q555/nl/count"][0] == 50340  # SURVEY §8 C1 edge count


def test_partition_chain_hand_trace(oracle_c):
    s = S.chain4()
    d = oracle_c.create(*S.as_args(s), 1.5, p=2, allow_narrow=True)
    for i in range(2):
        L = d.layout(i)
        np.testing.assert_array_equal(L["node_array"], GOLD[f"chain/p{i}/node_array"])
        np.testing.assert_array_equal(L["markers"], GOLD[f"chain/p{i}/markers"])
        for k, v in d.owned_edges(i).items():
            np.testing.assert_array_equal(v, GOLD[f"chain/p{i}/{k}"])
    # hand-trace values of test_partitioner.cpp:57-85
    assert list(d.layout(0)["node_array"]) == [0, 1, 2]
    assert len(d.owned_edges(0)["owned_edges"]) == 3 and len(d.owned_edges(0)["border_edge_list"]) == 1


def test_partition_quartz(oracle_c):
    z = np.tile(S.fixture("quartz").species, 12)
    d = oracle_c.create(GOLD["q322/pos"], z, GOLD["q322/lat"], None, 4.0, p=3, allow_narrow=True)
    np.testing.assert_array_equal(d.owner(), GOLD["q322/owner"])
    np.testing.assert_array_equal(d.rule()[1], GOLD["q322/rule"])
    for i in range(3):
        L = d.layout(i)
        np.testing.assert_array_equal(L["node_array"], GOLD[f"q322/p{i}/node_array"])
        np.testing.assert_array_equal(L["markers"], GOLD[f"q322/p{i}/markers"])
        np.testing.assert_array_equal(L["duplicates"], GOLD[f"q322/p{i}/duplicates"])
        for k, v in d.owned_edges(i).items():
            np.testing.assert_array_equal(v, GOLD[f"q322/p{i}/{k}"])


def test_line_graphs(oracle_c):
    water = (np.array([[10, 10, 10], [10.96, 10, 10], [9.76, 10.93, 10]], float), np.array([8, 1, 1], np.int32), np.eye(3) * 20)
    np.testing.assert_array_equal(oracle_c.line_graph(*water, None, 2.0, 1.2), GOLD["water/serial"])
    np.testing.assert_array_equal(oracle_c.line_graph(*water, None, 2.0, 1.2, brute=True), GOLD["water/serial"])
    tri = (np.array([[10, 10, 10], [11, 10, 10], [10.5, 10.87, 10]], float), np.full(3, 6, np.int32), np.eye(3) * 20)
    lg = oracle_c.line_graph(*tri, None, 1.5, 1.5)
    assert len(lg) == 6
    np.testing.assert_array_equal(lg, GOLD["tri/serial"])
    z = np.tile(S.fixture("quartz").species, 8)
    d = oracle_c.create(GOLD["q222/pos"], z, GOLD["q222/lat"], None, 4.0, r3=3.0, p=3, allow_narrow=True)
    b = d.bonds()
    np.testing.assert_array_equal(b["edge_of_bond"], GOLD["q222/edge_of_bond"])
    np.testing.assert_array_equal(b["bond_owner"], GOLD["q222/bond_owner"])
    for i in range(3):
        L = d.layout(i, bonds=True)
        np.testing.assert_array_equal(L["node_array"], GOLD[f"q222/p{i}/bond_node_array"])
        np.testing.assert_array_equal(L["markers"], GOLD[f"q222/p{i}/bond_markers"])
        np.testing.assert_array_equal(d.line_edges(i), GOLD[f"q222/p{i}/line_edges"])


def test_model_c1(oracle_c):
    p, z, l = fixture_args("quartz")
    pos, zz, lat = oracle_c.supercell(p, z, l, (5, 5, 5), 0.05, 1)
    prm = oracle_c.params_init(12345, 16, 8, 2, 5.0)
    np.testing.assert_array_equal(prm, GOLD["c1/params"])
    o = oracle_c.forward_serial(pos, zz, lat, None, prm, 16, 8, 2, 5.0)
    assert abs(o["energy"] - GOLD["c1/energy"][0]) <= 1e-9
    np.testing.assert_allclose(o["per_atom"], GOLD["c1/per_atom"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(o["forces"], GOLD["c1/forces"], atol=1e-10, rtol=0)
    np.testing.assert_allclose(o["stress"], GOLD["c1/stress"], atol=1e-12, rtol=0)
    # C2: the reference's own p=2 distributed result agrees with serial (acceptance C1 bar)
    assert abs(GOLD["c2/energy"][0] - GOLD["c1/energy"][0]) <= 1e-9
    np.testing.assert_allclose(GOLD["c2/forces"], GOLD["c1/forces"], atol=1e-10, rtol=0)


def test_model_three_body(oracle_c):
    p, z, l = fixture_args("quartz")
    pos, zz, lat = oracle_c.supercell(p, z, l, (3, 3, 3), 0.05, 1)
    prm = GOLD["tb/params"]
    o = oracle_c.forward_serial(pos, zz, lat, None, prm, 16, 8, 3, 5.0, 3.0)
    assert abs(o["energy"] - GOLD["tb/energy"][0]) <= 1e-9
    np.testing.assert_allclose(o["forces"], GOLD["tb/forces"], atol=1e-10, rtol=0)
    np.testing.assert_allclose(o["stress"], GOLD["tb/stress"], atol=1e-12, rtol=0)


def test_isolated_atom(oracle_c):
    prm = oracle_c.params_init(5, 16, 8, 2, 4.0)
    o = oracle_c.forward_serial(np.array([[25.0, 25, 25]]), np.array([26], np.int32), np.eye(3) * 50, None, prm, 16, 8, 2, 4.0)
    assert abs(o["energy"] - GOLD["iso/energy"][0]) <= 1e-14


@pytest.mark.parametrize("seed", [0, 3, 10, 17, 40, 81])
def test_live_reference_nl_and_partitions(oracle_c, oracle_ref, seed):
    """acceptance.cpp criteria 3/5 generators, C restatement == live reference."""
    s = S.random_gas(30 + seed * 14, seed)
    args = S.as_args(s)
    a = oracle_c.neighbor_list(*args, 3.2)
    b = oracle_ref.neighbor_list(*args, 3.2)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])
    p = 2 + seed % 3
    dc = oracle_c.create(*args, 3.2, r3=2.4, p=p, allow_narrow=True)
    dr = oracle_ref.create(*args, 3.2, r3=2.4, p=p, allow_narrow=True)
    np.testing.assert_array_equal(dc.owner(), dr.owner())
    for i in range(p):
        for bonds in (False, True):
            lc, lr = dc.layout(i, bonds), dr.layout(i, bonds)
            for k in lc:
                np.testing.assert_array_equal(lc[k], lr[k])
        np.testing.assert_array_equal(dc.line_edges(i), dr.line_edges(i))


def test_errors(oracle_c):
    from oracle.oracle import OracleError
    s = S.random_system(3, (10, 10, 10), 4)
    with pytest.raises(OracleError, match="more partitions than atoms"):
        oracle_c.create(*S.as_args(s), 2.0, p=5)
    with pytest.raises(OracleError, match="cutoff must be positive"):
        oracle_c.neighbor_list(*S.as_args(s), 0.0)
    big = S.random_system(200, (40, 10, 10), 3)
    with pytest.raises(OracleError, match="partition-width error"):
        oracle_c.create(*S.as_args(big), 3.0, p=16)


def test_bench_ref_systems(oracle_ref):
    """bench.py's reference arm builds its systems through the reference
    (never mapping the product library); they are bitwise the test builders."""
    import bench
    from tests import systems as S
    for spec, mk in [(("quartz", (6, 5, 4)), lambda: S.quartz((6, 5, 4))),
                     (("liquid", 3000), lambda: S.liquid(3000))]:
        pos, z, lat, _ = bench.ref_system(spec, oracle_ref)
        s = mk()
        np.testing.assert_array_equal(pos, s.positions)
        np.testing.assert_array_equal(z, s.species)
        np.testing.assert_array_equal(lat, s.lattice)


def test_bench_reference_arm_maps_no_product_library():
    import json
    import subprocess
    import sys
    from oracle.oracle import available
    if not available("ref"):
        pytest.skip("oracle/_ref not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--config", "c1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["native_libs"] == ["oracle/_ref/libgraphmd_ref.so"]
    assert line["config"]["workload"].startswith("c1")
