"""Generate tests/golden/golden.npz from the REFERENCE library itself.

Run in the build container (needs oracle/_ref/libgraphmd_ref.so, compiled from
/root/reference/proj/src by `make -C oracle ref`):

    python tests/golden/gen_golden.py

Every vector here is an output of the unmodified reference (through
oracle/ref_shim.cpp).  tests/test_oracle.py pins the C restatement
(oracle/gmd_oracle.c) against these vectors, and the GPU parity tests compare
the CUDA path with that pinned restatement.  Inputs are built from
tests/golden/fixtures.json (the reference's own fixture files) and the
reference's own Rng/make_supercell/random_perturb.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle  # noqa: E402


def fixture(name):
    d = json.load(open(os.path.join(HERE, "fixtures.json")))[name]
    return np.array(d["positions"]), np.array(d["species"], np.int32), np.array(d["lattice"])


def keyhash(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    R = Oracle("ref")
    out = {}
    qp, qz, ql = fixture("quartz")

    # --- neighbour-list known answers (test_neighborlist.cpp:31-65)
    cases = {
        "nl_dimer": (np.array([[50.0, 50, 50], [51.0, 50, 50]]), np.array([1, 1], np.int32), np.eye(3) * 100, 2.0),
        "nl_selfimage": (np.array([[0.3, 0.7, 1.1]]), np.array([2], np.int32), np.eye(3) * 2.0, 2.5),
    }
    for name, (p, z, l, rc) in cases.items():
        g = R.neighbor_list(p, z, l, None, rc)
        for k, v in g.items():
            out[f"{name}/{k}"] = v
    # quartz supercells used by the C1/C2 configs (full arrays for 3^3, hash for 5^3)
    for reps in [(3, 3, 3), (5, 5, 5)]:
        pos, z, lat = R.supercell(qp, qz, ql, reps, 0.05, 1)
        tag = "q%d%d%d" % reps
        out[f"{tag}/pos"] = pos
        out[f"{tag}/lat"] = lat
        g = R.neighbor_list(pos, z, lat, None, 5.0)
        if reps == (3, 3, 3):
            for k, v in g.items():
                out[f"{tag}/nl/{k}"] = v
        out[f"{tag}/nl/count"] = np.array([len(g["src"])])
        out[f"{tag}/nl/hash"] = np.frombuffer(keyhash(g["src"], g["dst"], g["off"]).encode(), np.uint8)

    # --- partitions: chain hand trace + quartz 3x2x2 p=3 (test_partitioner.cpp:57-127)
    chain = (np.array([[4.5 + i, 4.0, 4.0] for i in range(4)]), np.full(4, 6, np.int32), np.diag([12.0, 8.0, 8.0]))
    d = R.create(*chain, None, 1.5, p=2, allow_narrow=True)
    for i in range(2):
        L = d.layout(i)
        out[f"chain/p{i}/node_array"] = L["node_array"]
        out[f"chain/p{i}/markers"] = L["markers"]
        oe = d.owned_edges(i)
        for k, v in oe.items():
            out[f"chain/p{i}/{k}"] = v
    pos, z, lat = R.supercell(qp, qz, ql, (3, 2, 2), 0.05, 6)
    d = R.create(pos, z, lat, None, 4.0, p=3, allow_narrow=True)
    out["q322/pos"], out["q322/lat"] = pos, lat
    out["q322/owner"] = d.owner()
    out["q322/rule"] = d.rule()[1]
    for i in range(3):
        L = d.layout(i)
        out[f"q322/p{i}/node_array"] = L["node_array"]
        out[f"q322/p{i}/markers"] = L["markers"]
        out[f"q322/p{i}/duplicates"] = L["duplicates"]
        for k, v in d.owned_edges(i).items():
            out[f"q322/p{i}/{k}"] = v

    # --- line graphs (test_linegraph.cpp:69-147)
    water = (np.array([[10, 10, 10], [10.96, 10, 10], [9.76, 10.93, 10]], float), np.array([8, 1, 1], np.int32), np.eye(3) * 20)
    out["water/serial"] = R.line_graph(*water, None, 2.0, 1.2, 0.0)
    tri = (np.array([[10, 10, 10], [11, 10, 10], [10.5, 10.87, 10]], float), np.full(3, 6, np.int32), np.eye(3) * 20)
    out["tri/serial"] = R.line_graph(*tri, None, 1.5, 1.5, 0.0)
    pos, z, lat = R.supercell(qp, qz, ql, (2, 2, 2), 0.05, 9)
    out["q222/pos"], out["q222/lat"] = pos, lat
    d = R.create(pos, z, lat, None, 4.0, r3=3.0, p=3, allow_narrow=True)
    b = d.bonds()
    out["q222/edge_of_bond"] = b["edge_of_bond"]
    out["q222/bond_owner"] = b["bond_owner"]
    for i in range(3):
        L = d.layout(i, bonds=True)
        out[f"q222/p{i}/bond_node_array"] = L["node_array"]
        out[f"q222/p{i}/bond_markers"] = L["markers"]
        out[f"q222/p{i}/line_edges"] = d.line_edges(i)

    # --- model (test_potential.cpp:31-51; C1 config of BASELINE.json)
    pos, z, lat = R.supercell(qp, qz, ql, (5, 5, 5), 0.05, 1)
    prm = R.params_init(12345, 16, 8, 2, 5.0, 0.0)
    out["c1/params"] = prm
    o = R.forward_serial(pos, z, lat, None, prm, 16, 8, 2, 5.0, 0.0)
    for k in ("per_atom", "forces", "stress"):
        out[f"c1/{k}"] = o[k]
    out["c1/energy"] = np.array([o["energy"]])
    d = R.create(pos, z, lat, None, 5.0, p=2)
    o2 = d.forward(prm, 16, 8, 2, 5.0)
    out["c2/energy"] = np.array([o2["energy"]])
    out["c2/forces"] = o2["forces"]
    pos3, z3, lat3 = R.supercell(qp, qz, ql, (3, 3, 3), 0.05, 1)
    prm3 = R.params_init(7, 16, 8, 3, 5.0, 3.0)
    out["tb/params"] = prm3
    o3 = R.forward_serial(pos3, z3, lat3, None, prm3, 16, 8, 3, 5.0, 3.0)
    for k in ("per_atom", "forces", "stress"):
        out[f"tb/{k}"] = o3[k]
    out["tb/energy"] = np.array([o3["energy"]])
    iso = R.forward_serial(np.array([[25.0, 25, 25]]), np.array([26], np.int32), np.eye(3) * 50, None,
                           R.params_init(5, 16, 8, 2, 4.0), 16, 8, 2, 4.0)
    out["iso/energy"] = np.array([iso["energy"]])
    out["rng/normal3"] = R.rng_normal(3, 1001)
    out["rng/uniform7"] = R.rng_uniform(7, 999, 0.0, 100.0)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
