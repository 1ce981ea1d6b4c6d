"""Generate tests/golden/fixtures.json from the reference's fixture files.

Run here (the reference tree exists only in the build container):
    python tests/golden/gen_fixtures.py
Reads /root/reference/proj/fixtures/{quartz,water}.xyz (extended XYZ:
Lattice="ax ay az bx by bz cx cy cz", species symbol + Cartesian position per
line) and stores lattice / species numbers / positions as JSON so that neither
the GPU box nor the tests ever read /root/reference at run time.
"""
import json
import os
import re

SRC = "/root/reference/proj/fixtures"
Z = {"H": 1, "O": 8, "Si": 14}


def read(path):
    lines = open(path).read().splitlines()
    n = int(lines[0].strip())
    lat = [float(x) for x in re.search(r'Lattice="([^"]*)"', lines[1]).group(1).split()]
    species, pos = [], []
    for ln in lines[2:2 + n]:
        t = ln.split()
        species.append(Z[t[0]])
        pos.append([float(t[1]), float(t[2]), float(t[3])])
    return {"lattice": [lat[0:3], lat[3:6], lat[6:9]], "species": species, "positions": pos}


if __name__ == "__main__":
    out = {name: read(os.path.join(SRC, name + ".xyz")) for name in ("quartz", "water")}
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fixtures.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", dst)
    # the fixture file the reference's own tests open (fixture_path("quartz.xyz"),
    # proj/tests/helpers.hpp:15-21), re-serialised by the reference's save_xyz
    # (17 significant digits: loads back bitwise) for tests/cpp/ref/*
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    import numpy as np
    from oracle.oracle import Oracle
    q = out["quartz"]
    xyz = os.path.join(os.path.dirname(dst), "quartz.xyz")
    Oracle("ref").save_xyz(np.array(q["positions"]), np.array(q["species"], np.int32),
                           np.array(q["lattice"]), np.ones(3, np.uint8), xyz)
    print("wrote", xyz)
