"""Test systems mirroring the reference's generators (proj/tests/helpers.hpp:24-75,
acceptance.cpp:45-58) and the benchmark configs (BASELINE.json configs / SURVEY §8d).

Random streams come from the product library's host RNG (gmd_util_*), which
tests/test_abi.py pins against the oracle's mt19937_64 restatement."""
import json
import os

import numpy as np

from paper_2506_02023_b200 import graphmd as G

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixture(name):
    with open(os.path.join(GOLDEN, "fixtures.json")) as f:
        d = json.load(f)[name]
    return G.AtomicSystem(np.array(d["positions"]), np.array(d["lattice"]), np.array(d["species"], np.int32))


def random_system(n, box, seed, species=(14, 8)):
    u = G.rng_uniform(seed, 3 * n) if n else np.zeros(0)
    # Rng::uniform(0, box_k) in x, y, z order per atom (helpers.hpp:24-38)
    pos = np.zeros((n, 3))
    for k in range(3):
        pos[:, k] = 0.0 + (box[k] - 0.0) * u[k::3]
    lat = np.diag(np.asarray(box, dtype=np.float64))
    z = np.array([species[i % len(species)] for i in range(n)], np.int32)
    return G.AtomicSystem(pos, lat, z)


def random_triclinic(n, box, seed):
    s = random_system(n, (box, box, box), seed)
    s.lattice[1, 0] += 0.12 * box
    s.lattice[2, 0] -= 0.07 * box
    s.lattice[2, 1] += 0.09 * box
    return s


def random_gas(n, seed):
    edge = np.cbrt(n / 0.07)  # acceptance.cpp:51-58
    return random_triclinic(n, edge, seed) if seed % 3 == 0 else random_system(n, (edge, edge * 1.05, edge * 0.95), seed)


def chain4():
    return G.AtomicSystem(np.array([[4.5 + i, 4.0, 4.0] for i in range(4)]), np.diag([12.0, 8.0, 8.0]),
                          np.full(4, 6, np.int32))


def quartz(reps, amp=0.05, seed=1):
    return G.make_supercell(fixture("quartz"), reps, amp, seed)


def liquid(n, density=0.1, seed=7):
    """SURVEY §8d C4 generator: cube of edge cbrt(n/density), Rng(seed).uniform
    positions, species cycling O, H, H."""
    edge = np.cbrt(n / density)
    u = G.rng_uniform(seed, 3 * n, 0.0, edge)
    pos = u.reshape(n, 3)
    z = np.array([8 if i % 3 == 0 else 1 for i in range(n)], np.int32)
    return G.AtomicSystem(pos, np.diag([edge] * 3), z)


def as_args(s):
    return s.positions, s.species, s.lattice, np.array([1 if b else 0 for b in s.pbc], np.uint8)


def edge_keys(src, dst, off):
    """sorted (src, dst, ox, oy, oz) multiset as a structured array"""
    k = np.zeros(len(src), dtype=[("s", "i8"), ("d", "i8"), ("x", "i4"), ("y", "i4"), ("z", "i4")])
    k["s"], k["d"] = src, dst
    k["x"], k["y"], k["z"] = off[:, 0], off[:, 1], off[:, 2]
    return np.sort(k)
