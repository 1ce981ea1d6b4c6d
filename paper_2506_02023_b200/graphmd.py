"""Python mirror of the reference's graphmd plugin API over the C ABI.

Same names, argument meaning and error behaviour as the C++ reference
(`graphmd::Distributed`, `forward_distributed`, the graph / partition /
line-graph views), backed by libgraphmd_b200.so (include/graphmd_b200.h).

  reference                                  here
  Distributed::create_distributed            Distributed.create_distributed   engine.hpp:51-56
  forward_distributed(dist, params, timing)  forward_distributed              potential.hpp:58-60
  ToyPotentialParams::init                   ToyPotentialParams.init          potential.hpp:35-37
  build_neighbor_list                        build_neighbor_list              neighborlist.hpp:37-38
  AtomGraph / PartitionRule / SpanLayout /   same-named classes (numpy views)
  AtomPartition / PartitionedAtomGraph /
  BondSet / PartitionedLineGraph
  DistributedFeatures + transfer API         DistributedFeatures (CUDA tensor blocks)

There is no CPU fallback: importing works anywhere, but every computation
goes through the CUDA library and raises if it (or a GPU) is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgraphmd_b200.so")

GMD_OK, GMD_ERR_CONFIG, GMD_ERR_RUNTIME, GMD_ERR_CUDA, GMD_ERR_ARG = 0, 2, 3, 4, 5
GMD_ALLOW_NARROW, GMD_INPUT_DEVICE, GMD_EQUAL_WIDTH = 1, 2, 4
GMD_LINE_PARTS = 8  # build the per-partition line-graph edges inside gmd_build
GMD_OUTPUT_DEVICE, GMD_OUTPUT_F32 = 1, 2
GMD_F32, GMD_F64 = 0, 1

# every symbol include/graphmd_b200.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "gmd_version", "gmd_last_error", "gmd_create", "gmd_destroy", "gmd_build",
    "gmd_set_params", "gmd_params_size", "gmd_params_init", "gmd_forward", "gmd_num_nodes",
    "gmd_num_edges", "gmd_num_partitions", "gmd_get_graph", "gmd_get_system", "gmd_get_rule",
    "gmd_get_owner", "gmd_get_layout_size", "gmd_get_layout", "gmd_get_num_duplicates",
    "gmd_get_duplicates", "gmd_get_num_owned_edges", "gmd_get_owned_edges",
    "gmd_get_num_border_edges", "gmd_get_border_edges", "gmd_has_line_graph",
    "gmd_get_num_bonds", "gmd_get_bonds", "gmd_get_num_line_edges", "gmd_get_line_edges",
    "gmd_block_rows", "gmd_block_offset", "gmd_transfer", "gmd_transfer_transpose",
    "gmd_sync_duplicates", "gmd_distribute", "gmd_aggregate",
    "gmd_corrupt_transfer_plan_for_test", "gmd_util_rng_uniform", "gmd_util_supercell",
    "gmd_profile", "gmd_profile_read", "gmd_get_stream", "gmd_launch_count", "gmd_comm_nccl_id",
    "gmd_comm_init_nccl", "gmd_comm_init_local", "gmd_comm_info", "gmd_num_owned", "gmd_get_owned_ids", "gmd_num_interior",
    "gmd_md_masses", "gmd_md_maxwell_boltzmann", "gmd_md_evaluate", "gmd_md_step", "gmd_md_observe",
    "gmd_md_run", "gmd_comm_ipc_export", "gmd_comm_init_ipc",
    # free builder API (partitioner.hpp / linegraph.hpp / neighborlist.hpp)
    "gmd_partition_rule", "gmd_assign_owners", "gmd_build_partitions", "gmd_get_closure",
    "gmd_get_bond_tables", "gmd_brute_force_line_graph", "gmd_brute_force_neighbor_list",
    "gmd_get_csr", "gmd_util_ensure_periodic",
]


class Error(RuntimeError):
    """graphmd::Error (system.hpp:13-15)."""

    def __init__(self, msg: str, code: int = GMD_ERR_CONFIG):
        super().__init__(msg)
        self.code = code


_lib_cache = None


def lib():
    """The loaded CUDA library.  Fails loudly when it is missing."""
    global _lib_cache
    if _lib_cache is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2506_02023_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        V, I, I64, D, U32, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint32, C.c_uint64
        sig = {
            "gmd_version": (C.c_char_p, []),
            "gmd_last_error": (C.c_char_p, [V]),
            "gmd_create": (I, [I, C.POINTER(V)]),
            "gmd_destroy": (None, [V]),
            "gmd_build": (I, [V, I64, V, V, V, V, D, D, D, I, I, U32]),
            "gmd_set_params": (I, [V, I, I, I, D, D, V]),
            "gmd_params_size": (I64, [I, I, I]),
            "gmd_params_init": (I, [U64, I, I, I, D, D, V]),
            "gmd_forward": (I, [V, V, V, V, V, V, U32]),
            "gmd_num_nodes": (I, [V, V]),
            "gmd_num_edges": (I, [V, V]),
            "gmd_num_partitions": (I, [V, V]),
            "gmd_get_graph": (I, [V, V, V, V, V, V]),
            "gmd_get_system": (I, [V, V, V]),
            "gmd_get_rule": (I, [V, V, V]),
            "gmd_get_owner": (I, [V, V]),
            "gmd_get_layout_size": (I, [V, I, I, V]),
            "gmd_get_layout": (I, [V, I, I, V, V]),
            "gmd_get_num_duplicates": (I, [V, I, I, V]),
            "gmd_get_duplicates": (I, [V, I, I, V]),
            "gmd_get_num_owned_edges": (I, [V, I, V]),
            "gmd_get_owned_edges": (I, [V, I, V, V, V]),
            "gmd_get_num_border_edges": (I, [V, I, V]),
            "gmd_get_border_edges": (I, [V, I, V]),
            "gmd_has_line_graph": (I, [V, V]),
            "gmd_get_num_bonds": (I, [V, V]),
            "gmd_get_bonds": (I, [V, V, V]),
            "gmd_get_num_line_edges": (I, [V, I, V]),
            "gmd_get_line_edges": (I, [V, I, V]),
            "gmd_block_rows": (I, [V, I, V]),
            "gmd_block_offset": (I, [V, I, I, V]),
            "gmd_transfer": (I, [V, I, V, I, I]),
            "gmd_transfer_transpose": (I, [V, I, V, I, I]),
            "gmd_sync_duplicates": (I, [V, I, V, I, I]),
            "gmd_distribute": (I, [V, I, V, V, I, I]),
            "gmd_aggregate": (I, [V, I, V, V, I, I]),
            "gmd_corrupt_transfer_plan_for_test": (I, [V]),
            "gmd_util_rng_uniform": (I, [U64, I64, D, D, V]),
            "gmd_util_supercell": (I, [I64, V, V, V, I, I, I, D, U64, V, V, V]),
            "gmd_profile": (I, [V, I]),
            "gmd_profile_read": (I, [V, V, I, V, V, V]),
            "gmd_get_stream": (I, [V, C.POINTER(V)]),
            "gmd_launch_count": (I, [V]),
            "gmd_comm_nccl_id": (I, [V]),
            "gmd_comm_init_nccl": (I, [V, I, I, V]),
            "gmd_comm_init_local": (I, [V, I]),
            "gmd_comm_info": (I, [V, V, V]),
            "gmd_num_owned": (I, [V, V]),
            "gmd_num_interior": (I, [V, V]),
            "gmd_get_owned_ids": (I, [V, V]),
            "gmd_md_masses": (I, [I64, V, V]),
            "gmd_md_maxwell_boltzmann": (I, [I64, V, D, U64, V]),
            "gmd_md_evaluate": (I, [V, I64, V, V, V, V, D, D, D, I, U32, V, V, V]),
            "gmd_md_step": (I, [V, I64, V, V, V, V, V, V, V, D, D, D, D, I, U32, V, V]),
            "gmd_md_observe": (I, [V, I64, V, V, V, V, V]),
            "gmd_md_run": (I, [V, I64, V, V, V, V, V, V, D, I64, D, D, D, I, U32, V]),
            "gmd_comm_ipc_export": (I, [V, I, I, I64, V]),
            "gmd_comm_init_ipc": (I, [V, V]),
            "gmd_partition_rule": (I, [V, I64, V, V, I, I, V, V]),
            "gmd_assign_owners": (I, [V, I64, V, V, I, I, V, V, V]),
            "gmd_build_partitions": (I, [V, I64, V, V, I64, V, V, V, V, D, D, D, I, I, V, V, U32]),
            "gmd_get_closure": (I, [V, I, V, V]),
            "gmd_get_bond_tables": (I, [V, V]),
            "gmd_brute_force_line_graph": (I, [V, V, V]),
            "gmd_brute_force_neighbor_list": (I, [V, I64, V, V, V, D, V, V, V, V, V, V]),
            "gmd_get_csr": (I, [V, V, V]),
            "gmd_util_ensure_periodic": (I, [V, I64, V, V, V, D, V, V]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib_cache = L
    return _lib_cache


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Handle:
    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        rc = lib().gmd_create(device, C.byref(self.h))
        if rc != GMD_OK:
            raise Error(lib().gmd_last_error(None).decode() or "gmd_create failed", rc)
        self.device = device

    def check(self, rc):
        if rc != GMD_OK:
            raise Error(lib().gmd_last_error(self.h).decode(), rc)

    def __del__(self):
        try:
            if self.h:
                lib().gmd_destroy(self.h)
        except Exception:
            pass

    def i64(self, fn, *args):
        out = C.c_int64()
        self.check(fn(self.h, *args, C.byref(out)))
        return out.value


# ---------------------------------------------------------------------------
# system + fixtures (system.hpp)
# ---------------------------------------------------------------------------
@dataclass
class AtomicSystem:
    positions: np.ndarray
    lattice: np.ndarray = field(default_factory=lambda: np.eye(3))
    species: np.ndarray = None
    pbc: Sequence[bool] = (True, True, True)

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64).reshape(-1, 3)
        self.lattice = np.ascontiguousarray(self.lattice, dtype=np.float64).reshape(3, 3)
        if self.species is None:
            self.species = np.ones(len(self.positions), np.int32)
        self.species = np.ascontiguousarray(self.species, dtype=np.int32)

    def size(self) -> int:
        return len(self.positions)

    def any_pbc(self) -> bool:
        return any(self.pbc)

    def validate(self):
        if len(self.species) != len(self.positions):
            raise Error("species length does not match atom count")
        if self.any_pbc() and abs(np.linalg.det(self.lattice)) < 1e-10:
            raise Error("periodic system requires an invertible lattice")


def rng_uniform(seed: int, count: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """Rng(seed).uniform(lo, hi) stream (system.hpp:121-149)."""
    out = np.zeros(count)
    rc = lib().gmd_util_rng_uniform(seed, count, lo, hi, _p(out))
    if rc:
        raise Error("rng_uniform failed", rc)
    return out


def make_supercell(system: AtomicSystem, reps, amplitude: float = 0.0, seed: int = 0) -> AtomicSystem:
    """make_supercell (+ random_perturb when amplitude > 0) (system.cpp:188-240)."""
    n = system.size() * reps[0] * reps[1] * reps[2]
    op = np.zeros((n, 3))
    oz = np.zeros(n, np.int32)
    ol = np.zeros((3, 3))
    rc = lib().gmd_util_supercell(system.size(), _p(system.positions), _p(system.species),
                                  _p(system.lattice), reps[0], reps[1], reps[2], amplitude, seed,
                                  _p(op), _p(oz), _p(ol))
    if rc:
        raise Error("supercell repetitions must be >= 1" if rc == GMD_ERR_CONFIG else "supercell failed", rc)
    return AtomicSystem(op, ol, oz, tuple(system.pbc))


def random_perturb(system: AtomicSystem, amplitude: float, seed: int) -> AtomicSystem:
    if amplitude < 0.0:
        raise Error("perturbation amplitude must be >= 0")
    return make_supercell(system, (1, 1, 1), amplitude, seed)


# ---------------------------------------------------------------------------
# model parameters (potential.hpp:15-48)
# ---------------------------------------------------------------------------
@dataclass
class ToyPotentialParams:
    feature_width: int = 16
    basis_count: int = 8
    layers: int = 2
    r_atom: float = 4.0
    r_3body: float = 0.0
    seed: int = 0
    blob: np.ndarray = None

    def threebody(self) -> bool:
        return self.r_3body > 0.0

    @staticmethod
    def init(seed: int, feature_width: int = 16, basis_count: int = 8, layers: int = 2,
             r_atom: float = 4.0, r_3body: float = 0.0) -> "ToyPotentialParams":
        n = lib().gmd_params_size(feature_width, basis_count, layers)
        blob = np.zeros(n)
        rc = lib().gmd_params_init(seed, feature_width, basis_count, layers, r_atom, r_3body, _p(blob))
        if rc:
            raise Error("layer count must be >= 1", rc)
        p = ToyPotentialParams(feature_width, basis_count, layers, r_atom, r_3body, seed, blob)
        p.validate()
        return p

    def _sizes(self):
        F, K, L = self.feature_width, self.basis_count, self.layers
        return [("embedding", 119 * F), ("layer_w", L * F * F), ("layer_b", L * F),
                ("basis_proj", F * K), ("basis3_proj", F * K), ("w3", F * F), ("w4", F * F),
                ("readout", F)]

    def __getattr__(self, name):
        if name in ("embedding", "layer_w", "layer_b", "basis_proj", "basis3_proj", "w3", "w4", "readout"):
            off = 0
            for k, sz in self._sizes():
                if k == name:
                    return self.blob[off:off + sz]
                off += sz
        raise AttributeError(name)

    def validate(self):
        if self.layers < 1:
            raise Error("layer count must be >= 1")
        if self.feature_width < 1 or self.basis_count < 1:
            raise Error("feature and basis widths must be >= 1")
        if self.r_atom <= 0.0:
            raise Error("atom cutoff must be positive")
        if self.threebody() and self.r_3body > self.r_atom:
            raise Error("three-body cutoff cannot exceed the atom cutoff")
        if self.blob is None or len(self.blob) != sum(s for _, s in self._sizes()):
            raise Error("parameter array has the wrong size")
        off = 0
        for name, sz in self._sizes():  # potential.cpp:157-175, in table order
            if not np.all(np.isfinite(self.blob[off:off + sz])):
                raise Error(f"parameter array {name} contains a non-finite value")
            off += sz

    # binary parameter files (potential.cpp:178-260, docs/formats.md): magic
    # GMPT, u32 version 1, u32 F K L flags, f64 r_atom r_3body, u64 seed, then
    # each table as u64 count + raw little-endian doubles
    def save(self, path: str) -> None:
        import struct
        self.validate()
        try:
            f = open(path, "wb")
        except OSError:
            raise Error(f"cannot write file: {path}")
        with f:
            f.write(b"GMPT" + struct.pack("<5I2dQ", 1, self.feature_width, self.basis_count, self.layers,
                                          1 if self.threebody() else 0, self.r_atom, self.r_3body,
                                          self.seed))
            off = 0
            for _, sz in self._sizes():
                f.write(struct.pack("<Q", sz) + np.ascontiguousarray(self.blob[off:off + sz], "<f8").tobytes())
                off += sz

    @staticmethod
    def load(path: str) -> "ToyPotentialParams":
        import struct
        try:
            f = open(path, "rb")
        except OSError:
            raise Error(f"cannot open file: {path}")
        with f:
            data = f.read()
        if data[:4] != b"GMPT":
            raise Error("bad parameter file magic")
        if len(data) < 8 or struct.unpack_from("<I", data, 4)[0] != 1:
            raise Error("unsupported parameter file version")
        if len(data) < 48:
            raise Error("truncated parameter file")
        F, K, L, _flags = struct.unpack_from("<4I", data, 8)
        r_atom, r3, seed = struct.unpack_from("<2dQ", data, 24)
        off, tables = 48, []
        for _ in range(8):
            if off + 8 > len(data):
                raise Error("truncated parameter file")
            n = struct.unpack_from("<Q", data, off)[0]
            off += 8
            if off + 8 * n > len(data):
                raise Error("truncated parameter file")
            tables.append(np.frombuffer(data, "<f8", n, off).astype(np.float64))
            off += 8 * n
        p = ToyPotentialParams(F, K, L, r_atom, r3, seed, np.concatenate(tables))
        for (name, want), t in zip(p._sizes(), tables):  # per-table messages (potential.cpp:157-175)
            if len(t) != want:
                raise Error(f"parameter array {name} has the wrong size")
            if not np.all(np.isfinite(t)):
                raise Error(f"parameter array {name} contains a non-finite value")
        p.validate()
        return p


@dataclass
class StepTiming:
    graph_creation: float = 0.0
    feature_calculation: float = 0.0
    forward_pass: float = 0.0
    backward_pass: float = 0.0

    @staticmethod
    def category_names():
        return ["Graph Creation", "Feature Calculation", "Forward Pass", "Backward Pass"]

    def total(self):
        return self.graph_creation + self.feature_calculation + self.forward_pass + self.backward_pass

    def __iadd__(self, o):
        self.graph_creation += o.graph_creation
        self.feature_calculation += o.feature_calculation
        self.forward_pass += o.forward_pass
        self.backward_pass += o.backward_pass
        return self


@dataclass
class PotentialOutput:
    energy: float
    per_atom: np.ndarray
    forces: np.ndarray
    stress: np.ndarray


# ---------------------------------------------------------------------------
# graph / partition views (neighborlist.hpp, partitioner.hpp, linegraph.hpp)
# ---------------------------------------------------------------------------
@dataclass
class AtomGraph:
    src: np.ndarray
    dst: np.ndarray
    image_offset: np.ndarray
    distance: np.ndarray
    vector: np.ndarray
    cutoff: float
    num_nodes: int

    def num_edges(self) -> int:
        return len(self.src)

    def edges_into(self, node: int):
        lo = int(np.searchsorted(self.dst, node, "left"))
        hi = int(np.searchsorted(self.dst, node, "right"))
        return lo, hi

    def dump_csv(self, path: str) -> None:
        """AtomGraph::dump_csv (neighborlist.cpp:97-106): src,dst,ox,oy,oz,distance
        with 17 significant digits."""
        with open(path, "w") as f:
            f.write("src,dst,ox,oy,oz,distance\n")
            off = self.image_offset
            f.writelines(f"{s},{d},{o[0]},{o[1]},{o[2]},{x:.17g}\n"
                         for s, d, o, x in zip(self.src.tolist(), self.dst.tolist(), off.tolist(),
                                               self.distance.tolist()))


@dataclass
class PartitionRule:
    axis: int
    boundaries: np.ndarray
    p: int


@dataclass
class Span:
    begin: int
    end: int

    def size(self):
        return self.end - self.begin


@dataclass
class SpanLayout:
    node_array: np.ndarray
    markers: np.ndarray
    duplicates: np.ndarray
    p: int

    def pure_span(self):
        return Span(int(self.markers[0]), int(self.markers[1]))

    def to_span(self, j):
        return Span(int(self.markers[1 + j]), int(self.markers[2 + j]))

    def from_span(self, j):
        return Span(int(self.markers[1 + self.p + j]), int(self.markers[2 + self.p + j]))

    def owned_end(self):
        return int(self.markers[1 + self.p])

    def size(self):
        return len(self.node_array)

    def local_of(self, g):
        hit = np.nonzero(self.node_array == g)[0]
        return int(hit[0]) if len(hit) else -1


@dataclass
class Buckets:
    pure: List[np.ndarray]
    to: List[List[np.ndarray]]
    frm: List[List[np.ndarray]]  # `from` is a Python keyword


def _buckets(layouts: List[SpanLayout], p: int) -> Buckets:
    pure = [L.node_array[L.pure_span().begin:L.pure_span().end] for L in layouts]
    to = [[L.node_array[L.to_span(j).begin:L.to_span(j).end] for j in range(p)] for L in layouts]
    frm = [[to[i][j] for i in range(p)] for j in range(p)]
    return Buckets(pure, to, frm)


@dataclass
class AtomPartition:
    layout: SpanLayout
    owned_edges: np.ndarray
    local_src: np.ndarray
    local_dst: np.ndarray
    border_edge_list: np.ndarray


@dataclass
class PartitionedAtomGraph:
    rule: PartitionRule
    buckets: Buckets
    owner: np.ndarray
    parts: List[AtomPartition]
    p: int


@dataclass
class BondSet:
    edge_of_bond: np.ndarray
    bond_of_edge: np.ndarray
    r: float
    tau: float

    def size(self):
        return len(self.edge_of_bond)


@dataclass
class LineGraphPartition:
    layout: SpanLayout
    line_edges: np.ndarray  # (local e, local e') pairs, sorted by (global e', global e)


@dataclass
class PartitionedLineGraph:
    bonds: BondSet
    bond_owner: np.ndarray
    bond_buckets: Buckets
    parts: List[LineGraphPartition]
    p: int

    def dump_csv(self, path: str) -> None:
        """PartitionedLineGraph::dump_csv (linegraph.cpp:173-181): one line edge
        per row as (partition, global bond e, global bond e')."""
        with open(path, "w") as f:
            f.write("partition,bond_e_global,bond_ep_global\n")
            for i, part in enumerate(self.parts):
                na = part.layout.node_array
                le = np.asarray(part.line_edges).reshape(-1, 2)
                f.writelines(f"{i},{a},{b}\n" for a, b in zip(na[le[:, 0]].tolist(),
                                                            na[le[:, 1]].tolist()))


def partition_plan_to_json(parts: "PartitionedAtomGraph") -> str:
    """partition_plan_to_json (partitioner.cpp:220-236): the reference's
    nlohmann dump(2) layout (sorted keys, two-space indent)."""
    import json

    def lists(x):
        return [[int(v) for v in np.asarray(a).ravel()] for a in x]

    j = {"p": int(parts.p), "axis": int(parts.rule.axis),
         "boundaries": [float(b) for b in parts.rule.boundaries],
         "pure": lists(parts.buckets.pure),
         "to": [lists(row) for row in parts.buckets.to],
         "from": [lists(row) for row in parts.buckets.frm],
         "partitions": [{"node_array": [int(v) for v in pt.layout.node_array],
                         "markers": [int(v) for v in pt.layout.markers],
                         "owned_edge_count": int(len(pt.owned_edges))} for pt in parts.parts]}
    return _json_dump2(j, 0)


def _json_dump2(v, ind: int) -> str:
    """The layout the reference's JSON writer produces with dump(2): sorted
    keys, two-space indent, arrays of integers on one line, other arrays one
    element per line."""
    pad, pad1 = "  " * ind, "  " * (ind + 1)
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f'{pad1}"{k}": {_json_dump2(v[k], ind + 1)}' for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, list):
        if not v:
            return "[]"
        if all(isinstance(x, int) and not isinstance(x, bool) for x in v):
            return "[" + ",".join(str(x) for x in v) + "]"
        return "[\n" + ",\n".join(pad1 + _json_dump2(x, ind + 1) for x in v) + "\n" + pad + "]"
    if isinstance(v, float):
        return repr(v)
    return str(v)


EDGE_FEATURES = 2  # DistributedFeatures.bonds of owned-edge blocks


class DistributedFeatures:
    """Per-partition feature blocks in ONE CUDA tensor (rows x width); block i
    is rows [offsets[i], offsets[i+1]) aligned to partition i's layout (atom
    or bond layout, or its owned edges for edge features)."""

    def __init__(self, data, offsets, width, bonds):
        self.data, self.offsets, self.width, self.bonds = data, offsets, width, bonds

    def block(self, i):
        return self.data[self.offsets[i]:self.offsets[i + 1]]

    def row(self, i, local):
        return self.data[self.offsets[i] + local]


# ---------------------------------------------------------------------------
# Distributed (engine.hpp:49-151)
# ---------------------------------------------------------------------------
class Distributed:
    """Distributed execution handle on one GPU: partitioned graphs plus
    transfer plans, all resident in HBM."""

    def __init__(self, handle: _Handle, system: AtomicSystem, p: int, n_threads: int,
                 atom_cutoff: float, threebody_cutoff, tau):
        self._h = handle
        self._system_in = system
        self._p = p
        self._n_threads = n_threads if n_threads > 0 else 1
        self.atom_cutoff = atom_cutoff
        self.threebody_cutoff = threebody_cutoff
        self.threebody_tau = tau
        self._graph = self._parts = self._lines = self._system = None

    @staticmethod
    def create_distributed(system: AtomicSystem, atom_cutoff: float,
                           threebody_cutoff: Optional[float], p: int, n_threads: int,
                           allow_narrow: bool = False, threebody_tau: float = 0.0,
                           device: int = 0, handle: Optional[_Handle] = None,
                           equal_width: bool = False) -> "Distributed":
        """Distributed::create_distributed (engine.cpp:44-65).  Pass `handle`
        to reuse the device buffers of a previous build (per-step rebuilds)."""
        h = handle or _Handle(device)
        flags = (GMD_ALLOW_NARROW if allow_narrow else 0) | (GMD_EQUAL_WIDTH if equal_width else 0)
        pbc = np.array([1 if b else 0 for b in system.pbc], np.uint8)
        r3 = float(threebody_cutoff) if threebody_cutoff is not None else 0.0
        if threebody_cutoff is not None and r3 <= 0.0:
            raise Error("three-body cutoff must be positive")
        h.check(lib().gmd_build(h.h, system.size(), _p(system.positions), _p(system.species),
                                _p(system.lattice), _p(pbc), float(atom_cutoff), r3,
                                float(threebody_tau), int(p), int(n_threads), flags))
        return Distributed(h, system, p, n_threads, atom_cutoff, threebody_cutoff, threebody_tau)

    # ---- scalars
    def num_partitions(self):
        return self._p

    def num_threads(self):
        return self._n_threads

    def has_line_graph(self):
        out = C.c_int()
        self._h.check(lib().gmd_has_line_graph(self._h.h, C.byref(out)))
        return bool(out.value)

    def num_nodes(self):
        return self._h.i64(lib().gmd_num_nodes)

    def num_edges(self):
        return self._h.i64(lib().gmd_num_edges)

    # ---- views
    def system(self) -> AtomicSystem:
        if self._system is None:
            n = self.num_nodes()
            pos = np.zeros((n, 3))
            lat = np.zeros((3, 3))
            self._h.check(lib().gmd_get_system(self._h.h, _p(pos), _p(lat)))
            self._system = AtomicSystem(pos, lat, self._system_in.species.copy(), (True, True, True))
        return self._system

    def graph(self) -> AtomGraph:
        if self._graph is None:
            ne = self.num_edges()
            g = dict(src=np.zeros(ne, np.int64), dst=np.zeros(ne, np.int64),
                     off=np.zeros((ne, 3), np.int32), dist=np.zeros(ne), vec=np.zeros((ne, 3)))
            self._h.check(lib().gmd_get_graph(self._h.h, *(_p(g[k]) for k in ("src", "dst", "off", "dist", "vec"))))
            self._graph = AtomGraph(g["src"], g["dst"], g["off"], g["dist"], g["vec"],
                                    float(self.atom_cutoff), self.num_nodes())
        return self._graph

    def _layout(self, part, bonds) -> SpanLayout:
        h, L = self._h, lib()
        size = C.c_int64()
        h.check(L.gmd_get_layout_size(h.h, part, bonds, C.byref(size)))
        na = np.zeros(size.value, np.int64)
        mk = np.zeros(2 + 2 * self._p, np.int64)
        h.check(L.gmd_get_layout(h.h, part, bonds, _p(na), _p(mk)))
        nd = C.c_int64()
        h.check(L.gmd_get_num_duplicates(h.h, part, bonds, C.byref(nd)))
        dups = np.zeros((nd.value, 2), np.int64)
        h.check(L.gmd_get_duplicates(h.h, part, bonds, _p(dups)))
        return SpanLayout(na, mk, dups, self._p)

    def atom_parts(self) -> PartitionedAtomGraph:
        if self._parts is None:
            h, L, p = self._h, lib(), self._p
            axis = C.c_int()
            b = np.zeros(p + 1)
            h.check(L.gmd_get_rule(h.h, C.byref(axis), _p(b)))
            owner = np.zeros(self.num_nodes(), np.int32)
            h.check(L.gmd_get_owner(h.h, _p(owner)))
            parts = []
            for i in range(p):
                lay = self._layout(i, 0)
                cnt = C.c_int64()
                h.check(L.gmd_get_num_owned_edges(h.h, i, C.byref(cnt)))
                oe, ls, ld = (np.zeros(cnt.value, np.int64) for _ in range(3))
                h.check(L.gmd_get_owned_edges(h.h, i, _p(oe), _p(ls), _p(ld)))
                h.check(L.gmd_get_num_border_edges(h.h, i, C.byref(cnt)))
                bd = np.zeros(cnt.value, np.int64)
                h.check(L.gmd_get_border_edges(h.h, i, _p(bd)))
                parts.append(AtomPartition(lay, oe, ls, ld, bd))
            self._parts = PartitionedAtomGraph(PartitionRule(axis.value, b, p),
                                               _buckets([x.layout for x in parts], p), owner, parts, p)
        return self._parts

    def line_parts(self) -> PartitionedLineGraph:
        if not self.has_line_graph():
            raise Error("no line graph was built")
        if self._lines is None:
            h, L, p = self._h, lib(), self._p
            nb = self._h.i64(L.gmd_get_num_bonds)
            eob = np.zeros(nb, np.int64)
            own = np.zeros(nb, np.int32)
            h.check(L.gmd_get_bonds(h.h, _p(eob), _p(own)))
            boe = np.full(self.num_edges(), -1, np.int64)
            boe[eob] = np.arange(nb)
            parts = []
            for i in range(p):
                lay = self._layout(i, 1)
                cnt = C.c_int64()
                h.check(L.gmd_get_num_line_edges(h.h, i, C.byref(cnt)))
                le = np.zeros((cnt.value, 2), np.int64)
                h.check(L.gmd_get_line_edges(h.h, i, _p(le)))
                parts.append(LineGraphPartition(lay, le))
            bonds = BondSet(eob, boe, float(self.threebody_cutoff), float(self.threebody_tau))
            self._lines = PartitionedLineGraph(bonds, own, _buckets([x.layout for x in parts], p), parts, p)
        return self._lines

    def src_nodes(self, partition):
        return self.atom_parts().parts[partition].local_src

    def dst_nodes(self, partition):
        return self.atom_parts().parts[partition].local_dst

    def atom_rows(self, partition):
        return self.atom_parts().parts[partition].layout.size()

    def bond_rows(self, partition):
        return self.line_parts().parts[partition].layout.size()

    # ---- feature API (engine.hpp:74-129), blocks are CUDA tensors
    def _offsets(self, bonds):
        h, L = self._h, lib()
        offs = []
        for i in range(self._p):
            o = C.c_int64()
            h.check(L.gmd_block_offset(h.h, i, bonds, C.byref(o)))
            offs.append(o.value)
        tot = C.c_int64()
        h.check(L.gmd_block_rows(h.h, bonds, C.byref(tot)))
        offs.append(tot.value)
        return offs

    def _make(self, width, bonds, dtype):
        import torch
        offs = self._offsets(bonds)
        data = torch.zeros((offs[-1], width), dtype=dtype, device=f"cuda:{self._h.device}")
        return DistributedFeatures(data, offs, width, bonds)

    def make_atom_features(self, width, dtype=None):
        import torch
        return self._make(width, 0, dtype or torch.float64)

    def make_bond_features(self, width, dtype=None):
        import torch
        if not self.has_line_graph():
            raise Error("no line graph was built")
        return self._make(width, 1, dtype or torch.float64)

    @staticmethod
    def _dt(f):
        import torch
        if f.data.dtype == torch.float64:
            return GMD_F64
        if f.data.dtype == torch.float32:
            return GMD_F32
        raise Error("features must be float32 or float64", GMD_ERR_ARG)

    def _op(self, fn, f):
        if f.bonds == EDGE_FEATURES:
            raise Error("transfers apply to atom or bond feature blocks", GMD_ERR_ARG)
        self._h.check(fn(self._h.h, f.bonds, C.c_void_p(f.data.data_ptr()), f.width, self._dt(f)))

    def atom_transfer(self, f):
        self._op(lib().gmd_transfer, f)

    def bond_transfer(self, f):
        self._op(lib().gmd_transfer, f)

    def atom_transfer_transpose(self, f):
        self._op(lib().gmd_transfer_transpose, f)

    def bond_transfer_transpose(self, f):
        self._op(lib().gmd_transfer_transpose, f)

    def sync_atom_duplicates(self, f):
        self._op(lib().gmd_sync_duplicates, f)

    def sync_bond_duplicates(self, f):
        self._op(lib().gmd_sync_duplicates, f)

    def _distribute(self, features, width, bonds):
        import torch
        arr = np.ascontiguousarray(features, np.float64)
        n = self.num_nodes() if not bonds else self.line_parts().bonds.size()
        if arr.size != n * width:
            raise Error("node feature shape mismatch" if not bonds else "bond feature shape mismatch")
        f = self._make(width, bonds, torch.float64)
        self._h.check(lib().gmd_distribute(self._h.h, bonds, _p(arr), C.c_void_p(f.data.data_ptr()),
                                           width, GMD_F64))
        return f

    def distribute_node_features(self, features, width):
        return self._distribute(features, width, 0)

    def _aggregate(self, f):
        n = self.num_nodes() if not f.bonds else self.line_parts().bonds.size()
        out = np.zeros(n * f.width, np.float64 if self._dt(f) == GMD_F64 else np.float32)
        self._h.check(lib().gmd_aggregate(self._h.h, f.bonds, C.c_void_p(f.data.data_ptr()), _p(out),
                                          f.width, self._dt(f)))
        return out

    def aggregate(self, f):
        return self._aggregate(f)

    def aggregate_bonds(self, f):
        return self._aggregate(f)

    def corrupt_transfer_plan_for_test(self):
        self._h.check(lib().gmd_corrupt_transfer_plan_for_test(self._h.h))

    # owned-edge feature blocks (engine.cpp:103-120, 248-260): partition i
    # holds its owned edges' rows in owned_edges order (API plumbing, not the
    # model path: the gather / scatter run as device index ops)
    def _edge_order(self):
        parts = self.atom_parts().parts
        offs = np.concatenate([[0], np.cumsum([len(x.owned_edges) for x in parts])]).tolist()
        return np.concatenate([x.owned_edges for x in parts]).astype(np.int64), offs

    def distribute_edge_features(self, features, width):
        import torch
        arr = np.ascontiguousarray(features, np.float64)
        if arr.size != self.num_edges() * width:
            raise Error("edge feature shape mismatch")
        order, offs = self._edge_order()
        dev = f"cuda:{self._h.device}"
        src = torch.from_numpy(arr.reshape(-1, width)).to(dev)
        data = src[torch.from_numpy(order).to(dev)].contiguous()
        return DistributedFeatures(data, offs, width, EDGE_FEATURES)

    def aggregate_edges(self, f):
        import torch
        if f.bonds != EDGE_FEATURES:
            raise Error("aggregate_edges needs edge feature blocks", GMD_ERR_ARG)
        order, _ = self._edge_order()
        out = torch.zeros((self.num_edges(), f.width), dtype=f.data.dtype, device=f.data.device)
        out[torch.from_numpy(order).to(f.data.device)] = f.data
        return out.reshape(-1).cpu().numpy()

    def parallel_for_partitions(self, fn):
        """fn(partition) for every partition; the first failing partition's
        error is re-raised with its id (engine.cpp:262-284).  Callbacks run in
        partition order: the device work they enqueue is stream-ordered."""
        errors = [None] * self._p
        for i in range(self._p):
            try:
                fn(i)
            except Exception as e:  # noqa: BLE001 -- reported with the partition id
                errors[i] = str(e)
        for i, e in enumerate(errors):
            if e is not None:
                raise Error(f"worker for partition {i} failed: {e}", GMD_ERR_RUNTIME)

    def run_layered(self, layers, features):
        """Each layer on every partition, then the border exchange
        (engine.cpp:286-294)."""
        for layer in layers:
            self.parallel_for_partitions(lambda i: layer(i, features))
            self.sync_atom_duplicates(features)
            self.atom_transfer(features)

    # per-step reuse
    @property
    def handle(self):
        return self._h


def forward_distributed(dist: Distributed, params: ToyPotentialParams,
                        timing: Optional[StepTiming] = None) -> PotentialOutput:
    """forward_distributed (potential.cpp:563-985) on the GPU."""
    params.validate()
    h = dist.handle
    L = lib()
    h.check(L.gmd_set_params(h.h, params.feature_width, params.basis_count, params.layers,
                             params.r_atom, params.r_3body, _p(params.blob)))
    n = dist.num_nodes()
    e = C.c_double()
    pa = np.zeros(n)
    fo = np.zeros((n, 3))
    st = np.zeros(9)
    tm = np.zeros(4)
    h.check(L.gmd_forward(h.h, C.byref(e), _p(pa), _p(fo), _p(st), _p(tm), 0))
    if timing is not None:
        timing.feature_calculation += tm[1]
        timing.forward_pass += tm[2]
        timing.backward_pass += tm[3]
    return PotentialOutput(e.value, pa, fo, st.reshape(3, 3))


def forward_serial(system: AtomicSystem, params: ToyPotentialParams, device: int = 0) -> PotentialOutput:
    """forward_serial (potential.cpp:563): one partition, one worker."""
    r3 = params.r_3body if params.threebody() else None
    d = Distributed.create_distributed(system, params.r_atom, r3, 1, 1, True, device=device)
    return forward_distributed(d, params)


def ensure_periodic(system: AtomicSystem, cutoff: float, device: int = 0) -> AtomicSystem:
    """ensure_periodic (system.cpp:242-270) on the device: non-periodic axes
    padded to extent + 2 cutoff, positions shifted by cutoff - lo."""
    h = _Handle(device)
    n = system.size()
    out_pos = np.zeros((n, 3))
    out_lat = np.zeros((3, 3))
    pbc = np.array([1 if b else 0 for b in system.pbc], np.uint8)
    h.check(lib().gmd_util_ensure_periodic(h.h, n, _p(system.positions), _p(system.lattice), _p(pbc),
                                           cutoff, _p(out_pos), _p(out_lat)))
    return AtomicSystem(out_pos, out_lat, system.species.copy(), (True, True, True))


def finite_difference_forces(system: AtomicSystem, params: ToyPotentialParams, eps: float,
                             device: int = 0) -> np.ndarray:
    """finite_difference_forces (potential.cpp:991-1009): central differences
    of the GPU energy.  The energy sums fp32-computed per-atom terms, so the
    quotient carries ~1e-6 eV / (2 eps) of rounding noise (an fp32-level
    check, not the reference's fp64 1e-6 eV/A)."""
    if eps < 1e-6 or eps > 1e-2:
        raise Error("finite-difference step must lie in [1e-6, 1e-2] A")
    out = np.zeros((system.size(), 3))
    probe = AtomicSystem(system.positions.copy(), system.lattice, system.species, system.pbc)
    for i in range(system.size()):
        for k in range(3):
            x0 = system.positions[i, k]
            probe.positions[i, k] = x0 + eps
            ep = forward_serial(probe, params, device).energy
            probe.positions[i, k] = x0 - eps
            em = forward_serial(probe, params, device).energy
            probe.positions[i, k] = x0
            out[i, k] = -(ep - em) / (2.0 * eps)
    return out


def finite_difference_stress(system: AtomicSystem, params: ToyPotentialParams, eps: float,
                             device: int = 0) -> np.ndarray:
    """finite_difference_stress (potential.cpp:1011-1037): symmetrised strain
    derivative of the GPU energy over the volume."""
    if not (0.0 < eps <= 1e-3):
        raise Error("strain step must lie in (0, 1e-3]")
    base = ensure_periodic(system, params.r_atom, device)
    volume = abs(np.linalg.det(base.lattice))

    def deform(a, b, strain):  # x_a += strain x_b for every position and lattice row
        pos = base.positions.copy()
        lat = base.lattice.copy()
        pos[:, a] += strain * pos[:, b]
        lat[:, a] += strain * lat[:, b]
        return AtomicSystem(pos, lat, base.species, base.pbc)

    raw = np.zeros((3, 3))
    for a in range(3):
        for b in range(3):
            ep = forward_serial(deform(a, b, eps), params, device).energy
            em = forward_serial(deform(a, b, -eps), params, device).energy
            raw[a, b] = (ep - em) / (2.0 * eps * volume)
    return 0.5 * (raw + raw.T)


def build_neighbor_list(system: AtomicSystem, cutoff: float, n_threads: int = 0,
                        device: int = 0) -> AtomGraph:
    """build_neighbor_list (neighborlist.cpp:108-197) on the GPU."""
    d = Distributed.create_distributed(system, cutoff, None, 1, n_threads, True, device=device)
    return d.graph()


def profile_start(dist: "Distributed"):
    """Clear and enable per-kernel CUDA-event timing on the handle's stream."""
    dist.handle.check(lib().gmd_profile(dist.handle.h, 1))


def profile_read(dist: "Distributed", stop: bool = True):
    """{kernel name: (total device ms, launches)} since profile_start."""
    cap = 128
    names = C.create_string_buffer(8192)
    ms = np.zeros(cap)
    ln = np.zeros(cap, np.int32)
    cnt = C.c_int(cap)
    h = dist.handle
    h.check(lib().gmd_profile_read(h.h, names, 8192, _p(ms), _p(ln), C.byref(cnt)))
    out, parts = {}, names.raw.split(b"\0")
    for k in range(cnt.value):
        out[parts[k].decode()] = (float(ms[k]), int(ln[k]))
    if stop:
        h.check(lib().gmd_profile(h.h, 0))
    return out


def stream_ptr(dist: "Distributed") -> int:
    """cudaStream_t (as int) that every kernel of this handle runs on."""
    s = C.c_void_p()
    dist.handle.check(lib().gmd_get_stream(dist.handle.h, C.byref(s)))
    return s.value or 0


def launch_count() -> int:
    """Kernel launches issued by libgraphmd_b200.so in this process so far."""
    out = C.c_int64()
    lib().gmd_launch_count(C.byref(out))
    return out.value


# ---------------------------------------------------------------------------
# one rank per GPU
# ---------------------------------------------------------------------------
def nccl_unique_id() -> bytes:
    """ncclGetUniqueId on this process (rank 0); broadcast it to the peers."""
    buf = (C.c_uint8 * 128)()
    rc = lib().gmd_comm_nccl_id(buf)
    if rc:
        raise Error(lib().gmd_last_error(None).decode() or "ncclGetUniqueId failed", rc)
    return bytes(buf)


def comm_init_nccl(handle: "_Handle", rank: int, world: int, uid: bytes) -> None:
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    handle.check(lib().gmd_comm_init_nccl(handle.h, rank, world, buf))


def local_group(world: int, device: int = 0) -> List["_Handle"]:
    """`world` handles forming one in-process rank group (each rank must be
    driven from its own thread: build/forward block on the peers)."""
    hs = [_Handle(device) for _ in range(world)]
    arr = (C.c_void_p * world)(*[h.h.value for h in hs])
    rc = lib().gmd_comm_init_local(arr, world)
    if rc:
        raise Error("gmd_comm_init_local failed", rc)
    return hs


def num_interior(dist: "Distributed") -> int:
    """Owned atoms whose in-edges all come from owned atoms (rank mode)."""
    n = C.c_int64()
    dist.handle.check(lib().gmd_num_interior(dist.handle.h, C.byref(n)))
    return n.value


def owned_ids(dist: "Distributed") -> np.ndarray:
    """Global ids of the atoms this handle computes (its rank's slab)."""
    h = dist.handle
    n = C.c_int64()
    h.check(lib().gmd_num_owned(h.h, C.byref(n)))
    out = np.zeros(n.value, np.int64)
    h.check(lib().gmd_get_owned_ids(h.h, _p(out)))
    return out


def run_ranks(fns):
    """Run one callable per rank concurrently (ctypes releases the GIL)."""
    import threading
    res, errs = [None] * len(fns), [None] * len(fns)

    def body(i):
        try:
            res[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001 - reraised below
            errs[i] = e

    ts = [threading.Thread(target=body, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return res


def broadcast_bytes(payload: Optional[bytes], src: int = 0, size: int = 128) -> bytes:
    """Broadcast `size` bytes from rank `src` over the default torch.distributed
    group (gloo: CPU tensor, nccl: tensor on the current device)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.zeros(size, dtype=torch.uint8, device=dev)
    if dist.get_rank() == src:
        t.copy_(torch.tensor(list(payload), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def init_rank_comm(handle: "_Handle", rank: int, world: int) -> None:
    """NCCL halo transport for this process's handle (one process per GPU)."""
    uid = nccl_unique_id() if rank == 0 else None
    comm_init_nccl(handle, rank, world, broadcast_bytes(uid, 0))


def init_rank_comm_ipc(handle: "_Handle", rank: int, world: int, slot_rows: int) -> None:
    """CUDA-IPC peer transport (ranks on one node): export this rank's window,
    all-gather the 64-byte handles over the default torch.distributed group
    (gloo or nccl), attach the peers' windows."""
    import torch
    import torch.distributed as dist
    # collective-safe: every rank takes part in both collectives even when its
    # own export / attach fails, and all ranks agree on the outcome (so a
    # caller can fall back to the NCCL transport without a hang)
    hd = (C.c_uint8 * 64)()
    err = None
    try:
        handle.check(lib().gmd_comm_ipc_export(handle.h, rank, world, slot_rows, hd))
    except Error as e:
        err = e
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    mine = torch.tensor(list(bytes(hd)), dtype=torch.uint8, device=dev)
    allh = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allh, mine)
    if err is None:
        blob = bytes(b for t in allh for b in t.cpu().tolist())
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        try:
            handle.check(lib().gmd_comm_init_ipc(handle.h, buf))
        except Error as e:
            err = e
    ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if err is not None:
        raise err
    if int(ok.item()) == 0:
        raise Error("CUDA-IPC transport failed on a peer rank", GMD_ERR_RUNTIME)


def exchange_plan_consistent(scnt, rcnt, rank: int, all_scnt) -> bool:
    """The invariant the library checks at build time (engine.cpp:132-133):
    what rank j sends to `rank` (its TO_j[rank] block) is exactly the FROM
    span `rank` reserved for j.  all_scnt[j][k] = rows rank j sends to k."""
    return all(j == rank or int(all_scnt[j][rank]) == int(rcnt[j]) for j in range(len(rcnt)))


# ---------------------------------------------------------------------------
# extended-XYZ I/O (system.cpp:95-186, docs/formats.md)
# ---------------------------------------------------------------------------
_SYMBOLS = ("X H He Li Be B C N O F Ne Na Mg Al Si P S Cl Ar K Ca Sc Ti V Cr Mn Fe Co Ni Cu Zn "
            "Ga Ge As Se Br Kr Rb Sr Y Zr Nb Mo Tc Ru Rh Pd Ag Cd In Sn Sb Te I Xe Cs Ba La Ce "
            "Pr Nd Pm Sm Eu Gd Tb Dy Ho Er Tm Yb Lu Hf Ta W Re Os Ir Pt Au Hg Tl Pb Bi Po At Rn "
            "Fr Ra Ac Th Pa U Np Pu Am Cm Bk Cf Es Fm Md No Lr Rf Db Sg Bh Hs Mt Ds Rg Cn Nh Fl "
            "Mc Lv Ts Og").split()
_Z_OF = {sym: z for z, sym in enumerate(_SYMBOLS) if z > 0}


def z_to_symbol(z: int) -> str:
    if z < 1 or z > 118:
        raise Error("atomic number out of range")
    return _SYMBOLS[z]


def _parse_fail(path, line, what):
    raise Error(f"{path}:{line}: {what}")


def load_xyz(path: str) -> AtomicSystem:
    """load_xyz (system.cpp:95-163): count line, comment line with
    Lattice="..." (and optional pbc="T T F"), then `Symbol x y z` lines."""
    try:
        f = open(path)
    except OSError:
        raise Error(f"cannot open file: {path}")
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        _parse_fail(path, 1, "empty file")
    head = lines[0]
    try:  # std::stoul: leading whitespace, optional sign, then digits
        m = __import__("re").match(r"\s*([+-]?\d+)", head)
        natoms = int(m.group(1))
        if natoms < 0:
            natoms %= 1 << 64
    except (AttributeError, ValueError):
        _parse_fail(path, 1, f"expected atom count, got '{head}'")
    if len(lines) < 2:
        _parse_fail(path, 2, "missing comment line")
    com = lines[1]
    lattice = np.eye(3)
    pbc = [True, True, True]
    i = com.find('Lattice="')
    have_lattice = i >= 0
    if have_lattice:
        b = i + 9
        e = com.find('"', b)
        if e < 0:
            _parse_fail(path, 2, "unterminated Lattice field")
        toks = com[b:e].split()
        vals = []
        for t in toks[:9]:
            try:
                vals.append(float(t))
            except ValueError:
                break
        if len(vals) < 9:
            _parse_fail(path, 2, "Lattice needs 9 numbers")
        lattice = np.array(vals).reshape(3, 3)
    i = com.find('pbc="')
    if i >= 0:
        b = i + 5
        e = com.find('"', b)
        toks = (com[b:e] if e >= 0 else com[b:]).split()
        if len(toks) < 3:
            _parse_fail(path, 2, "pbc needs 3 flags")
        pbc = [t in ("T", "True", "true", "1") for t in toks[:3]]
    if not have_lattice:
        if any(pbc):
            _parse_fail(path, 2, "periodic system requires a Lattice field")
        lattice = np.eye(3)
    pos = np.zeros((natoms, 3))
    z = np.zeros(natoms, np.int32)
    for a in range(natoms):
        ln = a + 3
        if ln - 1 >= len(lines):
            _parse_fail(path, ln, "unexpected end of file")
        t = lines[ln - 1].split()
        try:
            sym, x, y, w = t[0], float(t[1]), float(t[2]), float(t[3])
        except (IndexError, ValueError):
            _parse_fail(path, ln, "expected 'symbol x y z'")
        if sym not in _Z_OF:
            _parse_fail(path, ln, f"unknown element symbol '{sym}'")
        z[a] = _Z_OF[sym]
        pos[a] = (x, y, w)
    s = AtomicSystem(pos, lattice, z, tuple(pbc))
    s.validate()
    return s


def save_xyz(system: AtomicSystem, path: str, comment_extra: str = "") -> None:
    """save_xyz (system.cpp:165-186): 17 significant digits."""
    g = lambda x: format(float(x), ".17g")  # noqa: E731  (= ostream precision 17)
    try:
        f = open(path, "w")
    except OSError:
        raise Error(f"cannot write file: {path}")
    with f:
        f.write(f"{system.size()}\n")
        f.write('Lattice="' + " ".join(g(v) for v in system.lattice.reshape(-1)) + '" pbc="'
                + " ".join("T" if b else "F" for b in system.pbc) + '"')
        if comment_extra:
            f.write(" " + comment_extra)
        f.write("\n")
        for r, zz in zip(system.positions, system.species):
            f.write(f"{z_to_symbol(int(zz))} {g(r[0])} {g(r[1])} {g(r[2])}\n")


# ---------------------------------------------------------------------------
# on-device MD: the caller of the hot path (md.hpp:14-89, md.cpp)
# ---------------------------------------------------------------------------
class units:  # md.hpp:14-21
    kAccel = 9.648533212e-3
    kKinetic = 103.642697
    kBoltzmann = 8.617333262e-5


def atomic_mass(z) -> np.ndarray:
    """atomic_mass (system.cpp:289-293) for an array of atomic numbers."""
    z = np.ascontiguousarray(np.atleast_1d(z), dtype=np.int32)
    out = np.zeros(len(z))
    rc = lib().gmd_md_masses(len(z), _p(z), _p(out))
    if rc:
        raise Error(lib().gmd_last_error(None).decode(), rc)
    return out


def maxwell_boltzmann_velocities(system: AtomicSystem, temperature: float, seed: int) -> np.ndarray:
    """maxwell_boltzmann_velocities (md.cpp:20-52): deterministic in seed,
    centre-of-mass momentum removed."""
    v = np.zeros((system.size(), 3))
    rc = lib().gmd_md_maxwell_boltzmann(system.size(), _p(system.species), temperature, seed, _p(v))
    if rc:
        raise Error(lib().gmd_last_error(None).decode(), rc)
    return v


@dataclass
class MDOptions:  # md.hpp:36-49
    dt: float = 1.0
    steps: int = 0
    partitions: int = 1
    threads: int = 0
    allow_narrow: bool = False
    seed: int = 0
    init_temperature: float = 300.0
    energy_csv: str = ""
    timing_csv: str = ""
    trajectory_xyz: str = ""   # snapshot prefix: PREFIX.<step>.xyz
    snapshot_every: int = 0    # 0 disables


@dataclass
class MDStepRecord:  # md.hpp:51-58
    step: int = 0
    potential: float = 0.0
    kinetic: float = 0.0
    total: float = 0.0
    max_force: float = 0.0
    timing: StepTiming = field(default_factory=StepTiming)


class MDState:
    """MDState (md.hpp:23-34) with the dynamic arrays resident on the GPU
    (torch float64 tensors): positions, velocities, forces, masses."""

    def __init__(self, system: AtomicSystem, velocities: np.ndarray, device: int = 0):
        import torch
        system.validate()
        self.system = system
        dev = f"cuda:{device}"
        self.handle = _Handle(device)
        self.pos = torch.tensor(system.positions, dtype=torch.float64, device=dev)
        self.vel = torch.tensor(velocities, dtype=torch.float64, device=dev)
        self.forces = torch.zeros_like(self.pos)
        self.masses = torch.tensor(atomic_mass(system.species), dtype=torch.float64, device=dev)
        self.species = torch.tensor(system.species, dtype=torch.int32, device=dev)
        self.potential_energy = 0.0
        self.step = 0
        self._have_forces = False

    def _observe(self):
        ke, fm = C.c_double(), C.c_double()
        self.handle.check(lib().gmd_md_observe(self.handle.h, self.size(), self.vel.data_ptr(),
                                               self.masses.data_ptr(), self.forces.data_ptr(),
                                               C.byref(ke), C.byref(fm)))
        return ke.value, fm.value

    def size(self) -> int:
        return self.system.size()

    def kinetic_energy(self) -> float:
        return self._observe()[0]

    def temperature(self) -> float:
        if self.size() == 0:
            return 0.0
        dof = max(1.0, 3.0 * self.size() - 3.0)
        return 2.0 * self.kinetic_energy() / (dof * units.kBoltzmann)

    def positions(self) -> np.ndarray:
        return self.pos.cpu().numpy()

    def velocities(self) -> np.ndarray:
        return self.vel.cpu().numpy()

    def forces_host(self) -> np.ndarray:
        return self.forces.cpu().numpy()

    def current_system(self) -> AtomicSystem:
        return AtomicSystem(self.positions(), self.system.lattice.copy(), self.system.species.copy(),
                            tuple(self.system.pbc))


@dataclass
class MDResult:
    state: MDState
    records: List[MDStepRecord]


def init_md_state(system: AtomicSystem, opts: MDOptions, device: int = 0) -> MDState:
    """init_md_state (md.cpp:71-83): masses, Maxwell-Boltzmann velocities."""
    return MDState(system, maxwell_boltzmann_velocities(system, opts.init_temperature, opts.seed),
                   device)


def _md_args(state: MDState, params: "ToyPotentialParams", opts: MDOptions):
    params.validate()
    h = state.handle
    h.check(lib().gmd_set_params(h.h, params.feature_width, params.basis_count, params.layers,
                                 params.r_atom, params.r_3body, _p(params.blob)))
    pbc = np.array([1 if b else 0 for b in state.system.pbc], np.uint8)
    flags = GMD_ALLOW_NARROW if opts.allow_narrow else 0
    return h, pbc, flags


def _timing(tm, timing: Optional[StepTiming]):
    if timing is not None:
        timing.graph_creation += tm[0]
        timing.feature_calculation += tm[1]
        timing.forward_pass += tm[2]
        timing.backward_pass += tm[3]


def md_evaluate(state: MDState, params: "ToyPotentialParams", opts: MDOptions,
                timing: Optional[StepTiming] = None) -> None:
    """evaluate (md.cpp:55-69) at the current device positions: graph rebuild +
    forward; forces and potential energy land in the state."""
    h, pbc, flags = _md_args(state, params, opts)
    e = C.c_double()
    tm = np.zeros(4)
    h.check(lib().gmd_md_evaluate(h.h, state.size(), state.pos.data_ptr(), state.species.data_ptr(),
                                  _p(state.system.lattice), _p(pbc), params.r_atom,
                                  params.r_3body if params.threebody() else 0.0, 0.0,
                                  opts.partitions, flags, state.forces.data_ptr(), C.byref(e),
                                  _p(tm)))
    _timing(tm, timing)
    state.potential_energy = e.value
    state._have_forces = True


def velocity_verlet_step(state: MDState, params: "ToyPotentialParams", opts: MDOptions,
                         timing: Optional[StepTiming] = None) -> None:
    """velocity_verlet_step (md.cpp:85-110), every array in HBM: half-kick +
    drift, wrap_positions, graph + partition rebuild, forward, half-kick."""
    if not state._have_forces:
        raise Error("step requires forces at the current positions")
    if opts.dt < 0.0:
        raise Error("time step must be >= 0")
    h, pbc, flags = _md_args(state, params, opts)
    e = C.c_double()
    tm = np.zeros(4)
    rc = lib().gmd_md_step(h.h, state.size(), state.pos.data_ptr(), state.vel.data_ptr(),
                           state.forces.data_ptr(), state.masses.data_ptr(),
                           state.species.data_ptr(), _p(state.system.lattice), _p(pbc), opts.dt,
                           params.r_atom, params.r_3body if params.threebody() else 0.0, 0.0,
                           opts.partitions, flags, C.byref(e), _p(tm))
    if rc:
        msg = lib().gmd_last_error(h.h).decode()
        if msg.startswith("non-finite force"):
            msg += f" at step {state.step + 1}"
        raise Error(msg, rc)
    _timing(tm, timing)
    state.step += 1
    state.potential_energy = e.value


def run_md(system: AtomicSystem, params: "ToyPotentialParams", opts: MDOptions,
           device: int = 0) -> MDResult:
    """run_md (md.cpp:112-160) on the GPU; records row 0 = initial state."""
    state = init_md_state(system, opts, device)
    records: List[MDStepRecord] = []

    def record(step, t):
        ke, fm = state._observe()
        records.append(MDStepRecord(step, state.potential_energy, ke, state.potential_energy + ke,
                                    fm, t))

    def snapshot(step):  # md.cpp:131-137
        if opts.trajectory_xyz and opts.snapshot_every > 0 and step % opts.snapshot_every == 0:
            save_xyz(state.current_system(), f"{opts.trajectory_xyz}.{step}.xyz")

    t0 = StepTiming()
    md_evaluate(state, params, opts, t0)
    record(0, t0)
    snapshot(0)
    for step in range(1, opts.steps + 1):
        t = StepTiming()
        velocity_verlet_step(state, params, opts, t)
        record(step, t)
        snapshot(step)
    if opts.energy_csv:
        write_energy_csv(opts.energy_csv, records)
    if opts.timing_csv:
        write_timing_csv(opts.timing_csv, [r.timing for r in records])
    return MDResult(state, records)


def write_energy_csv(path: str, records: List[MDStepRecord]) -> None:
    """write_energy_csv (md.cpp:162-179)."""
    cols = ",".join(n.lower().replace(" ", "_") + "_s" for n in StepTiming.category_names())
    with open(path, "w") as f:
        f.write("step,potential_ev,kinetic_ev,total_ev,max_force_ev_per_a," + cols + "\n")
        for r in records:
            t = r.timing
            f.write(f"{r.step},{r.potential:.12g},{r.kinetic:.12g},{r.total:.12g},"
                    f"{r.max_force:.12g},{t.graph_creation:.12g},{t.feature_calculation:.12g},"
                    f"{t.forward_pass:.12g},{t.backward_pass:.12g}\n")


def write_timing_csv(path: str, rows: List[StepTiming]) -> None:
    """write_timing_csv (engine.cpp:29-41): step, then the four categories."""
    with open(path, "w") as f:
        f.write("step," + ",".join(StepTiming.category_names()) + "\n")
        for i, t in enumerate(rows):
            f.write(f"{i},{t.graph_creation:.9g},{t.feature_calculation:.9g},"
                    f"{t.forward_pass:.9g},{t.backward_pass:.9g}\n")
