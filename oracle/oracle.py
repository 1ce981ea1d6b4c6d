"""ORACLE TEST INFRASTRUCTURE -- not part of the product.

ctypes bindings for the two CPU checkers:

* ``backend="c"``   -> oracle/libgmd_oracle.so, the plain-C fp64 restatement
  of the reference hot path (oracle/gmd_oracle.c);
* ``backend="ref"`` -> oracle/_ref/libgraphmd_ref.so, the UNMODIFIED reference
  library compiled from /root/reference/proj/src by oracle/Makefile, behind the
  extern "C" shim oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product path (paper_2506_02023_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "c": (os.path.join(HERE, "libgmd_oracle.so"), "orc_"),
    "ref": (os.path.join(HERE, "_ref", "libgraphmd_ref.so"), "gref_"),
}

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def available(backend: str) -> bool:
    return os.path.exists(LIBS[backend][0])


class OracleError(RuntimeError):
    pass


class Oracle:
    """Uniform view over the C restatement and the compiled reference."""

    def __init__(self, backend: str = "c"):
        path, pre = LIBS[backend]
        if not os.path.exists(path):
            raise OracleError(f"oracle library {path} not built (make -C oracle)")
        self.backend = backend
        self.lib = C.CDLL(path)
        self.pre = pre
        L = self.lib

        def f(name, res, *args):
            fn = getattr(L, pre + name)
            fn.restype = res
            fn.argtypes = list(args)
            return fn

        V = C.c_void_p
        I = C.c_int
        D = C.c_double
        U = C.c_uint64
        self._err = f("last_error", C.c_char_p)
        self._create = f("create", V, _i64, V, V, V, V, D, D, D, I, *(() if backend == "c" else (I,)), I)
        self._destroy = f("destroy", None, V)
        self._num_nodes = f("num_nodes", _i64, V)
        self._num_edges = f("num_edges", _i64, V)
        self._graph = f("graph", None, V, V, V, V, V, V)
        self._system = f("system", None, V, V, V)
        self._rule = f("rule", I, V, V)
        self._owner = f("owner", None, V, V)
        self._layout_size = f("layout_size", _i64, V, I, I)
        self._layout = f("layout", None, V, I, I, V, V)
        self._num_dups = f("num_dups", _i64, V, I, I)
        self._dups = f("dups", None, V, I, I, V)
        self._num_owned = f("num_owned_edges", _i64, V, I)
        self._owned = f("owned_edges", None, V, I, V, V, V)
        self._num_border = f("num_border", _i64, V, I)
        self._border = f("border", None, V, I, V)
        self._has_lg = f("has_line_graph", I, V)
        self._num_bonds = f("num_bonds", _i64, V)
        self._bonds = f("bonds", None, V, V, V)
        self._num_line = f("num_line_edges", _i64, V, I)
        self._line = f("line_edges", None, V, I, V)
        self._fwd_serial = f("forward_serial", I, _i64, V, V, V, V, I, I, I, D, D, V, V, V, V, V)
        self._params_init = f("params_init", None, U, I, I, I, D, D, V)
        self._supercell = f("supercell", None, _i64, V, V, V, I, I, I, D, U, V, V, V)
        self._rng_uniform = f("rng_uniform", None, U, _i64, D, D, V)
        self._rng_normal = f("rng_normal", None, U, _i64, V)
        if backend == "c":
            self._nl = f("neighbor_list", V, _i64, V, V, V, V, D, I)
        else:
            self._nl = f("neighbor_list", V, _i64, V, V, V, V, D, I, I)
            self._fwd = f("forward", I, V, I, I, I, D, D, V, V, V, V, V, V)
        if backend == "c":
            self._md = f("md_run", I, _i64, V, V, V, V, I, I, I, D, D, V, D, _i64, D, U, V, V, V, V)
        else:
            self._md = f("md_run", I, _i64, V, V, V, V, I, I, I, D, D, V, D, _i64, I, D, U, V, V,
                         V, V)
        if backend == "ref":
            self._dump_graph = f("dump_graph", I, V, C.c_char_p)
            self._dump_line = f("dump_line", I, V, C.c_char_p)
            self._plan_json = f("plan_json", _i64, V, V, _i64)
            self._save_xyz = f("save_xyz", I, _i64, V, V, V, V, C.c_char_p, C.c_char_p)
            self._load_xyz = f("load_xyz", _i64, C.c_char_p, V, V, V, V)
            self._psave = f("params_save", I, I, I, I, D, D, U, V, C.c_char_p)
            self._pload = f("params_load", _i64, C.c_char_p, V, V, V, V, _i64)
        self._g_ne = f("graph_num_edges", _i64, V)
        self._g_get = f("graph_get", None, V, V, V, V, V, V)
        self._g_free = f("graph_destroy", None, V)
        self._lg = f("line_graph", V, _i64, V, V, V, V, D, D, D, I)
        self._p_n = f("pairs_size", _i64, V)
        self._p_get = f("pairs_get", None, V, V)
        self._p_free = f("pairs_destroy", None, V)

    def error(self) -> str:
        return self._err().decode()

    # ---- helpers -------------------------------------------------------
    @staticmethod
    def _sysargs(pos, z, lat, pbc):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        z = np.ascontiguousarray(z, dtype=np.int32)
        lat = np.ascontiguousarray(lat, dtype=np.float64)
        pbc = np.ascontiguousarray(pbc if pbc is not None else [1, 1, 1], dtype=np.uint8)
        return pos, z, lat, pbc

    def params_init(self, seed, F=16, K=8, L=2, r_atom=4.0, r3=0.0):
        n = 119 * F + L * F * F + L * F + 2 * F * K + 2 * F * F + F
        blob = np.zeros(n, np.float64)
        self._params_init(seed, F, K, L, r_atom, r3, _ptr(blob))
        return blob

    def supercell(self, pos, z, lat, reps, amp=0.0, seed=0):
        pos, z, lat, _ = self._sysargs(pos, z, lat, None)
        n = len(z) * reps[0] * reps[1] * reps[2]
        op = np.zeros((n, 3))
        oz = np.zeros(n, np.int32)
        ol = np.zeros((3, 3))
        self._supercell(len(z), _ptr(pos), _ptr(z), _ptr(lat), reps[0], reps[1], reps[2],
                        amp, seed, _ptr(op), _ptr(oz), _ptr(ol))
        return op, oz, ol

    def rng_uniform(self, seed, count, lo=0.0, hi=1.0):
        out = np.zeros(count)
        self._rng_uniform(seed, count, lo, hi, _ptr(out))
        return out

    def rng_normal(self, seed, count):
        out = np.zeros(count)
        self._rng_normal(seed, count, _ptr(out))
        return out

    def neighbor_list(self, pos, z, lat, pbc, rc, brute=False, n_threads=1):
        pos, z, lat, pbc = self._sysargs(pos, z, lat, pbc)
        args = [len(z), _ptr(pos), _ptr(z), _ptr(lat), _ptr(pbc), rc, int(brute)]
        if self.backend == "ref":
            args.append(n_threads)
        g = self._nl(*args)
        if not g:
            raise OracleError(self.error())
        ne = self._g_ne(g)
        out = dict(src=np.zeros(ne, np.int64), dst=np.zeros(ne, np.int64),
                   off=np.zeros((ne, 3), np.int32), dist=np.zeros(ne), vec=np.zeros((ne, 3)))
        self._g_get(g, *(_ptr(out[k]) for k in ("src", "dst", "off", "dist", "vec")))
        self._g_free(g)
        return out

    def line_graph(self, pos, z, lat, pbc, rc, r, tau=0.0, brute=False):
        pos, z, lat, pbc = self._sysargs(pos, z, lat, pbc)
        ph = self._lg(len(z), _ptr(pos), _ptr(z), _ptr(lat), _ptr(pbc), rc, r, tau, int(brute))
        if not ph:
            raise OracleError(self.error())
        n = self._p_n(ph)
        out = np.zeros((n, 2), np.int64)
        self._p_get(ph, _ptr(out))
        self._p_free(ph)
        return out

    def forward_serial(self, pos, z, lat, pbc, params, F, K, L, r_atom, r3=0.0):
        pos, z, lat, pbc = self._sysargs(pos, z, lat, pbc)
        n = len(z)
        e = np.zeros(1)
        pa = np.zeros(n)
        fo = np.zeros((n, 3))
        st = np.zeros((3, 3))
        params = np.ascontiguousarray(params, np.float64)
        rc = self._fwd_serial(n, _ptr(pos), _ptr(z), _ptr(lat), _ptr(pbc), F, K, L, r_atom, r3,
                              _ptr(params), _ptr(e), _ptr(pa), _ptr(fo), _ptr(st))
        if rc:
            raise OracleError(self.error())
        return dict(energy=float(e[0]), per_atom=pa, forces=fo, stress=st)

    def save_xyz(self, pos, z, lat, pbc, path, comment=""):
        """save_xyz (system.cpp:165-186), backend "ref" only."""
        pos, z, lat, pbc = self._sysargs(pos, z, lat, pbc)
        if self._save_xyz(len(z), _ptr(pos), _ptr(z), _ptr(lat), _ptr(pbc), path.encode(),
                          comment.encode()):
            raise OracleError(self.error())

    def params_save(self, F, K, L, r_atom, r3, seed, blob, path):
        """ToyPotentialParams::save (potential.cpp:178-213), backend "ref" only."""
        blob = np.ascontiguousarray(blob, dtype=np.float64)
        if self._psave(F, K, L, r_atom, r3, seed, _ptr(blob), path.encode()):
            raise OracleError(self.error())

    def params_load(self, path):
        """ToyPotentialParams::load (potential.cpp:215-260): (F, K, L, r_atom, r3, seed, blob)."""
        hdr, r, seed = np.zeros(3, np.int32), np.zeros(2), np.zeros(1, np.uint64)
        n = self._pload(path.encode(), _ptr(hdr), _ptr(r), _ptr(seed), None, 0)
        if n < 0:
            raise OracleError(self.error())
        blob = np.zeros(n)
        self._pload(path.encode(), _ptr(hdr), _ptr(r), _ptr(seed), _ptr(blob), n)
        return int(hdr[0]), int(hdr[1]), int(hdr[2]), float(r[0]), float(r[1]), int(seed[0]), blob

    def load_xyz(self, path):
        """load_xyz (system.cpp:95-163), backend "ref" only: (pos, z, lat, pbc)."""
        n = self._load_xyz(path.encode(), None, None, None, None)
        if n < 0:
            raise OracleError(self.error())
        pos, z = np.zeros((n, 3)), np.zeros(n, np.int32)
        lat, pbc = np.zeros((3, 3)), np.zeros(3, np.uint8)
        self._load_xyz(path.encode(), _ptr(pos), _ptr(z), _ptr(lat), _ptr(pbc))
        return pos, z, lat, pbc.astype(bool)

    def md_run(self, pos, z, lat, pbc, params, F, K, L, r_atom, r3, dt, steps, temperature,
               seed, partitions=1):
        """run_md (md.cpp:112-160): final pos / vel / forces and the per-step
        records (potential, kinetic, total, max_force), row 0 = initial."""
        pos, z, lat, pbc = self._sysargs(pos, z, lat, pbc)
        n = len(z)
        op, ov, of = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 3))
        rec = np.zeros((steps + 1, 4))
        params = np.ascontiguousarray(params, np.float64)
        args = [n, _ptr(pos), _ptr(z), _ptr(lat), _ptr(pbc), F, K, L, r_atom, r3, _ptr(params), dt,
                steps]
        if self.backend == "ref":
            args.append(partitions)
        args += [temperature, seed, _ptr(op), _ptr(ov), _ptr(of), _ptr(rec)]
        if self._md(*args):
            raise OracleError(self.error())
        return dict(pos=op, vel=ov, forces=of, records=rec)

    def create(self, pos, z, lat, pbc, rc, r3=0.0, tau=0.0, p=1, allow_narrow=False, n_threads=1):
        pos, z, lat, pbc = self._sysargs(pos, z, lat, pbc)
        args = [len(z), _ptr(pos), _ptr(z), _ptr(lat), _ptr(pbc), rc, r3, tau, p]
        if self.backend == "ref":
            args.append(n_threads)
        args.append(int(allow_narrow))
        h = self._create(*args)
        if not h:
            raise OracleError(self.error())
        return OracleDist(self, h, p)


class OracleDist:
    """Snapshot of a create_distributed result as numpy arrays."""

    # the reference's own dump formats (backend "ref" only)
    def dump_graph(self, path):
        if self.o._dump_graph(self.h, path.encode()):
            raise OracleError(self.o.error())

    def dump_line(self, path):
        if self.o._dump_line(self.h, path.encode()):
            raise OracleError(self.o.error())

    def plan_json(self) -> str:
        n = self.o._plan_json(self.h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self.o._plan_json(self.h, buf, n + 1)
        return buf.value.decode()

    def __init__(self, o: Oracle, h, p):
        self.o, self.h, self.p = o, h, p

    def __del__(self):
        try:
            self.o._destroy(self.h)
        except Exception:
            pass

    def graph(self):
        o, h = self.o, self.h
        ne = o._num_edges(h)
        out = dict(src=np.zeros(ne, np.int64), dst=np.zeros(ne, np.int64),
                   off=np.zeros((ne, 3), np.int32), dist=np.zeros(ne), vec=np.zeros((ne, 3)))
        o._graph(h, *(_ptr(out[k]) for k in ("src", "dst", "off", "dist", "vec")))
        return out

    def num_nodes(self):
        return self.o._num_nodes(self.h)

    def system(self):
        n = self.num_nodes()
        pos = np.zeros((n, 3))
        lat = np.zeros((3, 3))
        self.o._system(self.h, _ptr(pos), _ptr(lat))
        return pos, lat

    def rule(self):
        b = np.zeros(self.p + 1)
        axis = self.o._rule(self.h, _ptr(b))
        return axis, b

    def owner(self):
        out = np.zeros(self.num_nodes(), np.int32)
        self.o._owner(self.h, _ptr(out))
        return out

    def layout(self, part, bonds=False):
        o, h = self.o, self.h
        n = o._layout_size(h, part, int(bonds))
        na = np.zeros(n, np.int64)
        mk = np.zeros(2 + 2 * self.p, np.int64)
        o._layout(h, part, int(bonds), _ptr(na), _ptr(mk))
        nd = o._num_dups(h, part, int(bonds))
        dups = np.zeros((nd, 2), np.int64)
        o._dups(h, part, int(bonds), _ptr(dups))
        return dict(node_array=na, markers=mk, duplicates=dups)

    def owned_edges(self, part):
        o, h = self.o, self.h
        n = o._num_owned(h, part)
        a, b, c = (np.zeros(n, np.int64) for _ in range(3))
        o._owned(h, part, _ptr(a), _ptr(b), _ptr(c))
        nb = o._num_border(h, part)
        bd = np.zeros(nb, np.int64)
        o._border(h, part, _ptr(bd))
        return dict(owned_edges=a, local_src=b, local_dst=c, border_edge_list=bd)

    def has_line_graph(self):
        return bool(self.o._has_lg(self.h))

    def bonds(self):
        nb = self.o._num_bonds(self.h)
        eob = np.zeros(nb, np.int64)
        own = np.zeros(nb, np.int32)
        self.o._bonds(self.h, _ptr(eob), _ptr(own))
        return dict(edge_of_bond=eob, bond_owner=own)

    def line_edges(self, part):
        n = self.o._num_line(self.h, part)
        out = np.zeros((n, 2), np.int64)
        self.o._line(self.h, part, _ptr(out))
        return out

    def forward(self, params, F, K, L, r_atom, r3=0.0):
        """forward_distributed (reference backend only)."""
        o = self.o
        n = self.num_nodes()
        e = np.zeros(1)
        pa = np.zeros(n)
        fo = np.zeros((n, 3))
        st = np.zeros((3, 3))
        tm = np.zeros(4)
        params = np.ascontiguousarray(params, np.float64)
        rc = o._fwd(self.h, F, K, L, r_atom, r3, _ptr(params), _ptr(e), _ptr(pa), _ptr(fo),
                    _ptr(st), _ptr(tm))
        if rc:
            raise OracleError(o.error())
        return dict(energy=float(e[0]), per_atom=pa, forces=fo, stress=st, timing=tm)

