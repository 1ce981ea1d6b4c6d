// ORACLE TEST INFRASTRUCTURE -- not part of the product.
//
// extern "C" shim over the UNMODIFIED reference library (graphmd, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load the resulting libgraphmd_ref.so, and only as the
// checker or the timed CPU baseline -- never as the product path.
//
// Every entry point forwards to the reference's public API:
//   Distributed::create_distributed   proj/include/graphmd/engine.hpp:51-56
//   forward_distributed               proj/include/graphmd/potential.hpp:58-60
//   forward_serial                    proj/include/graphmd/potential.hpp:51-53
//   build_neighbor_list / brute force proj/include/graphmd/neighborlist.hpp:37-42
//   serial_line_graph / brute force   proj/include/graphmd/linegraph.hpp:72-78
//   ToyPotentialParams::init          proj/include/graphmd/potential.hpp:35-37
//   make_supercell / random_perturb   proj/include/graphmd/system.hpp:99-105
#include "graphmd/md.hpp"

#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "graphmd/engine.hpp"
#include "graphmd/linegraph.hpp"
#include "graphmd/neighborlist.hpp"
#include "graphmd/partitioner.hpp"
#include "graphmd/potential.hpp"
#include "graphmd/system.hpp"

using namespace graphmd;

namespace {

thread_local std::string g_err;

AtomicSystem make_system(int64_t n, const double* pos, const int32_t* z,
                         const double* lat, const uint8_t* pbc) {
    AtomicSystem s;
    s.positions.resize(n);
    s.species.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        s.positions[i] = Vec3{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        s.species[i] = z[i];
    }
    for (int r = 0; r < 3; ++r)
        s.lattice[r] = Vec3{lat[3 * r], lat[3 * r + 1], lat[3 * r + 2]};
    for (int k = 0; k < 3; ++k) s.pbc[k] = pbc ? pbc[k] != 0 : true;
    return s;
}

ToyPotentialParams make_params(int F, int K, int L, double r_atom, double r3,
                               const double* blob) {
    ToyPotentialParams p;
    p.feature_width = F;
    p.basis_count = K;
    p.layers = L;
    p.r_atom = r_atom;
    p.r_3body = r3;
    const double* q = blob;
    auto take = [&](std::vector<double>& v, size_t n) {
        v.assign(q, q + n);
        q += n;
    };
    take(p.embedding, 119 * (size_t)F);
    take(p.layer_w, (size_t)L * F * F);
    take(p.layer_b, (size_t)L * F);
    take(p.basis_proj, (size_t)F * K);
    take(p.basis3_proj, (size_t)F * K);
    take(p.w3, (size_t)F * F);
    take(p.w4, (size_t)F * F);
    take(p.readout, (size_t)F);
    return p;
}

void put_output(const PotentialOutput& o, double* energy, double* per_atom,
                double* forces, double* stress) {
    if (energy) *energy = o.energy;
    if (per_atom) std::memcpy(per_atom, o.per_atom.data(), o.per_atom.size() * 8);
    if (forces)
        for (size_t i = 0; i < o.forces.size(); ++i) {
            forces[3 * i] = o.forces[i].x;
            forces[3 * i + 1] = o.forces[i].y;
            forces[3 * i + 2] = o.forces[i].z;
        }
    if (stress)
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) stress[3 * a + b] = o.stress[a][b];
}

void put_graph(const AtomGraph& g, int64_t* src, int64_t* dst, int32_t* off,
               double* dist, double* vec) {
    size_t ne = g.num_edges();
    for (size_t e = 0; e < ne; ++e) {
        if (src) src[e] = g.src[e];
        if (dst) dst[e] = g.dst[e];
        if (off)
            for (int k = 0; k < 3; ++k) off[3 * e + k] = g.image_offset[e][k];
        if (dist) dist[e] = g.distance[e];
        if (vec) {
            vec[3 * e] = g.vector[e].x;
            vec[3 * e + 1] = g.vector[e].y;
            vec[3 * e + 2] = g.vector[e].z;
        }
    }
}

struct Handle {
    Distributed dist;
};

struct GraphHandle {
    AtomGraph g;
};

struct PairsHandle {
    std::vector<std::pair<int64_t, int64_t>> v;
};

#define GUARD_BEGIN try {
#define GUARD_END(ret)                   \
    }                                    \
    catch (const std::exception& ex) {   \
        g_err = ex.what();               \
        return ret;                      \
    }

}  // namespace

extern "C" {

const char* gref_last_error() { return g_err.c_str(); }

// ---- Distributed handle ----------------------------------------------------
void* gref_create(int64_t n, const double* pos, const int32_t* z,
                  const double* lat, const uint8_t* pbc, double rc, double r3,
                  double tau, int p, int n_threads, int allow_narrow) {
    GUARD_BEGIN
    AtomicSystem s = make_system(n, pos, z, lat, pbc);
    std::optional<double> tb;
    if (r3 > 0.0) tb = r3;
    auto* h = new Handle{Distributed::create_distributed(
        s, rc, tb, p, n_threads, allow_narrow != 0, tau)};
    return h;
    GUARD_END(nullptr)
}

void gref_destroy(void* h) { delete static_cast<Handle*>(h); }

double gref_create_timed(int64_t n, const double* pos, const int32_t* z,
                         const double* lat, const uint8_t* pbc, double rc,
                         double r3, double tau, int p, int n_threads,
                         int allow_narrow, void** out) {
    auto t0 = std::chrono::steady_clock::now();
    *out = gref_create(n, pos, z, lat, pbc, rc, r3, tau, p, n_threads, allow_narrow);
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
        .count();
}

int64_t gref_num_nodes(void* h) {
    return static_cast<Handle*>(h)->dist.graph().num_nodes;
}
int64_t gref_num_edges(void* h) {
    return (int64_t) static_cast<Handle*>(h)->dist.graph().num_edges();
}
void gref_graph(void* h, int64_t* src, int64_t* dst, int32_t* off, double* dist,
                double* vec) {
    put_graph(static_cast<Handle*>(h)->dist.graph(), src, dst, off, dist, vec);
}
void gref_system(void* h, double* pos, double* lat) {
    const AtomicSystem& s = static_cast<Handle*>(h)->dist.system();
    for (size_t i = 0; i < s.size(); ++i) {
        pos[3 * i] = s.positions[i].x;
        pos[3 * i + 1] = s.positions[i].y;
        pos[3 * i + 2] = s.positions[i].z;
    }
    for (int r = 0; r < 3; ++r) {
        lat[3 * r] = s.lattice[r].x;
        lat[3 * r + 1] = s.lattice[r].y;
        lat[3 * r + 2] = s.lattice[r].z;
    }
}
int gref_rule(void* h, double* boundaries) {
    const PartitionRule& r = static_cast<Handle*>(h)->dist.atom_parts().rule;
    for (int k = 0; k <= r.p; ++k) boundaries[k] = r.boundaries[k];
    return r.axis;
}
void gref_owner(void* h, int32_t* owner) {
    const auto& o = static_cast<Handle*>(h)->dist.atom_parts().owner;
    for (size_t i = 0; i < o.size(); ++i) owner[i] = o[i];
}

static const SpanLayout& layout_of(void* h, int part, int bonds) {
    const Distributed& d = static_cast<Handle*>(h)->dist;
    return bonds ? d.line_parts().parts[part].layout
                 : d.atom_parts().parts[part].layout;
}
int64_t gref_layout_size(void* h, int part, int bonds) {
    return layout_of(h, part, bonds).size();
}
void gref_layout(void* h, int part, int bonds, int64_t* node_array,
                 int64_t* markers) {
    const SpanLayout& l = layout_of(h, part, bonds);
    std::memcpy(node_array, l.node_array.data(), l.node_array.size() * 8);
    std::memcpy(markers, l.markers.data(), l.markers.size() * 8);
}
int64_t gref_num_dups(void* h, int part, int bonds) {
    return (int64_t)layout_of(h, part, bonds).duplicates.size();
}
void gref_dups(void* h, int part, int bonds, int64_t* pairs) {
    const auto& d = layout_of(h, part, bonds).duplicates;
    for (size_t k = 0; k < d.size(); ++k) {
        pairs[2 * k] = d[k].first;
        pairs[2 * k + 1] = d[k].second;
    }
}
int64_t gref_num_owned_edges(void* h, int part) {
    return (int64_t) static_cast<Handle*>(h)
        ->dist.atom_parts()
        .parts[part]
        .owned_edges.size();
}
void gref_owned_edges(void* h, int part, int64_t* owned, int64_t* lsrc,
                      int64_t* ldst) {
    const AtomPartition& a = static_cast<Handle*>(h)->dist.atom_parts().parts[part];
    std::memcpy(owned, a.owned_edges.data(), a.owned_edges.size() * 8);
    std::memcpy(lsrc, a.local_src.data(), a.local_src.size() * 8);
    std::memcpy(ldst, a.local_dst.data(), a.local_dst.size() * 8);
}
int64_t gref_num_border(void* h, int part) {
    return (int64_t) static_cast<Handle*>(h)
        ->dist.atom_parts()
        .parts[part]
        .border_edge_list.size();
}
void gref_border(void* h, int part, int64_t* out) {
    const auto& b =
        static_cast<Handle*>(h)->dist.atom_parts().parts[part].border_edge_list;
    std::memcpy(out, b.data(), b.size() * 8);
}
int gref_has_line_graph(void* h) {
    return static_cast<Handle*>(h)->dist.has_line_graph() ? 1 : 0;
}
int64_t gref_num_bonds(void* h) {
    return (int64_t) static_cast<Handle*>(h)->dist.line_parts().bonds.size();
}
void gref_bonds(void* h, int64_t* edge_of_bond, int32_t* bond_owner) {
    const PartitionedLineGraph& lg = static_cast<Handle*>(h)->dist.line_parts();
    for (size_t b = 0; b < lg.bonds.size(); ++b) {
        edge_of_bond[b] = lg.bonds.edge_of_bond[b];
        bond_owner[b] = lg.bond_owner[b];
    }
}
int64_t gref_num_line_edges(void* h, int part) {
    return (int64_t) static_cast<Handle*>(h)
        ->dist.line_parts()
        .parts[part]
        .line_edges.size();
}
void gref_line_edges(void* h, int part, int64_t* pairs) {
    const auto& le =
        static_cast<Handle*>(h)->dist.line_parts().parts[part].line_edges;
    for (size_t k = 0; k < le.size(); ++k) {
        pairs[2 * k] = le[k].first;
        pairs[2 * k + 1] = le[k].second;
    }
}

int gref_forward(void* h, int F, int K, int L, double r_atom, double r3,
                 const double* blob, double* energy, double* per_atom,
                 double* forces, double* stress, double* timing4) {
    GUARD_BEGIN
    ToyPotentialParams p = make_params(F, K, L, r_atom, r3, blob);
    StepTiming t;
    PotentialOutput o = forward_distributed(static_cast<Handle*>(h)->dist, p, &t);
    put_output(o, energy, per_atom, forces, stress);
    if (timing4) {
        timing4[0] = t.graph_creation;
        timing4[1] = t.feature_calculation;
        timing4[2] = t.forward_pass;
        timing4[3] = t.backward_pass;
    }
    return 0;
    GUARD_END(1)
}

// ---- stateless helpers -----------------------------------------------------
int gref_forward_serial(int64_t n, const double* pos, const int32_t* z,
                        const double* lat, const uint8_t* pbc, int F, int K,
                        int L, double r_atom, double r3, const double* blob,
                        double* energy, double* per_atom, double* forces,
                        double* stress) {
    GUARD_BEGIN
    ToyPotentialParams p = make_params(F, K, L, r_atom, r3, blob);
    PotentialOutput o = forward_serial(make_system(n, pos, z, lat, pbc), p, 1);
    put_output(o, energy, per_atom, forces, stress);
    return 0;
    GUARD_END(1)
}

void gref_params_init(uint64_t seed, int F, int K, int L, double r_atom,
                      double r3, double* blob) {
    ToyPotentialParams p = ToyPotentialParams::init(seed, F, K, L, r_atom, r3);
    double* q = blob;
    for (const auto* v : {&p.embedding, &p.layer_w, &p.layer_b, &p.basis_proj,
                          &p.basis3_proj, &p.w3, &p.w4, &p.readout}) {
        std::memcpy(q, v->data(), v->size() * 8);
        q += v->size();
    }
}

// make_supercell followed by random_perturb (amp <= 0 skips the perturbation)
void gref_supercell(int64_t n, const double* pos, const int32_t* z,
                    const double* lat, int rx, int ry, int rz, double amp,
                    uint64_t seed, double* out_pos, int32_t* out_z,
                    double* out_lat) {
    AtomicSystem s = make_system(n, pos, z, lat, nullptr);
    AtomicSystem big = make_supercell(s, {rx, ry, rz});
    if (amp > 0.0) big = random_perturb(big, amp, seed);
    for (size_t i = 0; i < big.size(); ++i) {
        out_pos[3 * i] = big.positions[i].x;
        out_pos[3 * i + 1] = big.positions[i].y;
        out_pos[3 * i + 2] = big.positions[i].z;
        out_z[i] = big.species[i];
    }
    for (int r = 0; r < 3; ++r) {
        out_lat[3 * r] = big.lattice[r].x;
        out_lat[3 * r + 1] = big.lattice[r].y;
        out_lat[3 * r + 2] = big.lattice[r].z;
    }
}

// Rng(seed).uniform(lo, hi) stream (system.hpp:121-149)
void gref_rng_uniform(uint64_t seed, int64_t count, double lo, double hi,
                      double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = r.uniform(lo, hi);
}
void gref_rng_normal(uint64_t seed, int64_t count, double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = r.normal();
}

void* gref_neighbor_list(int64_t n, const double* pos, const int32_t* z,
                         const double* lat, const uint8_t* pbc, double rc,
                         int brute, int n_threads) {
    GUARD_BEGIN
    AtomicSystem s = make_system(n, pos, z, lat, pbc);
    auto* g = new GraphHandle{brute ? brute_force_neighbor_list(s, rc)
                                    : build_neighbor_list(s, rc, n_threads)};
    return g;
    GUARD_END(nullptr)
}
int64_t gref_graph_num_edges(void* g) {
    return (int64_t) static_cast<GraphHandle*>(g)->g.num_edges();
}
void gref_graph_get(void* g, int64_t* src, int64_t* dst, int32_t* off,
                    double* dist, double* vec) {
    put_graph(static_cast<GraphHandle*>(g)->g, src, dst, off, dist, vec);
}
void gref_graph_destroy(void* g) { delete static_cast<GraphHandle*>(g); }

// serial_line_graph (brute=0) or brute_force_line_graph (brute=1) as pairs of
// global edge ids, sorted.
void* gref_line_graph(int64_t n, const double* pos, const int32_t* z,
                      const double* lat, const uint8_t* pbc, double rc, double r,
                      double tau, int brute) {
    GUARD_BEGIN
    AtomicSystem s = make_system(n, pos, z, lat, pbc);
    AtomGraph g = build_neighbor_list(s, rc, 1);
    auto* ph = new PairsHandle{brute ? brute_force_line_graph(g, r, tau)
                                     : serial_line_graph(g, r, tau)};
    return ph;
    GUARD_END(nullptr)
}
int64_t gref_pairs_size(void* ph) {
    return (int64_t) static_cast<PairsHandle*>(ph)->v.size();
}
void gref_pairs_get(void* ph, int64_t* out) {
    const auto& v = static_cast<PairsHandle*>(ph)->v;
    for (size_t k = 0; k < v.size(); ++k) {
        out[2 * k] = v[k].first;
        out[2 * k + 1] = v[k].second;
    }
}
void gref_pairs_destroy(void* ph) { delete static_cast<PairsHandle*>(ph); }

int gref_fd_forces(int64_t n, const double* pos, const int32_t* z,
                   const double* lat, const uint8_t* pbc, int F, int K, int L,
                   double r_atom, double r3, const double* blob, double eps,
                   double* forces) {
    GUARD_BEGIN
    ToyPotentialParams p = make_params(F, K, L, r_atom, r3, blob);
    auto f = finite_difference_forces(make_system(n, pos, z, lat, pbc), p, eps);
    for (size_t i = 0; i < f.size(); ++i) {
        forces[3 * i] = f[i].x;
        forces[3 * i + 1] = f[i].y;
        forces[3 * i + 2] = f[i].z;
    }
    return 0;
    GUARD_END(1)
}

// run_md (md.cpp:112-160) with the given options; final state + records
// rec[(steps + 1) x 4] = (potential, kinetic, total, max_force)
int gref_md_run(int64_t n, const double* pos, const int32_t* z, const double* lat,
                const uint8_t* pbc, int F, int K, int L, double r_atom, double r3,
                const double* blob, double dt, int64_t steps, int partitions,
                double temperature, uint64_t seed, double* out_pos, double* out_vel,
                double* out_forces, double* rec) {
    GUARD_BEGIN
    ToyPotentialParams p = make_params(F, K, L, r_atom, r3, blob);
    MDOptions o;
    o.dt = dt;
    o.steps = steps;
    o.partitions = partitions;
    o.threads = 1;
    o.allow_narrow = true;
    o.seed = seed;
    o.init_temperature = temperature;
    MDResult r = run_md(make_system(n, pos, z, lat, pbc), p, o);
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            out_pos[3 * i + k] = r.state.system.positions[i][k];
            out_vel[3 * i + k] = r.state.velocities[i][k];
            out_forces[3 * i + k] = r.state.forces[i][k];
        }
    for (size_t s = 0; s < r.records.size(); ++s) {
        rec[4 * s] = r.records[s].potential;
        rec[4 * s + 1] = r.records[s].kinetic;
        rec[4 * s + 2] = r.records[s].total;
        rec[4 * s + 3] = r.records[s].max_force;
    }
    return 0;
    GUARD_END(1)
}

// the reference's own dump formats (neighborlist.cpp:97-106,
// linegraph.cpp:173-181, partitioner.cpp:220-236)
int gref_dump_graph(void* h, const char* path) {
    GUARD_BEGIN
    static_cast<Handle*>(h)->dist.graph().dump_csv(path);
    return 0;
    GUARD_END(1)
}
int gref_dump_line(void* h, const char* path) {
    GUARD_BEGIN
    static_cast<Handle*>(h)->dist.line_parts().dump_csv(path);
    return 0;
    GUARD_END(1)
}
int64_t gref_plan_json(void* h, char* buf, int64_t cap) {
    std::string js;
    try {
        js = partition_plan_to_json(static_cast<Handle*>(h)->dist.atom_parts());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
    if ((int64_t)js.size() < cap) std::memcpy(buf, js.c_str(), js.size() + 1);
    return (int64_t)js.size();
}

// parameter files (potential.cpp:178-260)
int gref_params_save(int F, int K, int L, double r_atom, double r3, uint64_t seed,
                     const double* blob, const char* path) {
    GUARD_BEGIN
    ToyPotentialParams p = make_params(F, K, L, r_atom, r3, blob);
    p.seed = seed;
    p.save(path);
    return 0;
    GUARD_END(1)
}
// returns the blob length (or -1); hdr = F, K, L; r = r_atom, r_3body
int64_t gref_params_load(const char* path, int32_t* hdr, double* r, uint64_t* seed, double* blob,
                         int64_t cap) {
    try {
        ToyPotentialParams p = ToyPotentialParams::load(path);
        std::vector<double> b;
        for (const auto* v : {&p.embedding, &p.layer_w, &p.layer_b, &p.basis_proj, &p.basis3_proj,
                              &p.w3, &p.w4, &p.readout})
            b.insert(b.end(), v->begin(), v->end());
        hdr[0] = p.feature_width;
        hdr[1] = p.basis_count;
        hdr[2] = p.layers;
        r[0] = p.r_atom;
        r[1] = p.r_3body;
        *seed = p.seed;
        if ((int64_t)b.size() <= cap) std::memcpy(blob, b.data(), b.size() * sizeof(double));
        return (int64_t)b.size();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// extended-XYZ I/O (system.cpp:95-186)
int gref_save_xyz(int64_t n, const double* pos, const int32_t* z, const double* lat,
                  const uint8_t* pbc, const char* path, const char* comment) {
    GUARD_BEGIN
    save_xyz(make_system(n, pos, z, lat, pbc), path, comment ? comment : "");
    return 0;
    GUARD_END(1)
}
// n = atom count or -1 (error text in gref_last_error); when pos != null the
// system is copied out (pos n x 3, z n, lat 9, pbc 3)
int64_t gref_load_xyz(const char* path, double* pos, int32_t* z, double* lat, uint8_t* pbc) {
    try {
        AtomicSystem s = load_xyz(path);
        const int64_t n = (int64_t)s.size();
        if (pos) {
            for (int64_t i = 0; i < n; ++i) {
                for (int k = 0; k < 3; ++k) pos[3 * i + k] = s.positions[i][k];
                z[i] = s.species[i];
            }
            for (int r = 0; r < 3; ++r)
                for (int k = 0; k < 3; ++k) lat[3 * r + k] = s.lattice[r][k];
            for (int k = 0; k < 3; ++k) pbc[k] = s.pbc[k] ? 1 : 0;
        }
        return n;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
