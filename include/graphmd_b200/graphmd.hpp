// graphmd_b200/graphmd.hpp -- C++ drop-in for the reference's plugin API.
//
// Callers of the reference (md.cpp, graphmd_cli, tests) include this header
// instead of <graphmd/engine.hpp> + <graphmd/potential.hpp> and link
// libgraphmd_b200.so; the names, argument meanings and the Error type are the
// reference's (proj/include/graphmd/{system,neighborlist,partitioner,
// linegraph,engine,potential}.hpp), the work runs on the GPU through the C ABI
// in graphmd_b200.h.  Views (graph(), atom_parts(), line_parts()) are
// materialized from device data on first use.
#pragma once

#include <algorithm>
#include <array>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <unordered_map>
#include <vector>

#include "../graphmd_b200.h"

namespace graphmd {

// ---- errors (system.hpp:13-15) -----------------------------------------
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};

namespace detail {
inline void check(const gmd_handle* h, int rc) {
    if (rc != GMD_OK) throw Error(gmd_last_error(h));
}
}  // namespace detail

// ---- geometry (system.hpp:17-94) -----------------------------------------
struct Vec3 {
    double x = 0, y = 0, z = 0;
    Vec3() = default;
    Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
    double& operator[](int i) { return i == 0 ? x : i == 1 ? y : z; }
    double operator[](int i) const { return i == 0 ? x : i == 1 ? y : z; }
    Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
    Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
    Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
    Vec3 operator/(double s) const { return {x / s, y / s, z / s}; }
    Vec3 operator-() const { return {-x, -y, -z}; }
    Vec3& operator+=(const Vec3& o) { return *this = *this + o; }
    Vec3& operator-=(const Vec3& o) { return *this = *this - o; }
    Vec3& operator*=(double s) { return *this = *this * s; }
    double dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
    Vec3 cross(const Vec3& o) const {
        return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x};
    }
    double norm2() const { return dot(*this); }
    double norm() const { return std::sqrt(norm2()); }
};
inline Vec3 operator*(double s, const Vec3& v) { return v * s; }

struct Mat3 {
    std::array<Vec3, 3> rows{};
    Vec3& operator[](int i) { return rows[i]; }
    const Vec3& operator[](int i) const { return rows[i]; }
    double det() const { return rows[0].dot(rows[1].cross(rows[2])); }
    Vec3 rowvec_mul(const Vec3& v) const { return rows[0] * v.x + rows[1] * v.y + rows[2] * v.z; }
    static Mat3 identity() {
        Mat3 m;
        m.rows = {Vec3{1, 0, 0}, Vec3{0, 1, 0}, Vec3{0, 0, 1}};
        return m;
    }
    // system.cpp:55-70 operand order (columns of the inverse are (b x c) / d, ...)
    Mat3 inverse() const {
        const double d = det();
        if (std::abs(d) < 1e-10) throw Error("lattice is singular (|det| < 1e-10)");
        const Vec3 bc = rows[1].cross(rows[2]) / d, ca = rows[2].cross(rows[0]) / d,
                   ab = rows[0].cross(rows[1]) / d;
        Mat3 inv;
        inv.rows = {Vec3{bc.x, ca.x, ab.x}, Vec3{bc.y, ca.y, ab.y}, Vec3{bc.z, ca.z, ab.z}};
        return inv;
    }
};

struct FractionalCoords {
    std::vector<Vec3> coords;
};

struct AtomicSystem {
    std::vector<Vec3> positions;
    Mat3 lattice = Mat3::identity();
    std::vector<int> species;
    std::array<bool, 3> pbc{true, true, true};
    std::size_t size() const { return positions.size(); }
    bool any_pbc() const { return pbc[0] || pbc[1] || pbc[2]; }
    void validate() const {
        if (species.size() != positions.size()) throw Error("species length does not match atom count");
        if (any_pbc() && std::abs(lattice.det()) < 1e-10)
            throw Error("periodic system requires an invertible lattice");
    }
    FractionalCoords fractional() const {  // f = r L^-1 (system.cpp:79-85)
        const Mat3 inv = lattice.inverse();
        FractionalCoords f;
        f.coords.reserve(positions.size());
        for (const Vec3& r : positions) f.coords.push_back(inv.rowvec_mul(r));
        return f;
    }
    double perpendicular_width(int axis) const {  // |det| / |b x c| (system.cpp:87-93)
        const double area = lattice[(axis + 1) % 3].cross(lattice[(axis + 2) % 3]).norm();
        if (area <= 0.0) throw Error("degenerate cell");
        return std::abs(lattice.det()) / area;
    }
};

// Rng (system.hpp:121-149): mt19937_64, uniform = (u64 >> 11) 2^-53,
// Box-Muller normals with a cached spare -- the reference's streams exactly
class Rng {
public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = 0.0;
        while (u1 == 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * M_PI * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
        return r * std::cos(a);
    }
    std::uint64_t next_u64() { return gen_(); }

private:
    std::mt19937_64 gen_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

// wrap_positions (system.cpp:215-229): positions folded into the cell
inline AtomicSystem wrap_positions(const AtomicSystem& system) {
    system.validate();
    AtomicSystem out = system;
    const FractionalCoords f = system.fractional();
    for (std::size_t i = 0; i < out.size(); ++i) {
        Vec3 fr = f.coords[i];
        for (int k = 0; k < 3; ++k) {
            fr[k] -= std::floor(fr[k]);
            if (fr[k] >= 1.0) fr[k] = 0.0;
        }
        out.positions[i] = out.lattice.rowvec_mul(fr);
    }
    return out;
}

// make_supercell + random_perturb on the library's host RNG (system.cpp:188-240)
inline AtomicSystem make_supercell(const AtomicSystem& s, const std::array<int, 3>& reps,
                                   double amplitude = 0.0, std::uint64_t seed = 0) {
    const std::size_t n = s.size(), f = (std::size_t)reps[0] * reps[1] * reps[2];
    std::vector<double> pos(3 * n), lat(9), opos(3 * n * f), olat(9);
    std::vector<int32_t> z(s.species.begin(), s.species.end()), oz(n * f);
    for (std::size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) pos[3 * i + k] = s.positions[i][k];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) lat[3 * r + k] = s.lattice[r][k];
    int rc = gmd_util_supercell((int64_t)n, pos.data(), z.data(), lat.data(), reps[0], reps[1],
                                reps[2], amplitude, seed, opos.data(), oz.data(), olat.data());
    if (rc != GMD_OK) throw Error("supercell repetitions must be >= 1");
    AtomicSystem o;
    o.pbc = s.pbc;
    o.positions.resize(n * f);
    o.species.assign(oz.begin(), oz.end());
    for (std::size_t i = 0; i < n * f; ++i) o.positions[i] = {opos[3 * i], opos[3 * i + 1], opos[3 * i + 2]};
    for (int r = 0; r < 3; ++r) o.lattice[r] = {olat[3 * r], olat[3 * r + 1], olat[3 * r + 2]};
    return o;
}
inline AtomicSystem random_perturb(const AtomicSystem& s, double amplitude, std::uint64_t seed) {
    if (amplitude < 0.0) throw Error("perturbation amplitude must be >= 0");
    return make_supercell(s, {1, 1, 1}, amplitude, seed);
}

// ---- extended-XYZ I/O (system.cpp:95-186, docs/formats.md) ----------------
namespace detail {
inline const char* const* element_symbols() {  // index = atomic number, 0 = "X"
    static const char* const s[119] = {
        "X",  "H",  "He", "Li", "Be", "B",  "C",  "N",  "O",  "F",  "Ne", "Na", "Mg", "Al", "Si",
        "P",  "S",  "Cl", "Ar", "K",  "Ca", "Sc", "Ti", "V",  "Cr", "Mn", "Fe", "Co", "Ni", "Cu",
        "Zn", "Ga", "Ge", "As", "Se", "Br", "Kr", "Rb", "Sr", "Y",  "Zr", "Nb", "Mo", "Tc", "Ru",
        "Rh", "Pd", "Ag", "Cd", "In", "Sn", "Sb", "Te", "I",  "Xe", "Cs", "Ba", "La", "Ce", "Pr",
        "Nd", "Pm", "Sm", "Eu", "Gd", "Tb", "Dy", "Ho", "Er", "Tm", "Yb", "Lu", "Hf", "Ta", "W",
        "Re", "Os", "Ir", "Pt", "Au", "Hg", "Tl", "Pb", "Bi", "Po", "At", "Rn", "Fr", "Ra", "Ac",
        "Th", "Pa", "U",  "Np", "Pu", "Am", "Cm", "Bk", "Cf", "Es", "Fm", "Md", "No", "Lr", "Rf",
        "Db", "Sg", "Bh", "Hs", "Mt", "Ds", "Rg", "Cn", "Nh", "Fl", "Mc", "Lv", "Ts", "Og"};
    return s;
}
[[noreturn]] inline void parse_fail(const std::string& path, int line, const std::string& what) {
    throw Error(path + ":" + std::to_string(line) + ": " + what);
}
}  // namespace detail

inline const std::string& z_to_symbol(int z) {
    static const std::vector<std::string> cache(detail::element_symbols(), detail::element_symbols() + 119);
    if (z < 1 || z > 118) throw Error("atomic number out of range");
    return cache[z];
}

// load_xyz: atom count, comment line with Lattice="..." (and optional
// pbc="T T F"), then `Symbol x y z` lines
inline AtomicSystem load_xyz(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open file: " + path);
    std::string line;
    if (!std::getline(in, line)) detail::parse_fail(path, 1, "empty file");
    std::size_t natoms = 0;
    try {
        natoms = std::stoul(line);
    } catch (...) {
        detail::parse_fail(path, 1, "expected atom count, got '" + line + "'");
    }
    if (!std::getline(in, line)) detail::parse_fail(path, 2, "missing comment line");
    AtomicSystem sys;
    const auto lat = line.find("Lattice=\"");
    const bool have_lattice = lat != std::string::npos;
    if (have_lattice) {
        const auto b = lat + 9, e = line.find('"', b);
        if (e == std::string::npos) detail::parse_fail(path, 2, "unterminated Lattice field");
        std::istringstream ls(line.substr(b, e - b));
        double v[9];
        for (double& x : v)
            if (!(ls >> x)) detail::parse_fail(path, 2, "Lattice needs 9 numbers");
        for (int r = 0; r < 3; ++r) sys.lattice[r] = {v[3 * r], v[3 * r + 1], v[3 * r + 2]};
    }
    const auto pb = line.find("pbc=\"");
    if (pb != std::string::npos) {
        const auto b = pb + 5, e = line.find('"', b);
        std::istringstream ps(line.substr(b, e == std::string::npos ? std::string::npos : e - b));
        std::string tok;
        for (int k = 0; k < 3; ++k) {
            if (!(ps >> tok)) detail::parse_fail(path, 2, "pbc needs 3 flags");
            sys.pbc[k] = tok == "T" || tok == "True" || tok == "true" || tok == "1";
        }
    }
    if (!have_lattice) {
        if (sys.any_pbc()) detail::parse_fail(path, 2, "periodic system requires a Lattice field");
        sys.lattice = Mat3::identity();
    }
    const char* const* sym = detail::element_symbols();
    for (std::size_t i = 0; i < natoms; ++i) {
        const int lineno = (int)i + 3;
        if (!std::getline(in, line)) detail::parse_fail(path, lineno, "unexpected end of file");
        std::istringstream as(line);
        std::string s;
        double x, y, z;
        if (!(as >> s >> x >> y >> z)) detail::parse_fail(path, lineno, "expected 'symbol x y z'");
        int zz = 0;
        for (int k = 1; k <= 118 && !zz; ++k)
            if (s == sym[k]) zz = k;
        if (!zz) detail::parse_fail(path, lineno, "unknown element symbol '" + s + "'");
        sys.species.push_back(zz);
        sys.positions.push_back({x, y, z});
    }
    sys.validate();
    return sys;
}

// save_xyz: 17 significant digits (round-trips every double)
inline void save_xyz(const AtomicSystem& system, const std::string& path,
                     const std::string& comment_extra = "") {
    std::ofstream out(path);
    if (!out) throw Error("cannot write file: " + path);
    out.precision(17);
    out << system.size() << "\n";
    out << "Lattice=\"";
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) out << system.lattice[i][k] << (i == 2 && k == 2 ? "" : " ");
    out << "\" pbc=\"" << (system.pbc[0] ? "T" : "F") << " " << (system.pbc[1] ? "T" : "F") << " "
        << (system.pbc[2] ? "T" : "F") << "\"";
    if (!comment_extra.empty()) out << " " << comment_extra;
    out << "\n";
    for (std::size_t i = 0; i < system.size(); ++i) {
        const Vec3& r = system.positions[i];
        out << z_to_symbol(system.species[i]) << " " << r.x << " " << r.y << " " << r.z << "\n";
    }
}

// ---- graph / partition / line-graph views -----------------------------
using Offset3 = std::array<int, 3>;

struct AtomGraph {  // neighborlist.hpp:17-33
    std::vector<std::int64_t> src, dst;
    std::vector<Offset3> image_offset;
    std::vector<double> distance;
    std::vector<Vec3> vector;
    double cutoff = 0.0;
    std::int64_t num_nodes = 0;
    std::size_t num_edges() const { return src.size(); }
    std::pair<std::size_t, std::size_t> edges_into(std::int64_t node) const {
        std::size_t lo = 0, hi = dst.size();
        while (lo < hi) {
            std::size_t m = (lo + hi) / 2;
            if (dst[m] < node) lo = m + 1; else hi = m;
        }
        std::size_t e = lo;
        while (e < dst.size() && dst[e] == node) ++e;
        return {lo, e};
    }
    // neighborlist.cpp:97-106
    void dump_csv(const std::string& path) const {
        std::ofstream out(path);
        if (!out) throw Error("cannot write file: " + path);
        out.precision(17);
        out << "src,dst,ox,oy,oz,distance\n";
        for (std::size_t e = 0; e < num_edges(); ++e)
            out << src[e] << "," << dst[e] << "," << image_offset[e][0] << ","
                << image_offset[e][1] << "," << image_offset[e][2] << "," << distance[e] << "\n";
    }
};

struct PartitionRule {  // partitioner.hpp:16-20
    int axis = 0;
    std::vector<double> boundaries;
    int p = 1;
};
enum class BoundaryMode { kQuantile, kEqualWidth };

struct Buckets {
    std::vector<std::vector<std::int64_t>> pure;
    std::vector<std::vector<std::vector<std::int64_t>>> to, from;
};

struct Span {
    std::int64_t begin = 0, end = 0;
    std::int64_t size() const { return end - begin; }
};

struct SpanLayout {  // partitioner.hpp:45-63
    std::vector<std::int64_t> node_array;
    std::vector<std::int64_t> markers;
    std::unordered_map<std::int64_t, std::int64_t> global_to_local;  // canonical (first) row
    std::vector<std::pair<std::int64_t, std::int64_t>> duplicates;
    int p = 1;
    Span pure_span() const { return {markers[0], markers[1]}; }
    Span to_span(int j) const { return {markers[1 + j], markers[2 + j]}; }
    Span from_span(int j) const { return {markers[1 + p + j], markers[2 + p + j]}; }
    std::int64_t owned_end() const { return markers[1 + p]; }
    std::int64_t size() const { return (std::int64_t)node_array.size(); }
    std::int64_t local_of(std::int64_t g) const {
        auto it = global_to_local.find(g);
        return it == global_to_local.end() ? -1 : it->second;
    }
};

struct AtomPartition {
    SpanLayout layout;
    std::vector<std::int64_t> owned_edges, local_src, local_dst, border_edge_list;
};

struct PartitionedAtomGraph {
    PartitionRule rule;
    Buckets buckets;
    std::vector<int> owner;
    std::vector<AtomPartition> parts;
    int p = 1;
};

struct BondSet {  // linegraph.hpp:15-24
    std::vector<std::int64_t> edge_of_bond, bond_of_edge;
    std::vector<std::vector<std::int64_t>> by_src, by_dst;  // atom -> bond ids (ascending)
    double r = 0.0, tau = 0.0;
    std::size_t size() const { return edge_of_bond.size(); }
};

struct LineGraphPartition {
    SpanLayout layout;
    std::vector<std::pair<std::int64_t, std::int64_t>> line_edges;
};

// linegraph.hpp:31-37: per-partition tables (node -> bond ids with both ends
// in the partition's two-hop closure), bond owners and bond buckets
struct EdgeTables {
    BondSet bonds;
    std::vector<std::unordered_map<std::int64_t, std::vector<std::int64_t>>> per_partition;
    std::vector<int> bond_owner;
    Buckets bond_buckets;
};

struct PartitionedLineGraph {
    BondSet bonds;
    std::vector<int> bond_owner;
    Buckets bond_buckets;
    std::vector<LineGraphPartition> parts;
    int p = 1;
    // linegraph.cpp:173-181
    void dump_csv(const std::string& path) const {
        std::ofstream out(path);
        if (!out) throw Error("cannot write file: " + path);
        out << "partition,bond_e_global,bond_ep_global\n";
        for (int i = 0; i < p; ++i)
            for (const auto& [le, lep] : parts[i].line_edges)
                out << i << "," << parts[i].layout.node_array[le] << ","
                    << parts[i].layout.node_array[lep] << "\n";
    }
};

namespace detail {
// ---- views of a built handle (gmd_build or gmd_build_partitions) ----------
inline SpanLayout read_layout(gmd_handle* h, int p, int i, int bonds) {
    SpanLayout L;
    L.p = p;
    int64_t sz = 0, nd = 0;
    check(h, gmd_get_layout_size(h, i, bonds, &sz));
    L.node_array.resize(sz);
    L.markers.resize(2 + 2 * p);
    check(h, gmd_get_layout(h, i, bonds, L.node_array.data(), L.markers.data()));
    check(h, gmd_get_num_duplicates(h, i, bonds, &nd));
    std::vector<int64_t> d(2 * nd);
    check(h, gmd_get_duplicates(h, i, bonds, d.data()));
    for (int64_t k = 0; k < nd; ++k) L.duplicates.emplace_back(d[2 * k], d[2 * k + 1]);
    L.global_to_local.reserve(L.node_array.size() * 2);
    for (std::size_t r = 0; r < L.node_array.size(); ++r) L.global_to_local.emplace(L.node_array[r], (std::int64_t)r);
    return L;
}

// PURE / TO / FROM lists are the layout's spans (build_span_layout order)
inline Buckets buckets_of(const std::vector<const SpanLayout*>& lays) {
    const int p = (int)lays.size();
    Buckets b;
    b.pure.resize(p);
    b.to.assign(p, std::vector<std::vector<std::int64_t>>(p));
    b.from.assign(p, std::vector<std::vector<std::int64_t>>(p));
    for (int i = 0; i < p; ++i) {
        const SpanLayout& L = *lays[i];
        Span s = L.pure_span();
        b.pure[i].assign(L.node_array.begin() + s.begin, L.node_array.begin() + s.end);
        for (int j = 0; j < p; ++j) {
            Span t = L.to_span(j);
            b.to[i][j].assign(L.node_array.begin() + t.begin, L.node_array.begin() + t.end);
        }
    }
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) b.from[j][i] = b.to[i][j];
    return b;
}

inline PartitionedAtomGraph read_atom_parts(gmd_handle* h, int p) {
    PartitionedAtomGraph pg;
    pg.p = p;
    pg.rule.p = p;
    pg.rule.boundaries.resize(p + 1);
    check(h, gmd_get_rule(h, &pg.rule.axis, pg.rule.boundaries.data()));
    int64_t n = 0;
    gmd_num_nodes(h, &n);
    std::vector<int32_t> own(n);
    check(h, gmd_get_owner(h, own.data()));
    pg.owner.assign(own.begin(), own.end());
    std::vector<const SpanLayout*> lays;
    pg.parts.reserve(p);
    for (int i = 0; i < p; ++i) {
        AtomPartition ap;
        ap.layout = read_layout(h, p, i, 0);
        int64_t c = 0;
        check(h, gmd_get_num_owned_edges(h, i, &c));
        ap.owned_edges.resize(c);
        ap.local_src.resize(c);
        ap.local_dst.resize(c);
        check(h, gmd_get_owned_edges(h, i, ap.owned_edges.data(), ap.local_src.data(), ap.local_dst.data()));
        check(h, gmd_get_num_border_edges(h, i, &c));
        ap.border_edge_list.resize(c);
        check(h, gmd_get_border_edges(h, i, ap.border_edge_list.data()));
        pg.parts.push_back(std::move(ap));
    }
    for (const auto& ap : pg.parts) lays.push_back(&ap.layout);
    pg.buckets = buckets_of(lays);
    return pg;
}

// BondSet with by_src / by_dst lists (linegraph.cpp:25-43 order: ascending bond id)
inline BondSet read_bonds(gmd_handle* h, double r, double tau, std::vector<int>* owner) {
    BondSet bs;
    int64_t nb = 0, ne = 0, n = 0;
    check(h, gmd_get_num_bonds(h, &nb));
    gmd_num_edges(h, &ne);
    gmd_num_nodes(h, &n);
    bs.edge_of_bond.resize(nb);
    std::vector<int32_t> own(nb);
    check(h, gmd_get_bonds(h, bs.edge_of_bond.data(), own.data()));
    if (owner) owner->assign(own.begin(), own.end());
    bs.bond_of_edge.assign(ne, -1);
    for (int64_t b = 0; b < nb; ++b) bs.bond_of_edge[bs.edge_of_bond[b]] = b;
    bs.r = r;
    bs.tau = tau;
    bs.by_src.assign(n, {});
    bs.by_dst.assign(n, {});
    if (nb) {
        std::vector<int32_t> row(n + 1), src(ne);
        check(h, gmd_get_csr(h, row.data(), src.data()));
        std::vector<int32_t> dst_of(ne);
        for (int64_t v = 0; v < n; ++v)
            for (int32_t e = row[v]; e < row[v + 1]; ++e) dst_of[e] = (int32_t)v;
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t e = bs.edge_of_bond[b];
            bs.by_src[src[e]].push_back(b);
            bs.by_dst[dst_of[e]].push_back(b);
        }
    }
    return bs;
}

inline PartitionedLineGraph read_line_parts(gmd_handle* h, int p, double r, double tau) {
    PartitionedLineGraph lg;
    lg.p = p;
    lg.bonds = read_bonds(h, r, tau, &lg.bond_owner);
    std::vector<const SpanLayout*> lays;
    lg.parts.reserve(p);
    for (int i = 0; i < p; ++i) {
        LineGraphPartition part;
        part.layout = read_layout(h, p, i, 1);
        int64_t c = 0;
        check(h, gmd_get_num_line_edges(h, i, &c));
        std::vector<int64_t> pairs(2 * c);
        check(h, gmd_get_line_edges(h, i, pairs.data()));
        part.line_edges.resize(c);
        for (int64_t k = 0; k < c; ++k) part.line_edges[k] = {pairs[2 * k], pairs[2 * k + 1]};
        lg.parts.push_back(std::move(part));
    }
    for (const auto& pt : lg.parts) lays.push_back(&pt.layout);
    lg.bond_buckets = buckets_of(lays);
    return lg;
}
}  // namespace detail

namespace detail {
// the reference's JSON layout with dump(2): sorted keys, two-space indent,
// integer arrays inline, other arrays one element per line
inline std::string json_ints(const std::vector<std::int64_t>& v) {
    std::string s = "[";
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    return s + "]";
}
inline std::string json_lines(const std::vector<std::string>& items, int ind) {
    if (items.empty()) return "[]";
    std::string pad(2 * ind, ' '), pad1(2 * ind + 2, ' '), s = "[\n";
    for (std::size_t i = 0; i < items.size(); ++i) s += pad1 + items[i] + (i + 1 < items.size() ? ",\n" : "\n");
    return s + pad + "]";
}
inline std::string json_double(double x) {  // shortest round-trip, ".0" for integral values
    char buf[32];
    for (int prec = 1; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, x);
        if (std::strtod(buf, nullptr) == x) break;
    }
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}
}  // namespace detail

// partitioner.cpp:220-236
inline std::string partition_plan_to_json(const PartitionedAtomGraph& parts) {
    using detail::json_ints;
    using detail::json_lines;
    auto nested = [](const std::vector<std::vector<std::int64_t>>& v, int ind) {
        std::vector<std::string> it;
        for (const auto& x : v) it.push_back(json_ints(x));
        return json_lines(it, ind);
    };
    auto nested2 = [&](const std::vector<std::vector<std::vector<std::int64_t>>>& v) {
        std::vector<std::string> it;
        for (const auto& x : v) it.push_back(nested(x, 2));
        return json_lines(it, 1);
    };
    std::vector<std::string> b, pj;
    for (double x : parts.rule.boundaries) b.push_back(detail::json_double(x));
    for (const AtomPartition& part : parts.parts)
        pj.push_back("{\n      \"markers\": " + json_ints(part.layout.markers) +
                     ",\n      \"node_array\": " + json_ints(part.layout.node_array) +
                     ",\n      \"owned_edge_count\": " + std::to_string(part.owned_edges.size()) +
                     "\n    }");
    return "{\n  \"axis\": " + std::to_string(parts.rule.axis) + ",\n  \"boundaries\": " +
           json_lines(b, 1) + ",\n  \"from\": " + nested2(parts.buckets.from) +
           ",\n  \"p\": " + std::to_string(parts.p) + ",\n  \"partitions\": " + json_lines(pj, 1) +
           ",\n  \"pure\": " + nested(parts.buckets.pure, 1) + ",\n  \"to\": " +
           nested2(parts.buckets.to) + "\n}";
}

// ---- engine (engine.hpp:18-151) -----------------------------------------
struct DistributedFeatures {
    std::vector<std::vector<double>> blocks;
    std::int64_t width = 0;
    double* row(int part, std::int64_t local) { return blocks[part].data() + local * width; }
    const double* row(int part, std::int64_t local) const { return blocks[part].data() + local * width; }
};

struct StepTiming {
    double graph_creation = 0, feature_calculation = 0, forward_pass = 0, backward_pass = 0;
    static const std::vector<std::string>& category_names() {
        static const std::vector<std::string> n = {"Graph Creation", "Feature Calculation",
                                                   "Forward Pass", "Backward Pass"};
        return n;
    }
    double total() const { return graph_creation + feature_calculation + forward_pass + backward_pass; }
    StepTiming& operator+=(const StepTiming& o) {
        graph_creation += o.graph_creation;
        feature_calculation += o.feature_calculation;
        forward_pass += o.forward_pass;
        backward_pass += o.backward_pass;
        return *this;
    }
};

class Distributed {
public:
    static Distributed create_distributed(const AtomicSystem& system, double atom_cutoff,
                                          std::optional<double> threebody_cutoff, int p,
                                          int n_threads, bool allow_narrow = false,
                                          double threebody_tau = 0.0, int device = 0) {
        Distributed d;
        gmd_handle* raw = nullptr;
        int rc = gmd_create(device, &raw);
        if (rc != GMD_OK) throw Error(gmd_last_error(nullptr));
        d.h_.reset(raw, [](gmd_handle* x) { gmd_destroy(x); });
        d.p_ = p;
        d.n_threads_ = n_threads > 0 ? n_threads : 1;
        d.cutoff_ = atom_cutoff;
        d.r3_ = threebody_cutoff;
        d.tau_ = threebody_tau;
        const std::size_t n = system.size();
        std::vector<double> pos(3 * n), lat(9);
        std::vector<int32_t> z(system.species.begin(), system.species.end());
        for (std::size_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) pos[3 * i + k] = system.positions[i][k];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) lat[3 * r + k] = system.lattice[r][k];
        uint8_t pbc[3] = {system.pbc[0], system.pbc[1], system.pbc[2]};
        if (z.size() != n) throw Error("species length does not match atom count");
        detail::check(d.h_.get(),
                      gmd_build(d.h_.get(), (int64_t)n, pos.data(), z.data(), lat.data(), pbc,
                                atom_cutoff, threebody_cutoff ? *threebody_cutoff : 0.0,
                                threebody_tau, p, n_threads, allow_narrow ? GMD_ALLOW_NARROW : 0u));
        d.system_ = system;
        return d;
    }

    int num_partitions() const { return p_; }
    int num_threads() const { return n_threads_; }
    bool has_line_graph() const {
        int y = 0;
        gmd_has_line_graph(h_.get(), &y);
        return y != 0;
    }
    gmd_handle* handle() const { return h_.get(); }

    const AtomicSystem& system() const {  // after ensure_periodic
        if (!sys_ready_) {
            int64_t n = 0;
            gmd_num_nodes(h_.get(), &n);
            std::vector<double> pos(3 * n), lat(9);
            detail::check(h_.get(), gmd_get_system(h_.get(), pos.data(), lat.data()));
            AtomicSystem s;
            s.species = system_.species;
            s.positions.resize(n);
            for (int64_t i = 0; i < n; ++i) s.positions[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            for (int r = 0; r < 3; ++r) s.lattice[r] = {lat[3 * r], lat[3 * r + 1], lat[3 * r + 2]};
            periodic_ = s;
            sys_ready_ = true;
        }
        return periodic_;
    }

    const AtomGraph& graph() const {
        if (!graph_) {
            auto g = std::make_unique<AtomGraph>();
            int64_t ne = 0, n = 0;
            gmd_num_edges(h_.get(), &ne);
            gmd_num_nodes(h_.get(), &n);
            std::vector<int32_t> off(3 * ne);
            std::vector<double> vec(3 * ne);
            g->src.resize(ne);
            g->dst.resize(ne);
            g->distance.resize(ne);
            detail::check(h_.get(), gmd_get_graph(h_.get(), g->src.data(), g->dst.data(), off.data(),
                                                  g->distance.data(), vec.data()));
            g->image_offset.resize(ne);
            g->vector.resize(ne);
            for (int64_t e = 0; e < ne; ++e) {
                g->image_offset[e] = {off[3 * e], off[3 * e + 1], off[3 * e + 2]};
                g->vector[e] = {vec[3 * e], vec[3 * e + 1], vec[3 * e + 2]};
            }
            g->cutoff = cutoff_;
            g->num_nodes = n;
            graph_ = std::move(g);
        }
        return *graph_;
    }

    const PartitionedAtomGraph& atom_parts() const {
        if (!parts_) parts_ = std::make_unique<PartitionedAtomGraph>(detail::read_atom_parts(h_.get(), p_));
        return *parts_;
    }

    const PartitionedLineGraph& line_parts() const {
        if (!has_line_graph()) throw Error("no line graph was built");
        if (!lines_)
            lines_ = std::make_unique<PartitionedLineGraph>(
                detail::read_line_parts(h_.get(), p_, r3_ ? *r3_ : 0.0, tau_));
        return *lines_;
    }

    const std::vector<std::int64_t>& src_nodes(int i) const { return atom_parts().parts[i].local_src; }
    const std::vector<std::int64_t>& dst_nodes(int i) const { return atom_parts().parts[i].local_dst; }
    std::int64_t atom_rows(int i) const { return atom_parts().parts[i].layout.size(); }
    std::int64_t bond_rows(int i) const { return line_parts().parts[i].layout.size(); }

    // ---- features: host blocks, exchanged on the GPU -------------------
    DistributedFeatures make_atom_features(std::int64_t width) const { return make(width, 0); }
    DistributedFeatures make_bond_features(std::int64_t width) const {
        if (!has_line_graph()) throw Error("no line graph was built");
        return make(width, 1);
    }
    DistributedFeatures distribute_node_features(const std::vector<double>& f, std::int64_t width) const {
        int64_t n = 0;
        gmd_num_nodes(h_.get(), &n);
        if ((int64_t)f.size() != n * width) throw Error("node feature shape mismatch");
        DistributedFeatures out = make(width, 0);
        std::vector<double> flat(flat_rows(0) * width);
        detail::check(h_.get(), gmd_distribute(h_.get(), 0, f.data(), flat.data(), (int)width,
                                               GMD_F64 | GMD_HOST_MEMORY));
        unflatten(flat, out, 0);
        return out;
    }
    void atom_transfer(DistributedFeatures& f) const { op(gmd_transfer, f, 0); }
    void bond_transfer(DistributedFeatures& f) const { op(gmd_transfer, f, 1); }
    void atom_transfer_transpose(DistributedFeatures& f) const { op(gmd_transfer_transpose, f, 0); }
    void bond_transfer_transpose(DistributedFeatures& f) const { op(gmd_transfer_transpose, f, 1); }
    void sync_atom_duplicates(DistributedFeatures& f) const { op(gmd_sync_duplicates, f, 0); }
    void sync_bond_duplicates(DistributedFeatures& f) const { op(gmd_sync_duplicates, f, 1); }
    std::vector<double> aggregate(const DistributedFeatures& f) const { return agg(f, 0); }
    std::vector<double> aggregate_bonds(const DistributedFeatures& f) const { return agg(f, 1); }
    void corrupt_transfer_plan_for_test() { detail::check(h_.get(), gmd_corrupt_transfer_plan_for_test(h_.get())); }

    // owned-edge feature blocks (engine.cpp:103-120, 248-260): partition i
    // holds the rows of its owned edges in owned_edges order
    DistributedFeatures distribute_edge_features(const std::vector<double>& f, std::int64_t width) const {
        const PartitionedAtomGraph& ap = atom_parts();
        if (f.size() != graph().num_edges() * (std::size_t)width) throw Error("edge feature shape mismatch");
        DistributedFeatures out;
        out.width = width;
        out.blocks.resize(p_);
        for (int i = 0; i < p_; ++i) {
            const auto& owned = ap.parts[i].owned_edges;
            out.blocks[i].resize(owned.size() * width);
            for (std::size_t k = 0; k < owned.size(); ++k)
                std::copy(f.begin() + owned[k] * width, f.begin() + (owned[k] + 1) * width,
                          out.blocks[i].begin() + k * width);
        }
        return out;
    }
    std::vector<double> aggregate_edges(const DistributedFeatures& f) const {
        const PartitionedAtomGraph& ap = atom_parts();
        std::vector<double> out(graph().num_edges() * f.width, 0.0);
        for (int i = 0; i < p_; ++i) {
            const auto& owned = ap.parts[i].owned_edges;
            for (std::size_t k = 0; k < owned.size(); ++k)
                std::copy(f.row(i, (std::int64_t)k), f.row(i, (std::int64_t)k) + f.width,
                          out.begin() + owned[k] * f.width);
        }
        return out;
    }

    using LayerFn = std::function<void(int partition, DistributedFeatures&)>;

    // fn(partition) for every partition; a failure is rethrown with the id of
    // the first failing partition (engine.cpp:262-284).  Callbacks run in
    // partition order on the calling thread: the device work they enqueue is
    // ordered on the handle's stream, so there is no host parallelism to add.
    void parallel_for_partitions(const std::function<void(int)>& fn) const {
        std::vector<std::string> errors(p_);
        bool failed = false;
        for (int i = 0; i < p_; ++i) {
            try {
                fn(i);
            } catch (const std::exception& e) {
                errors[i] = e.what();
                failed = true;
            }
        }
        if (failed)
            for (int i = 0; i < p_; ++i)
                if (!errors[i].empty())
                    throw Error("worker for partition " + std::to_string(i) + " failed: " + errors[i]);
    }

    // each layer on every partition, then the border exchange (engine.cpp:286-294)
    void run_layered(const std::vector<LayerFn>& layers, DistributedFeatures& features) const {
        for (const LayerFn& layer : layers) {
            parallel_for_partitions([&](int i) { layer(i, features); });
            sync_atom_duplicates(features);
            atom_transfer(features);
        }
    }

private:
    std::shared_ptr<gmd_handle> h_;
    int p_ = 1, n_threads_ = 1;
    double cutoff_ = 0, tau_ = 0;
    std::optional<double> r3_;
    AtomicSystem system_;
    mutable AtomicSystem periodic_;
    mutable bool sys_ready_ = false;
    mutable std::unique_ptr<AtomGraph> graph_;
    mutable std::unique_ptr<PartitionedAtomGraph> parts_;
    mutable std::unique_ptr<PartitionedLineGraph> lines_;

    std::int64_t flat_rows(int bonds) const {
        int64_t r = 0;
        detail::check(h_.get(), gmd_block_rows(h_.get(), bonds, &r));
        return r;
    }
    std::int64_t block_offset(int i, int bonds) const {
        int64_t r = 0;
        detail::check(h_.get(), gmd_block_offset(h_.get(), i, bonds, &r));
        return r;
    }
    DistributedFeatures make(std::int64_t width, int bonds) const {
        DistributedFeatures f;
        f.width = width;
        f.blocks.resize(p_);
        for (int i = 0; i < p_; ++i) {
            std::int64_t rows = (i + 1 < p_ ? block_offset(i + 1, bonds) : flat_rows(bonds)) - block_offset(i, bonds);
            f.blocks[i].assign(rows * width, 0.0);
        }
        return f;
    }
    std::vector<double> flatten(const DistributedFeatures& f) const {
        std::vector<double> flat;
        for (const auto& b : f.blocks) flat.insert(flat.end(), b.begin(), b.end());
        return flat;
    }
    void unflatten(const std::vector<double>& flat, DistributedFeatures& f, int) const {
        std::size_t o = 0;
        for (auto& b : f.blocks) {
            std::copy(flat.begin() + o, flat.begin() + o + b.size(), b.begin());
            o += b.size();
        }
    }
    template <typename Fn>
    void op(Fn fn, DistributedFeatures& f, int bonds) const {
        if (bonds && !has_line_graph()) throw Error("no line graph was built");
        std::vector<double> flat = flatten(f);
        detail::check(h_.get(), fn(h_.get(), bonds, flat.data(), (int)f.width, GMD_F64 | GMD_HOST_MEMORY));
        unflatten(flat, f, bonds);
    }
    std::vector<double> agg(const DistributedFeatures& f, int bonds) const {
        int64_t n = 0;
        if (bonds) detail::check(h_.get(), gmd_get_num_bonds(h_.get(), &n));
        else gmd_num_nodes(h_.get(), &n);
        std::vector<double> flat = flatten(f), out(n * f.width);
        detail::check(h_.get(), gmd_aggregate(h_.get(), bonds, flat.data(), out.data(), (int)f.width,
                                              GMD_F64 | GMD_HOST_MEMORY));
        return out;
    }
};

// ---- model (potential.hpp:15-69) ----------------------------------------
struct ToyPotentialParams {
    int feature_width = 16, basis_count = 8, layers = 2;
    double r_atom = 4.0, r_3body = 0.0;
    std::uint64_t seed = 0;
    std::vector<double> embedding, layer_w, layer_b, basis_proj, basis3_proj, w3, w4, readout;

    bool threebody() const { return r_3body > 0.0; }
    static ToyPotentialParams init(std::uint64_t seed, int F = 16, int K = 8, int L = 2,
                                   double r_atom = 4.0, double r_3body = 0.0) {
        ToyPotentialParams p;
        p.feature_width = F;
        p.basis_count = K;
        p.layers = L;
        p.r_atom = r_atom;
        p.r_3body = r_3body;
        p.seed = seed;
        std::vector<double> blob(gmd_params_size(F, K, L));
        if (gmd_params_init(seed, F, K, L, r_atom, r_3body, blob.data()) != GMD_OK)
            throw Error("layer count must be >= 1");
        p.unpack(blob);
        p.validate();
        return p;
    }
    std::vector<double> blob() const {
        std::vector<double> b;
        for (const auto* v : {&embedding, &layer_w, &layer_b, &basis_proj, &basis3_proj, &w3, &w4, &readout})
            b.insert(b.end(), v->begin(), v->end());
        return b;
    }
    void validate() const {
        if (layers < 1) throw Error("layer count must be >= 1");
        if (feature_width < 1 || basis_count < 1) throw Error("feature and basis widths must be >= 1");
        if (r_atom <= 0.0) throw Error("atom cutoff must be positive");
        if (threebody() && r_3body > r_atom) throw Error("three-body cutoff cannot exceed the atom cutoff");
        validate_tables();  // sizes and finiteness per table (potential.cpp:157-175)
    }

    // binary parameter files (potential.cpp:178-260): GMPT, u32 version 1,
    // u32 F K L flags, f64 r_atom r_3body, u64 seed, u64-counted tables
    void save(const std::string& path) const {
        validate();
        std::ofstream out(path, std::ios::binary);
        if (!out) throw Error("cannot write file: " + path);
        out.write("GMPT", 4);
        auto put = [&](const auto& v) { out.write(reinterpret_cast<const char*>(&v), sizeof v); };
        put((std::uint32_t)1);
        put((std::uint32_t)feature_width);
        put((std::uint32_t)basis_count);
        put((std::uint32_t)layers);
        put((std::uint32_t)(threebody() ? 1u : 0u));
        put(r_atom);
        put(r_3body);
        put(seed);
        for (const auto* v : {&embedding, &layer_w, &layer_b, &basis_proj, &basis3_proj, &w3, &w4, &readout}) {
            put((std::uint64_t)v->size());
            out.write(reinterpret_cast<const char*>(v->data()), (std::streamsize)(v->size() * sizeof(double)));
        }
    }
    static ToyPotentialParams load(const std::string& path) {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Error("cannot open file: " + path);
        char magic[4] = {};
        in.read(magic, 4);
        if (!in || std::string(magic, 4) != "GMPT") throw Error("bad parameter file magic");
        auto get = [&](auto& v) { in.read(reinterpret_cast<char*>(&v), sizeof v); };
        std::uint32_t ver = 0, F = 0, K = 0, L = 0, flags = 0;
        get(ver);
        if (!in || ver != 1) throw Error("unsupported parameter file version");
        ToyPotentialParams p;
        get(F);
        get(K);
        get(L);
        get(flags);
        get(p.r_atom);
        get(p.r_3body);
        get(p.seed);
        p.feature_width = (int)F;
        p.basis_count = (int)K;
        p.layers = (int)L;
        for (auto* v : {&p.embedding, &p.layer_w, &p.layer_b, &p.basis_proj, &p.basis3_proj, &p.w3, &p.w4, &p.readout}) {
            std::uint64_t n = 0;
            get(n);
            if (!in) throw Error("truncated parameter file");
            v->resize((std::size_t)n);
            in.read(reinterpret_cast<char*>(v->data()), (std::streamsize)(n * sizeof(double)));
        }
        if (!in) throw Error("truncated parameter file");
        p.validate_tables();
        p.validate();
        return p;
    }

private:
    void validate_tables() const {  // potential.cpp:157-175 messages
        const std::size_t F = feature_width, K = basis_count, L = layers;
        auto expect = [](const std::vector<double>& v, std::size_t n, const char* name) {
            if (v.size() != n) throw Error(std::string("parameter array ") + name + " has the wrong size");
            for (double x : v)
                if (!std::isfinite(x)) throw Error(std::string("parameter array ") + name + " contains a non-finite value");
        };
        expect(embedding, 119 * F, "embedding");
        expect(layer_w, L * F * F, "layer_w");
        expect(layer_b, L * F, "layer_b");
        expect(basis_proj, F * K, "basis_proj");
        expect(basis3_proj, F * K, "basis3_proj");
        expect(w3, F * F, "w3");
        expect(w4, F * F, "w4");
        expect(readout, F, "readout");
    }
    void unpack(const std::vector<double>& b) {
        const std::size_t F = feature_width, K = basis_count, L = layers;
        std::size_t o = 0;
        auto take = [&](std::vector<double>& v, std::size_t n) {
            v.assign(b.begin() + o, b.begin() + o + n);
            o += n;
        };
        take(embedding, 119 * F);
        take(layer_w, L * F * F);
        take(layer_b, L * F);
        take(basis_proj, F * K);
        take(basis3_proj, F * K);
        take(w3, F * F);
        take(w4, F * F);
        take(readout, F);
    }
};

struct PotentialOutput {
    double energy = 0.0;
    std::vector<double> per_atom;
    std::vector<Vec3> forces;
    Mat3 stress;
};

inline PotentialOutput forward_distributed(const Distributed& dist, const ToyPotentialParams& params,
                                           StepTiming* timing = nullptr) {
    params.validate();
    gmd_handle* h = dist.handle();
    std::vector<double> blob = params.blob();
    detail::check(h, gmd_set_params(h, params.feature_width, params.basis_count, params.layers,
                                    params.r_atom, params.r_3body, blob.data()));
    int64_t n = 0;
    gmd_num_nodes(h, &n);
    PotentialOutput out;
    out.per_atom.resize(n);
    std::vector<double> f(3 * n);
    double st[9], tm[4];
    detail::check(h, gmd_forward(h, &out.energy, out.per_atom.data(), f.data(), st, tm, 0));
    out.forces.resize(n);
    for (int64_t i = 0; i < n; ++i) out.forces[i] = {f[3 * i], f[3 * i + 1], f[3 * i + 2]};
    for (int a = 0; a < 3; ++a) out.stress[a] = {st[3 * a], st[3 * a + 1], st[3 * a + 2]};
    if (timing) {
        timing->feature_calculation += tm[1];
        timing->forward_pass += tm[2];
        timing->backward_pass += tm[3];
    }
    return out;
}

// forward_serial (potential.hpp:51-53): the unpartitioned evaluation, i.e.
// one partition on one GPU (bitwise equal to every partition count here)
inline PotentialOutput forward_serial(const AtomicSystem& system, const ToyPotentialParams& params,
                                      int n_threads = 0, StepTiming* timing = nullptr) {
    Distributed d = Distributed::create_distributed(
        system, params.r_atom,
        params.threebody() ? std::optional<double>(params.r_3body) : std::nullopt, 1, n_threads,
        true);
    return forward_distributed(d, params, timing);
}

// neighborlist.hpp:37-38 on the GPU
inline AtomGraph build_neighbor_list(const AtomicSystem& system, double cutoff, int n_threads = 0) {
    return Distributed::create_distributed(system, cutoff, std::nullopt, 1, n_threads, true).graph();
}

// ---- free builders (partitioner.hpp:66-109, linegraph.hpp:26-78,
// neighborlist.hpp:40-42, potential.hpp:62-69), device-backed through the
// gmd_build_partitions / gmd_partition_rule / brute-force entry points ----
namespace detail {
using Handle = std::shared_ptr<gmd_handle>;
inline Handle make_handle(int device = 0) {
    gmd_handle* raw = nullptr;
    if (gmd_create(device, &raw) != GMD_OK) throw Error(gmd_last_error(nullptr));
    return Handle(raw, [](gmd_handle* x) { gmd_destroy(x); });
}
inline void flat_system(const AtomicSystem& s, std::vector<double>& pos, std::vector<double>& lat) {
    pos.resize(3 * s.size());
    lat.resize(9);
    for (std::size_t i = 0; i < s.size(); ++i)
        for (int k = 0; k < 3; ++k) pos[3 * i + k] = s.positions[i][k];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) lat[3 * r + k] = s.lattice[r][k];
}
// a caller's AtomGraph as the partitions of `owner` (or of system + rule)
inline Handle partitions_of(const AtomGraph& g, const AtomicSystem* sys, const PartitionRule& rule,
                            const std::vector<int>* owner, double r3, double tau, bool allow_narrow) {
    Handle h = make_handle();
    const std::size_t ne = g.num_edges();
    std::vector<int32_t> off(3 * ne);
    for (std::size_t e = 0; e < ne; ++e)
        for (int k = 0; k < 3; ++k) off[3 * e + k] = g.image_offset[e][k];
    std::vector<double> pos, lat;
    if (sys) flat_system(*sys, pos, lat);
    std::vector<int32_t> own;
    if (owner) own.assign(owner->begin(), owner->end());
    if (owner && (std::int64_t)own.size() != g.num_nodes) throw Error("owner table does not match the graph");
    if (sys && (std::int64_t)sys->size() != g.num_nodes) throw Error("system does not match the graph");
    check(h.get(), gmd_build_partitions(h.get(), g.num_nodes, sys ? pos.data() : nullptr,
                                        sys ? lat.data() : nullptr, (int64_t)ne, g.src.data(),
                                        g.dst.data(), off.data(), g.distance.data(), g.cutoff, r3, tau,
                                        rule.axis, rule.p, rule.boundaries.data(),
                                        owner ? own.data() : nullptr, allow_narrow ? GMD_ALLOW_NARROW : 0u));
    return h;
}
inline void check_rule(const PartitionRule& rule) {
    if (rule.p < 1 || (int)rule.boundaries.size() != rule.p + 1)
        throw Error("partition rule needs p + 1 boundaries");
}
}  // namespace detail

// ensure_periodic (system.cpp:242-270) on the device
inline AtomicSystem ensure_periodic(const AtomicSystem& system, double cutoff) {
    if (system.pbc[0] && system.pbc[1] && system.pbc[2]) return system;
    auto h = detail::make_handle();
    std::vector<double> pos, lat, opos(3 * system.size()), olat(9);
    detail::flat_system(system, pos, lat);
    const uint8_t pbc[3] = {system.pbc[0], system.pbc[1], system.pbc[2]};
    detail::check(h.get(), gmd_util_ensure_periodic(h.get(), (int64_t)system.size(), pos.data(), lat.data(),
                                                    pbc, cutoff, opos.data(), olat.data()));
    AtomicSystem out = system;
    for (std::size_t i = 0; i < out.size(); ++i) out.positions[i] = {opos[3 * i], opos[3 * i + 1], opos[3 * i + 2]};
    for (int r = 0; r < 3; ++r) out.lattice[r] = {olat[3 * r], olat[3 * r + 1], olat[3 * r + 2]};
    out.pbc = {true, true, true};
    out.validate();
    return out;
}

inline int symbol_to_z(const std::string& symbol) {  // system.cpp:272-277
    for (int z = 1; z <= 118; ++z)
        if (symbol == detail::element_symbols()[z]) return z;
    throw Error("unknown element symbol '" + symbol + "'");
}

// choose_partition_rule (partitioner.cpp:46-91): quantile walls by a device
// radix select over the wrapped fractions
inline PartitionRule choose_partition_rule(const AtomicSystem& system, int p,
                                           BoundaryMode mode = BoundaryMode::kQuantile) {
    if (p < 1) throw Error("partition count must be >= 1");
    if (p > 64) throw Error("partition count limited to 64");
    if (static_cast<std::size_t>(p) > system.size()) throw Error("more partitions than atoms");
    system.validate();
    auto h = detail::make_handle();
    std::vector<double> pos, lat;
    detail::flat_system(system, pos, lat);
    PartitionRule rule;
    rule.p = p;
    rule.boundaries.resize(p + 1);
    detail::check(h.get(), gmd_partition_rule(h.get(), (int64_t)system.size(), pos.data(), lat.data(), p,
                                              mode == BoundaryMode::kEqualWidth ? 1 : 0, &rule.axis,
                                              rule.boundaries.data()));
    return rule;
}

// which_partition (partitioner.cpp:93-108): half-open slabs, ties to the right
inline int which_partition(const PartitionRule& rule, double frac) {
    if (frac >= 1.0) return rule.p - 1;
    auto it = std::upper_bound(rule.boundaries.begin() + 1, rule.boundaries.end() - 1, frac);
    return static_cast<int>(it - rule.boundaries.begin()) - 1;
}

// fractional_along_axis (partitioner.cpp:38-44) on the device
inline std::vector<double> fractional_along_axis(const AtomicSystem& system, int axis) {
    auto h = detail::make_handle();
    std::vector<double> pos, lat, out(system.size());
    detail::flat_system(system, pos, lat);
    detail::check(h.get(), gmd_assign_owners(h.get(), (int64_t)system.size(), pos.data(), lat.data(), axis,
                                             0, nullptr, out.data(), nullptr));
    return out;
}

inline int which_partition(std::int64_t node, const AtomicSystem& system, const PartitionRule& rule) {
    if (node < 0 || static_cast<std::size_t>(node) >= system.size()) throw Error("node id out of range");
    return which_partition(rule, fractional_along_axis(system, rule.axis)[node]);
}

// build_span_layout (partitioner.cpp:153-180): [PURE | TO... | FROM...] of
// caller-supplied buckets (first occurrence is canonical)
inline SpanLayout build_span_layout(const Buckets& buckets, int partition) {
    const int p = static_cast<int>(buckets.pure.size());
    SpanLayout L;
    L.p = p;
    L.markers.assign(2 + 2 * p, 0);
    auto append = [&](const std::vector<std::int64_t>& ids) {
        for (std::int64_t g : ids) {
            const std::int64_t r = static_cast<std::int64_t>(L.node_array.size());
            L.node_array.push_back(g);
            auto ins = L.global_to_local.emplace(g, r);
            if (!ins.second) L.duplicates.emplace_back(ins.first->second, r);
        }
    };
    append(buckets.pure[partition]);
    L.markers[1] = L.size();
    for (int j = 0; j < p; ++j) {
        append(buckets.to[partition][j]);
        L.markers[2 + j] = L.size();
    }
    for (int j = 0; j < p; ++j) {
        append(buckets.from[partition][j]);
        L.markers[2 + p + j] = L.size();
    }
    return L;
}

// build_atom_partitions / assign_to_partitions (partitioner.cpp:110-218) of
// the caller's graph: owners, requirement masks, stable compaction into span
// layouts and edge ownership all run on the GPU
inline PartitionedAtomGraph build_atom_partitions(const AtomGraph& graph, const AtomicSystem& system,
                                                  const PartitionRule& rule, bool allow_narrow = false) {
    detail::check_rule(rule);
    auto h = detail::partitions_of(graph, &system, rule, nullptr, 0.0, 0.0, allow_narrow);
    PartitionedAtomGraph out = detail::read_atom_parts(h.get(), rule.p);
    out.rule = rule;
    return out;
}

inline Buckets assign_to_partitions(const AtomGraph& graph, const AtomicSystem& system,
                                    const PartitionRule& rule, bool allow_narrow = false) {
    return build_atom_partitions(graph, system, rule, allow_narrow).buckets;
}

// collect_bonds (linegraph.cpp:25-43): edges with d <= r + tau, on the device
inline BondSet collect_bonds(const AtomGraph& graph, double r, double tau) {
    if (r > graph.cutoff) throw Error("three-body range cannot exceed the atom graph cutoff");
    if (tau < 0.0) throw Error("tolerance tau must be >= 0");
    PartitionRule one;
    one.boundaries = {0.0, 1.0};
    const std::vector<int> zero(graph.num_nodes, 0);
    if (r <= 0.0) {  // no bond can pass d <= r + tau with d > 0 ... unless tau > 0
        BondSet b;
        b.r = r;
        b.tau = tau;
        b.bond_of_edge.assign(graph.num_edges(), -1);
        b.by_src.assign(graph.num_nodes, {});
        b.by_dst.assign(graph.num_nodes, {});
        if (r + tau <= 0.0) return b;
    }
    auto h = detail::partitions_of(graph, nullptr, one, &zero, r > 0.0 ? r : 1e-300, r > 0.0 ? tau : r + tau - 1e-300, true);
    BondSet b = detail::read_bonds(h.get(), r, tau, nullptr);
    return b;
}

// build_two_hop_closure (linegraph.cpp:45-65): u64 partition masks per node,
// two gather hops along the CSR on the device
inline std::vector<std::vector<std::int64_t>> build_two_hop_closure(const PartitionedAtomGraph& atom_parts,
                                                                    const AtomGraph& graph) {
    auto h = detail::partitions_of(graph, nullptr, atom_parts.rule, &atom_parts.owner, 0.0, 0.0, true);
    std::vector<std::vector<std::int64_t>> out(atom_parts.p);
    for (int i = 0; i < atom_parts.p; ++i) {
        int64_t c = 0;
        detail::check(h.get(), gmd_get_closure(h.get(), i, &c, nullptr));
        out[i].resize(c);
        detail::check(h.get(), gmd_get_closure(h.get(), i, &c, out[i].data()));
    }
    return out;
}

// build_edge_tables (linegraph.cpp:67-122).  Table membership is computed on
// the device from the two-hop closure; the closure passed in must be that
// closure (the reference's only construction of it)
inline EdgeTables build_edge_tables(const AtomGraph& graph,
                                    const std::vector<std::vector<std::int64_t>>& closure,
                                    const PartitionedAtomGraph& atom_parts, double r, double tau) {
    if (r > graph.cutoff) throw Error("three-body range cannot exceed the atom graph cutoff");
    if (tau < 0.0) throw Error("tolerance tau must be >= 0");
    auto h = detail::partitions_of(graph, nullptr, atom_parts.rule, &atom_parts.owner, r, tau, true);
    for (int i = 0; i < atom_parts.p; ++i) {
        int64_t c = 0;
        detail::check(h.get(), gmd_get_closure(h.get(), i, &c, nullptr));
        std::vector<std::int64_t> mine(c);
        detail::check(h.get(), gmd_get_closure(h.get(), i, &c, mine.data()));
        std::vector<std::int64_t> given = i < (int)closure.size() ? closure[i] : std::vector<std::int64_t>{};
        std::sort(given.begin(), given.end());
        if (given != mine)
            throw Error("build_edge_tables: closure is not build_two_hop_closure(atom_parts, graph)");
    }
    EdgeTables t;
    PartitionedLineGraph lg = detail::read_line_parts(h.get(), atom_parts.p, r, tau);
    t.bonds = std::move(lg.bonds);
    t.bond_owner = std::move(lg.bond_owner);
    t.bond_buckets = std::move(lg.bond_buckets);
    std::vector<uint64_t> mask(t.bonds.size());
    if (!mask.empty()) detail::check(h.get(), gmd_get_bond_tables(h.get(), mask.data()));
    t.per_partition.resize(atom_parts.p);
    for (std::size_t b = 0; b < t.bonds.size(); ++b) {
        const std::int64_t v = graph.src[t.bonds.edge_of_bond[b]];
        for (uint64_t m = mask[b]; m; m &= m - 1)
            t.per_partition[__builtin_ctzll(m)][v].push_back((std::int64_t)b);
    }
    return t;
}

// build_line_graph_partitions (linegraph.cpp:124-171): bond layouts and the
// (e', e)-ordered line edges per partition, on the device
inline PartitionedLineGraph build_line_graph_partitions(const EdgeTables& tables, const AtomGraph& graph,
                                                        const PartitionedAtomGraph& atom_parts) {
    auto h = detail::partitions_of(graph, nullptr, atom_parts.rule, &atom_parts.owner, tables.bonds.r,
                                   tables.bonds.tau, true);
    PartitionedLineGraph lg = detail::read_line_parts(h.get(), atom_parts.p, tables.bonds.r, tables.bonds.tau);
    if (lg.bonds.edge_of_bond != tables.bonds.edge_of_bond)
        throw Error("build_line_graph_partitions: tables do not belong to this graph");
    return lg;
}

// serial_line_graph (linegraph.cpp:183-199): the p = 1 line graph as sorted
// global (edge e, edge e') pairs
inline std::vector<std::pair<std::int64_t, std::int64_t>> serial_line_graph(const AtomGraph& graph, double r,
                                                                             double tau) {
    if (r > graph.cutoff) throw Error("three-body range cannot exceed the atom graph cutoff");
    if (tau < 0.0) throw Error("tolerance tau must be >= 0");
    PartitionRule one;
    one.boundaries = {0.0, 1.0};
    const std::vector<int> zero(graph.num_nodes, 0);
    auto h = detail::partitions_of(graph, nullptr, one, &zero, r, tau, true);
    PartitionedLineGraph lg = detail::read_line_parts(h.get(), 1, r, tau);
    std::vector<std::pair<std::int64_t, std::int64_t>> out;
    out.reserve(lg.parts[0].line_edges.size());
    const auto& na = lg.parts[0].layout.node_array;
    for (const auto& [le, lep] : lg.parts[0].line_edges)
        out.emplace_back(lg.bonds.edge_of_bond[na[le]], lg.bonds.edge_of_bond[na[lep]]);
    std::sort(out.begin(), out.end());
    return out;
}

// brute_force_line_graph (linegraph.cpp:201-219): independent per-center
// enumeration of (in-bond, out-bond) pairs on the device, N <= 2000
inline std::vector<std::pair<std::int64_t, std::int64_t>> brute_force_line_graph(const AtomGraph& graph, double r,
                                                                                  double tau) {
    if (graph.num_nodes > 2000) throw Error("brute force guard: N > 2000");
    if (r > graph.cutoff) throw Error("three-body range cannot exceed the atom graph cutoff");
    if (tau < 0.0) throw Error("tolerance tau must be >= 0");
    PartitionRule one;
    one.boundaries = {0.0, 1.0};
    const std::vector<int> zero(graph.num_nodes, 0);
    auto h = detail::partitions_of(graph, nullptr, one, &zero, r, tau, true);
    int64_t c = 0;
    detail::check(h.get(), gmd_brute_force_line_graph(h.get(), &c, nullptr));
    std::vector<int64_t> pairs(2 * c);
    detail::check(h.get(), gmd_brute_force_line_graph(h.get(), &c, pairs.data()));
    std::vector<std::pair<std::int64_t, std::int64_t>> out(c);
    for (int64_t k = 0; k < c; ++k) out[k] = {pairs[2 * k], pairs[2 * k + 1]};
    return out;
}

// brute_force_neighbor_list (neighborlist.cpp:199-239): every (dst, src,
// image) of the span tested on the device with the reference's fp64
// expressions, N <= 5000
inline AtomGraph brute_force_neighbor_list(const AtomicSystem& system, double cutoff) {
    if (cutoff <= 0.0) throw Error("cutoff must be positive");
    if (system.size() == 0) throw Error("cannot build neighbor list for empty system");
    if (system.size() > 5000) throw Error("brute force guard: N > 5000");
    auto h = detail::make_handle();
    std::vector<double> pos, lat;
    detail::flat_system(system, pos, lat);
    const uint8_t pbc[3] = {system.pbc[0], system.pbc[1], system.pbc[2]};
    int64_t ne = 0;
    const int64_t n = (int64_t)system.size();
    detail::check(h.get(), gmd_brute_force_neighbor_list(h.get(), n, pos.data(), lat.data(), pbc, cutoff, &ne,
                                                         nullptr, nullptr, nullptr, nullptr, nullptr));
    AtomGraph g;
    g.cutoff = cutoff;
    g.num_nodes = n;
    g.src.resize(ne);
    g.dst.resize(ne);
    g.distance.resize(ne);
    std::vector<int32_t> off(3 * ne);
    std::vector<double> vec(3 * ne);
    detail::check(h.get(), gmd_brute_force_neighbor_list(h.get(), n, pos.data(), lat.data(), pbc, cutoff, &ne,
                                                         g.src.data(), g.dst.data(), off.data(),
                                                         g.distance.data(), vec.data()));
    g.image_offset.resize(ne);
    g.vector.resize(ne);
    for (int64_t e = 0; e < ne; ++e) {
        g.image_offset[e] = {off[3 * e], off[3 * e + 1], off[3 * e + 2]};
        g.vector[e] = {vec[3 * e], vec[3 * e + 1], vec[3 * e + 2]};
    }
    return g;
}

// finite_difference_forces / _stress (potential.cpp:991-1037): central
// differences of the GPU energy (forward_serial).  The energy is a sum of
// fp32-computed per-atom terms, so the difference quotient carries
// ~1e-6 eV / (2 eps) of rounding noise -- a check at fp32 tolerance, not the
// reference's fp64 1e-6 eV/A
inline std::vector<Vec3> finite_difference_forces(const AtomicSystem& system, const ToyPotentialParams& params,
                                                  double eps) {
    if (eps < 1e-6 || eps > 1e-2) throw Error("finite-difference step must lie in [1e-6, 1e-2] A");
    std::vector<Vec3> forces(system.size(), Vec3{});
    AtomicSystem probe = system;
    for (std::size_t i = 0; i < system.size(); ++i)
        for (int k = 0; k < 3; ++k) {
            probe.positions[i][k] = system.positions[i][k] + eps;
            const double ep = forward_serial(probe, params).energy;
            probe.positions[i][k] = system.positions[i][k] - eps;
            const double em = forward_serial(probe, params).energy;
            probe.positions[i][k] = system.positions[i][k];
            forces[i][k] = -(ep - em) / (2.0 * eps);
        }
    return forces;
}

inline Mat3 finite_difference_stress(const AtomicSystem& system, const ToyPotentialParams& params, double eps) {
    if (eps <= 0.0 || eps > 1e-3) throw Error("strain step must lie in (0, 1e-3]");
    const AtomicSystem base = ensure_periodic(system, params.r_atom);
    const double volume = std::abs(base.lattice.det());
    auto deform = [&](int a, int b, double strain) {  // x_a += strain x_b, positions and lattice
        AtomicSystem s = base;
        for (Vec3& r : s.positions) r[a] += strain * r[b];
        for (int row = 0; row < 3; ++row) s.lattice[row][a] += strain * s.lattice[row][b];
        return s;
    };
    Mat3 raw{}, out{};
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            raw[a][b] = (forward_serial(deform(a, b, eps), params).energy -
                         forward_serial(deform(a, b, -eps), params).energy) /
                        (2.0 * eps * volume);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) out[a][b] = 0.5 * (raw[a][b] + raw[b][a]);
    return out;
}

// ---- md.hpp (md.cpp:11-179): the caller of the hot path --------------------
namespace units {
inline constexpr double kAccel = 9.648533212e-3;
inline constexpr double kKinetic = 103.642697;
inline constexpr double kBoltzmann = 8.617333262e-5;
}  // namespace units

inline double atomic_mass(int z) {
    double m = 0.0;
    int32_t zz = z;
    if (gmd_md_masses(1, &zz, &m) != GMD_OK) throw Error(gmd_last_error(nullptr));
    return m;
}

struct MDState {
    AtomicSystem system;
    std::vector<Vec3> velocities;  // A/fs
    std::vector<double> masses;    // amu
    std::vector<Vec3> forces;      // eV/A at the current positions
    double potential_energy = 0.0;
    std::int64_t step = 0;
    double kinetic_energy() const {
        double e = 0.0;
        for (std::size_t i = 0; i < velocities.size(); ++i)
            e += 0.5 * masses[i] * velocities[i].norm2();
        return e * units::kKinetic;
    }
    double temperature() const {
        if (velocities.empty()) return 0.0;
        const double dof = std::max<double>(1.0, 3.0 * velocities.size() - 3.0);
        return 2.0 * kinetic_energy() / (dof * units::kBoltzmann);
    }
};

struct MDOptions {
    double dt = 1.0;
    std::int64_t steps = 0;
    int partitions = 1;
    int threads = 0;
    bool allow_narrow = false;
    std::uint64_t seed = 0;
    double init_temperature = 300.0;
    std::string energy_csv;
    std::string timing_csv;
    std::string trajectory_xyz;       // snapshot prefix: PREFIX.<step>.xyz
    std::int64_t snapshot_every = 0;  // 0 disables
};

struct MDStepRecord {
    std::int64_t step = 0;
    double potential = 0.0, kinetic = 0.0, total = 0.0, max_force = 0.0;
    StepTiming timing;
};

struct MDResult {
    MDState state;
    std::vector<MDStepRecord> records;
};

inline std::vector<Vec3> maxwell_boltzmann_velocities(const AtomicSystem& system,
                                                      double temperature, std::uint64_t seed) {
    const std::size_t n = system.size();
    std::vector<int32_t> z(system.species.begin(), system.species.end());
    std::vector<double> v(3 * n);
    if (gmd_md_maxwell_boltzmann((int64_t)n, z.data(), temperature, seed, v.data()) != GMD_OK)
        throw Error(gmd_last_error(nullptr));
    std::vector<Vec3> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
    return out;
}

inline MDState init_md_state(const AtomicSystem& system, const MDOptions& opts) {
    MDState st;
    st.system = system;
    st.system.validate();
    st.masses.resize(system.size());
    for (std::size_t i = 0; i < system.size(); ++i) st.masses[i] = atomic_mass(system.species[i]);
    st.velocities = maxwell_boltzmann_velocities(system, opts.init_temperature, opts.seed);
    return st;
}

namespace detail {
// `steps` velocity-Verlet steps of st on the device (gmd_md_run): host state
// in and out, the trajectory in between stays in HBM
inline std::vector<double> md_device(MDState& st, const ToyPotentialParams& params,
                                     const MDOptions& opts, std::int64_t steps, int device = 0) {
    params.validate();
    if (opts.dt < 0.0) throw Error("time step must be >= 0");
    gmd_handle* raw = nullptr;
    if (gmd_create(device, &raw) != GMD_OK) throw Error(gmd_last_error(nullptr));
    std::unique_ptr<gmd_handle, void (*)(gmd_handle*)> h(raw, [](gmd_handle* x) { gmd_destroy(x); });
    std::vector<double> blob = params.blob();
    check(h.get(), gmd_set_params(h.get(), params.feature_width, params.basis_count, params.layers,
                                  params.r_atom, params.r_3body, blob.data()));
    const std::size_t n = st.system.size();
    std::vector<double> pos(3 * n), vel(3 * n), frc(3 * n), lat(9), rec(8 * (steps + 1));
    std::vector<int32_t> z(st.system.species.begin(), st.system.species.end());
    for (std::size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            pos[3 * i + k] = st.system.positions[i][k];
            vel[3 * i + k] = st.velocities.empty() ? 0.0 : st.velocities[i][k];
        }
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) lat[3 * r + k] = st.system.lattice[r][k];
    uint8_t pbc[3] = {st.system.pbc[0], st.system.pbc[1], st.system.pbc[2]};
    check(h.get(), gmd_md_run(h.get(), (int64_t)n, pos.data(), vel.data(), frc.data(), z.data(),
                              lat.data(), pbc, opts.dt, steps, params.r_atom,
                              params.threebody() ? params.r_3body : 0.0, 0.0, opts.partitions,
                              opts.allow_narrow ? GMD_ALLOW_NARROW : 0u, rec.data()));
    st.velocities.resize(n);
    st.forces.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        st.system.positions[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        st.velocities[i] = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
        st.forces[i] = {frc[3 * i], frc[3 * i + 1], frc[3 * i + 2]};
    }
    st.potential_energy = rec[8 * steps];
    st.step += steps;
    return rec;
}
}  // namespace detail

// velocity_verlet_step (md.cpp:85-110) on the device; the forces of the
// current positions are recomputed on entry (deterministic, equal to
// state.forces when those belong to the current positions)
inline void velocity_verlet_step(MDState& state, const ToyPotentialParams& params,
                                 const MDOptions& opts, StepTiming* timing = nullptr) {
    if (state.forces.size() != state.system.size())
        throw Error("step requires forces at the current positions");
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<double> rec = detail::md_device(state, params, opts, 1);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timing) {  // device categories; the host side of the step (handle,
        // parameter and state transfers) is counted as graph creation, so the
        // categories partition the step's wall time as the reference's do
        const double dev = rec[12] + rec[13] + rec[14] + rec[15];
        timing->graph_creation += rec[12] + std::max(0.0, wall - dev);
        timing->feature_calculation += rec[13];
        timing->forward_pass += rec[14];
        timing->backward_pass += rec[15];
    }
}

inline void write_energy_csv(const std::string& path, const std::vector<MDStepRecord>& records) {
    std::ofstream out(path);
    if (!out) throw Error("cannot write file: " + path);
    out << "step,potential_ev,kinetic_ev,total_ev,max_force_ev_per_a";
    for (const std::string& name : StepTiming::category_names()) {
        std::string col = name;
        for (char& c : col) c = c == ' ' ? '_' : static_cast<char>(std::tolower(c));
        out << "," << col << "_s";
    }
    out << "\n";
    out.precision(12);
    for (const MDStepRecord& r : records)
        out << r.step << "," << r.potential << "," << r.kinetic << "," << r.total << ","
            << r.max_force << "," << r.timing.graph_creation << "," << r.timing.feature_calculation
            << "," << r.timing.forward_pass << "," << r.timing.backward_pass << "\n";
}

// write_timing_csv (engine.cpp:29-41): step, then the four categories
inline void write_timing_csv(const std::string& path, const std::vector<StepTiming>& rows) {
    std::ofstream out(path);
    if (!out) throw Error("cannot write file: " + path);
    out << "step";
    for (const std::string& name : StepTiming::category_names()) out << "," << name;
    out << "\n";
    out.precision(9);
    for (std::size_t i = 0; i < rows.size(); ++i)
        out << i << "," << rows[i].graph_creation << "," << rows[i].feature_calculation << ","
            << rows[i].forward_pass << "," << rows[i].backward_pass << "\n";
}

// run_md (md.cpp:112-160): the trajectory runs device-resident between
// snapshots (one gmd_md_run per snapshot interval; the forces at a
// segment's first positions are re-evaluated, bitwise equal to the previous
// segment's last evaluation, and that duplicate record is dropped)
inline MDResult run_md(const AtomicSystem& system, const ToyPotentialParams& params,
                       const MDOptions& opts) {
    MDResult res;
    res.state = init_md_state(system, opts);
    res.state.step = 0;
    const bool snap = !opts.trajectory_xyz.empty() && opts.snapshot_every > 0;
    auto snapshot = [&](std::int64_t step) {
        if (snap && step % opts.snapshot_every == 0)
            save_xyz(res.state.system, opts.trajectory_xyz + "." + std::to_string(step) + ".xyz");
    };
    auto push = [&](const std::vector<double>& rec, std::int64_t s, std::int64_t step) {
        MDStepRecord r;
        r.step = step;
        r.potential = rec[8 * s];
        r.kinetic = rec[8 * s + 1];
        r.total = rec[8 * s + 2];
        r.max_force = rec[8 * s + 3];
        r.timing.graph_creation = rec[8 * s + 4];
        r.timing.feature_calculation = rec[8 * s + 5];
        r.timing.forward_pass = rec[8 * s + 6];
        r.timing.backward_pass = rec[8 * s + 7];
        res.records.push_back(r);
    };
    const std::int64_t seg = snap ? opts.snapshot_every : std::max<std::int64_t>(opts.steps, 0);
    std::int64_t done = 0;
    snapshot(0);
    do {
        const std::int64_t k = std::min(seg, opts.steps - done);
        std::vector<double> rec = detail::md_device(res.state, params, opts, k);
        if (done == 0) push(rec, 0, 0);
        for (std::int64_t s = 1; s <= k; ++s) push(rec, s, done + s);
        done += k;
        if (k > 0) snapshot(done);
    } while (done < opts.steps);
    if (!opts.energy_csv.empty()) write_energy_csv(opts.energy_csv, res.records);
    if (!opts.timing_csv.empty()) {
        std::vector<StepTiming> rows;
        for (const MDStepRecord& r : res.records) rows.push_back(r.timing);
        write_timing_csv(opts.timing_csv, rows);
    }
    return res;
}

}  // namespace graphmd
