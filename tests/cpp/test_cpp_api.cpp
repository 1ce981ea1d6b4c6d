// C++ drop-in parity tests: the reference's own test scenarios
// (proj/tests/test_{neighborlist,partitioner,linegraph,engine,potential}.cpp)
// written against include/graphmd_b200/graphmd.hpp, i.e. the reference API
// running on the GPU, checked against the fp64 oracle (oracle/gmd_oracle.h).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/graphmd_b200/graphmd.hpp"
#include "../../oracle/gmd_oracle.h"

using namespace graphmd;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                    \
    do {                                                                            \
        ++g_checks;                                                                 \
        if (!(c)) {                                                                 \
            ++g_fail;                                                               \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);      \
        }                                                                           \
    } while (0)
#define CHECK_THROWS(stmt)                  \
    do {                                    \
        bool thrown = false;                \
        try {                               \
            stmt;                           \
        } catch (const Error&) {            \
            thrown = true;                  \
        }                                   \
        CHECK(thrown);                      \
    } while (0)

static std::vector<std::pair<std::string, std::function<void()>>>& registry() {
    static std::vector<std::pair<std::string, std::function<void()>>> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define TEST(name)                         \
    static void name();                    \
    static Reg reg_##name(#name, name);    \
    static void name()

// ---- systems (proj/tests/helpers.hpp:24-75, fixtures/quartz.xyz via JSON) --
static AtomicSystem random_system(int64_t n, Vec3 box, uint64_t seed) {
    AtomicSystem s;
    std::vector<double> u(3 * n);
    if (n) gmd_util_rng_uniform(seed, 3 * n, 0.0, 1.0, u.data());
    for (int k = 0; k < 3; ++k) s.lattice[k] = Mat3::identity()[k] * box[k];
    for (int64_t i = 0; i < n; ++i) {
        s.positions.push_back({box.x * u[3 * i], box.y * u[3 * i + 1], box.z * u[3 * i + 2]});
        s.species.push_back(i % 2 ? 8 : 14);
    }
    return s;
}

static AtomicSystem quartz_cell() {
    // alpha-quartz fixture (proj/fixtures/quartz.xyz), values from tests/golden/fixtures.json
    AtomicSystem s;
    s.lattice[0] = {4.9134, 0.0, 0.0};
    s.lattice[1] = {-2.4567, 4.255129219, 0.0};
    s.lattice[2] = {0.0, 0.0, 5.4052};
    const double p[9][3] = {{2.30782398, 0.0, 0.0},          {-1.15391199, 1.9986341941, 3.6034666667},
                            {1.30278801, 2.2564950248, 1.8017333333}, {1.37427798, 1.1369705273, 0.64213776},
                            {0.29750637, 1.7586449062, 2.96150908},   {3.24161565, 0.6216743789, 4.2457846},
                            {0.78491565, 3.6334548401, 1.1594154},    {2.75420637, 2.4964843128, 2.44369092},
                            {-1.08242202, 3.1181586916, 4.76306224}};
    for (int i = 0; i < 9; ++i) {
        s.positions.push_back({p[i][0], p[i][1], p[i][2]});
        s.species.push_back(i < 3 ? 14 : 8);
    }
    return s;
}

static AtomicSystem chain4() {
    AtomicSystem s;
    s.lattice[0] = {12, 0, 0};
    s.lattice[1] = {0, 8, 0};
    s.lattice[2] = {0, 0, 8};
    for (int i = 0; i < 4; ++i) {
        s.positions.push_back({4.5 + i, 4.0, 4.0});
        s.species.push_back(6);
    }
    return s;
}

struct Flat {
    std::vector<double> pos, lat;
    std::vector<int32_t> z;
    uint8_t pbc[3];
};
static Flat flat(const AtomicSystem& s) {
    Flat f;
    for (auto& r : s.positions) f.pos.insert(f.pos.end(), {r.x, r.y, r.z});
    for (int r = 0; r < 3; ++r) f.lat.insert(f.lat.end(), {s.lattice[r].x, s.lattice[r].y, s.lattice[r].z});
    f.z.assign(s.species.begin(), s.species.end());
    for (int k = 0; k < 3; ++k) f.pbc[k] = s.pbc[k];
    return f;
}

using EdgeKey = std::tuple<int64_t, int64_t, int, int, int>;
static std::vector<EdgeKey> keys(const AtomGraph& g) {
    std::vector<EdgeKey> k;
    for (size_t e = 0; e < g.num_edges(); ++e)
        k.emplace_back(g.src[e], g.dst[e], g.image_offset[e][0], g.image_offset[e][1], g.image_offset[e][2]);
    std::sort(k.begin(), k.end());
    return k;
}
static std::vector<EdgeKey> oracle_keys(const AtomicSystem& s, double rc, int brute) {
    Flat f = flat(s);
    void* g = orc_neighbor_list((int64_t)s.size(), f.pos.data(), f.z.data(), f.lat.data(), f.pbc, rc, brute);
    int64_t ne = orc_graph_num_edges(g);
    std::vector<int64_t> src(ne), dst(ne);
    std::vector<int32_t> off(3 * ne);
    orc_graph_get(g, src.data(), dst.data(), off.data(), nullptr, nullptr);
    orc_graph_destroy(g);
    std::vector<EdgeKey> k;
    for (int64_t e = 0; e < ne; ++e) k.emplace_back(src[e], dst[e], off[3 * e], off[3 * e + 1], off[3 * e + 2]);
    std::sort(k.begin(), k.end());
    return k;
}

// ---- neighbour list (test_neighborlist.cpp) ------------------------------
TEST(two_atoms_two_edges) {
    AtomicSystem s = random_system(0, {100, 100, 100}, 0);
    s.positions = {{50, 50, 50}, {51, 50, 50}};
    s.species = {1, 1};
    CHECK(build_neighbor_list(s, 2.0).num_edges() == 2);
}

TEST(self_image_cell) {
    AtomicSystem s;
    for (int k = 0; k < 3; ++k) s.lattice[k] = Mat3::identity()[k] * 2.0;
    s.positions = {{0.3, 0.7, 1.1}};
    s.species = {2};
    AtomGraph g = build_neighbor_list(s, 2.5);
    CHECK(g.num_edges() == 6);
    CHECK(keys(g) == oracle_keys(s, 2.5, 1));
    for (size_t e = 0; e < g.num_edges(); ++e) CHECK(std::abs(g.distance[e] - 2.0) < 1e-12);
}

TEST(quartz_333_vs_oracle_and_invariants) {
    AtomicSystem s = make_supercell(quartz_cell(), {3, 3, 3});
    AtomGraph g = build_neighbor_list(s, 5.0);
    CHECK(keys(g) == oracle_keys(s, 5.0, 1));
    for (size_t e = 1; e < g.num_edges(); ++e) CHECK(g.dst[e] >= g.dst[e - 1]);
    for (size_t e = 0; e < g.num_edges(); e += 97)
        CHECK(std::abs(g.vector[e].norm() - g.distance[e]) <= 1e-12 * g.distance[e]);
}

TEST(randomized_multiset_equality) {
    for (uint64_t seed = 0; seed < 25; ++seed) {
        double box = 4.0 + (seed % 7);
        int64_t n = 5 + (int64_t)seed * 7 % 60;
        AtomicSystem s = random_system(n, {box, box + 1.0, box - 0.5}, seed);
        double rc = 2.0 + 0.37 * (seed % 5);
        CHECK(keys(build_neighbor_list(s, rc)) == oracle_keys(s, rc, 1));
    }
}

TEST(neighbor_errors) {
    AtomicSystem s = random_system(3, {5, 5, 5}, 0);
    CHECK_THROWS(build_neighbor_list(s, 0.0));
    CHECK_THROWS(build_neighbor_list(s, -1.0));
    AtomicSystem empty;
    CHECK_THROWS(build_neighbor_list(empty, 2.0));
}

// ---- partitioner (test_partitioner.cpp) ----------------------------------
TEST(chain_hand_trace) {
    Distributed d = Distributed::create_distributed(chain4(), 1.5, std::nullopt, 2, 1, true);
    const auto& ap = d.atom_parts();
    CHECK(d.graph().num_edges() == 6);
    CHECK(ap.rule.axis == 0);
    CHECK(ap.buckets.pure[0] == std::vector<int64_t>{0});
    CHECK(ap.buckets.pure[1] == std::vector<int64_t>{3});
    CHECK(ap.buckets.to[0][1] == std::vector<int64_t>{1});
    CHECK(ap.buckets.to[1][0] == std::vector<int64_t>{2});
    CHECK(ap.buckets.from[1][0] == std::vector<int64_t>{1});
    const SpanLayout& l0 = ap.parts[0].layout;
    CHECK(l0.node_array == (std::vector<int64_t>{0, 1, 2}));
    CHECK(l0.pure_span().begin == 0 && l0.pure_span().end == 1);
    CHECK(l0.to_span(1).begin == 1 && l0.to_span(1).end == 2);
    CHECK(l0.from_span(1).begin == 2 && l0.from_span(1).end == 3);
    CHECK(l0.owned_end() == 2);
    CHECK(ap.parts[0].owned_edges.size() == 3 && ap.parts[1].owned_edges.size() == 3);
    CHECK(ap.parts[0].border_edge_list.size() == 1);
}

TEST(quartz_partitions_vs_oracle) {
    AtomicSystem s = random_perturb(make_supercell(quartz_cell(), {3, 2, 2}), 0.05, 6);
    Flat f = flat(s);
    for (int p : {2, 3, 4}) {
        Distributed d = Distributed::create_distributed(s, 4.0, std::nullopt, p, 2, true);
        void* o = orc_create((int64_t)s.size(), f.pos.data(), f.z.data(), f.lat.data(), f.pbc, 4.0, 0.0, 0.0, p, 1);
        const auto& ap = d.atom_parts();
        std::vector<int32_t> own(s.size());
        orc_owner(o, own.data());
        CHECK(std::equal(own.begin(), own.end(), ap.owner.begin()));
        for (int i = 0; i < p; ++i) {
            int64_t sz = orc_layout_size(o, i, 0);
            std::vector<int64_t> na(sz), mk(2 + 2 * p);
            orc_layout(o, i, 0, na.data(), mk.data());
            CHECK(na == ap.parts[i].layout.node_array);
            CHECK(mk == ap.parts[i].layout.markers);
            int64_t ne = orc_num_owned_edges(o, i);
            std::vector<int64_t> oe(ne), ls(ne), ld(ne);
            orc_owned_edges(o, i, oe.data(), ls.data(), ld.data());
            CHECK(oe == ap.parts[i].owned_edges);
            CHECK(ls == ap.parts[i].local_src);
            CHECK(ld == ap.parts[i].local_dst);
        }
        for (int i = 0; i < p; ++i)
            for (int j = 0; j < p; ++j) CHECK(ap.buckets.to[i][j] == ap.buckets.from[j][i]);
        orc_destroy(o);
    }
}

TEST(narrow_slab_guard) {
    AtomicSystem s = random_system(200, {40, 10, 10}, 3);
    CHECK_THROWS(Distributed::create_distributed(s, 3.0, std::nullopt, 16, 1, false));
    CHECK_THROWS(Distributed::create_distributed(random_system(3, {10, 10, 10}, 4), 2.0, std::nullopt, 5, 1));
}

// ---- line graph (test_linegraph.cpp) -------------------------------------
TEST(triangle_and_dimer_line_graphs) {
    AtomicSystem tri;
    for (int k = 0; k < 3; ++k) tri.lattice[k] = Mat3::identity()[k] * 20.0;
    tri.positions = {{10, 10, 10}, {11, 10, 10}, {10.5, 10.87, 10}};
    tri.species = {6, 6, 6};
    Distributed d = Distributed::create_distributed(tri, 1.5, 1.5, 1, 1, true);
    CHECK(d.line_parts().parts[0].line_edges.size() == 6);
    AtomicSystem dimer;
    for (int k = 0; k < 3; ++k) dimer.lattice[k] = Mat3::identity()[k] * 25.0;
    dimer.positions = {{12, 12, 12}, {13, 12, 12}};
    dimer.species = {8, 8};
    Distributed d2 = Distributed::create_distributed(dimer, 1.5, 1.5, 1, 1, true);
    CHECK(d2.line_parts().parts[0].line_edges.empty());
}

TEST(distributed_line_union_equals_serial) {
    AtomicSystem s = random_perturb(make_supercell(quartz_cell(), {2, 2, 2}), 0.05, 9);
    Flat f = flat(s);
    void* ph = orc_line_graph((int64_t)s.size(), f.pos.data(), f.z.data(), f.lat.data(), f.pbc, 4.0, 3.0, 0.0, 0);
    std::vector<int64_t> ser(2 * orc_pairs_size(ph));
    orc_pairs_get(ph, ser.data());
    orc_pairs_destroy(ph);
    std::vector<std::pair<int64_t, int64_t>> want;
    for (size_t k = 0; k < ser.size(); k += 2) want.emplace_back(ser[k], ser[k + 1]);
    for (int p : {1, 2, 3}) {
        Distributed d = Distributed::create_distributed(s, 4.0, 3.0, p, 1, true);
        const auto& lg = d.line_parts();
        std::vector<std::pair<int64_t, int64_t>> got;
        for (const auto& part : lg.parts)
            for (const auto& [le, lep] : part.line_edges)
                got.emplace_back(lg.bonds.edge_of_bond[part.layout.node_array[le]],
                                 lg.bonds.edge_of_bond[part.layout.node_array[lep]]);
        std::sort(got.begin(), got.end());
        CHECK(got == want);
    }
}

// ---- engine (test_engine.cpp) ----------------------------------------------
TEST(transfer_transpose_adjoint) {
    AtomicSystem s = random_perturb(make_supercell(quartz_cell(), {3, 2, 2}), 0.05, 3);
    Distributed d = Distributed::create_distributed(s, 4.0, 3.0, 3, 2, true);
    DistributedFeatures x = d.make_atom_features(2), y = d.make_atom_features(2);
    std::vector<double> r(100000);
    gmd_util_rng_uniform(1, (int64_t)r.size(), -1.0, 1.0, r.data());
    size_t k = 0;
    for (int p = 0; p < 3; ++p) {
        const SpanLayout& l = d.atom_parts().parts[p].layout;
        for (auto& v : x.blocks[p]) v = r[k++ % r.size()];
        for (auto& v : y.blocks[p]) v = r[k++ % r.size()];
        for (int64_t row = l.owned_end(); row < l.size(); ++row)
            for (int c = 0; c < 2; ++c) x.row(p, row)[c] = 0.0;
    }
    d.sync_atom_duplicates(x);
    DistributedFeatures tx = x, ty = y;
    d.atom_transfer(tx);
    d.atom_transfer_transpose(ty);
    auto dot = [](const DistributedFeatures& a, const DistributedFeatures& b) {
        double acc = 0;
        for (size_t p = 0; p < a.blocks.size(); ++p)
            for (size_t i = 0; i < a.blocks[p].size(); ++i) acc += a.blocks[p][i] * b.blocks[p][i];
        return acc;
    };
    CHECK(std::abs(dot(tx, y) - dot(x, ty)) <= 1e-12 * std::max(1.0, std::abs(dot(tx, y))));
}

TEST(distribute_aggregate_identity) {
    AtomicSystem s = random_system(25, {8, 8, 8}, 1);
    Distributed d = Distributed::create_distributed(s, 3.0, std::nullopt, 1, 1);
    std::vector<double> feats(25 * 4);
    for (size_t i = 0; i < feats.size(); ++i) feats[i] = 0.5 * i;
    CHECK(d.aggregate(d.distribute_node_features(feats, 4)) == feats);
}

// test_engine.cpp:149-203 (run_layered, worker failure) + edge features
TEST(run_layered_and_worker_failure) {
    auto run = [&](int p) {
        Distributed dist = Distributed::create_distributed(chain4(), 1.5, std::nullopt, p, 1, true);
        std::vector<double> init{1.0, 2.0, 3.0, 4.0};
        DistributedFeatures f = dist.distribute_node_features(init, 1);
        std::vector<Distributed::LayerFn> layers;
        layers.push_back([&dist](int part, DistributedFeatures& feats) {
            const AtomPartition& ap = dist.atom_parts().parts[part];
            std::vector<double> sum(dist.atom_rows(part), 0.0);
            std::vector<int> cnt(dist.atom_rows(part), 0);
            for (std::size_t e = 0; e < ap.owned_edges.size(); ++e) {
                sum[ap.local_dst[e]] += *feats.row(part, ap.local_src[e]);
                cnt[ap.local_dst[e]]++;
            }
            for (std::int64_t r = 0; r < ap.layout.owned_end(); ++r)
                if (ap.layout.local_of(ap.layout.node_array[r]) == r && cnt[r])
                    *feats.row(part, r) = sum[r] / cnt[r];
        });
        dist.run_layered(layers, f);
        return dist.aggregate(f);
    };
    const std::vector<double> serial = run(1);
    CHECK(serial == (std::vector<double>{2.0, 2.0, 3.0, 3.0}));
    CHECK(run(2) == serial);
    Distributed dist = Distributed::create_distributed(chain4(), 1.5, std::nullopt, 2, 1, true);
    std::vector<double> init{5, 6, 7, 8};
    DistributedFeatures f = dist.distribute_node_features(init, 1);
    dist.run_layered(std::vector<Distributed::LayerFn>(3, [](int, DistributedFeatures&) {}), f);
    CHECK(dist.aggregate(f) == init);

    Distributed d2 = Distributed::create_distributed(random_system(40, {10, 8, 8}, 11), 3.0, std::nullopt, 2, 2, true);
    bool thrown = false;
    try {
        d2.parallel_for_partitions([](int p) {
            if (p == 1) throw Error("boom");
        });
    } catch (const Error& e) {
        thrown = true;
        CHECK(std::string(e.what()).find("partition 1") != std::string::npos);
        CHECK(std::string(e.what()).find("boom") != std::string::npos);
    }
    CHECK(thrown);

    // owned-edge features round trip; every edge lands in exactly one block
    std::vector<double> ef(d2.graph().num_edges() * 3);
    for (std::size_t i = 0; i < ef.size(); ++i) ef[i] = 0.25 * i - 7.0;
    DistributedFeatures eb = d2.distribute_edge_features(ef, 3);
    std::size_t rows = 0;
    for (int i = 0; i < 2; ++i) rows += eb.blocks[i].size() / 3;
    CHECK(rows == d2.graph().num_edges());
    CHECK(d2.aggregate_edges(eb) == ef);
    bool shape = false;
    try {
        d2.distribute_edge_features(std::vector<double>(5), 3);
    } catch (const Error& e) {
        shape = std::string(e.what()) == "edge feature shape mismatch";
    }
    CHECK(shape);
}

// ---- potential (test_potential.cpp) ---------------------------------------
static void compare_to_oracle(const AtomicSystem& s, const ToyPotentialParams& prm, const PotentialOutput& out) {
    Flat f = flat(s);
    std::vector<double> blob = prm.blob(), pa(s.size()), fo(3 * s.size()), st(9);
    double e = 0;
    int rc = orc_forward_serial((int64_t)s.size(), f.pos.data(), f.z.data(), f.lat.data(), f.pbc,
                                prm.feature_width, prm.basis_count, prm.layers, prm.r_atom, prm.r_3body,
                                blob.data(), &e, pa.data(), fo.data(), st.data());
    CHECK(rc == 0);
    double df = 0, da = 0, ds = 0;
    for (size_t i = 0; i < s.size(); ++i) {
        da = std::max(da, std::abs(out.per_atom[i] - pa[i]));
        for (int k = 0; k < 3; ++k) df = std::max(df, std::abs(out.forces[i][k] - fo[3 * i + k]));
    }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) ds = std::max(ds, std::abs(out.stress[a][b] - st[3 * a + b]));
    CHECK(std::abs(out.energy - e) / s.size() <= 2e-6);  // tests/conftest.py tolerances
    CHECK(da <= 2e-5);
    CHECK(df <= 2e-4);
    CHECK(ds <= 2e-6);
}

TEST(isolated_atom_closed_form) {
    AtomicSystem s;
    for (int k = 0; k < 3; ++k) s.lattice[k] = Mat3::identity()[k] * 50.0;
    s.positions = {{25, 25, 25}};
    s.species = {26};
    ToyPotentialParams prm = ToyPotentialParams::init(5);
    Distributed d = Distributed::create_distributed(s, prm.r_atom, std::nullopt, 1, 1);
    PotentialOutput out = forward_distributed(d, prm);
    double expected = 0.0;
    for (int f = 0; f < prm.feature_width; ++f) {
        double h = prm.embedding[26 * prm.feature_width + f];
        for (int l = 0; l < prm.layers; ++l) h += std::tanh(prm.layer_b[l * prm.feature_width + f]);
        expected += prm.readout[f] * h;
    }
    CHECK(std::abs(out.energy - expected) < 1e-5);
    CHECK(out.forces[0].norm() == 0.0);
}

TEST(distributed_equals_serial_oracle) {
    AtomicSystem s = random_perturb(make_supercell(quartz_cell(), {3, 3, 3}), 0.05, 1);
    for (double r3 : {0.0, 3.0}) {
        ToyPotentialParams prm = ToyPotentialParams::init(12345, 16, 8, 2, 5.0, r3);
        std::optional<double> tb;
        if (r3 > 0) tb = r3;
        PotentialOutput ref;
        for (int p : {1, 2, 3, 4}) {
            Distributed d = Distributed::create_distributed(s, 5.0, tb, p, 2, true);
            StepTiming t;
            PotentialOutput out = forward_distributed(d, prm, &t);
            compare_to_oracle(s, prm, out);
            CHECK(t.forward_pass > 0 && t.backward_pass > 0);
            if (p == 1) ref = out;
            else {  // partition-invariant on the GPU: bitwise equal
                CHECK(out.energy == ref.energy);
                for (size_t i = 0; i < s.size(); ++i)
                    for (int k = 0; k < 3; ++k) CHECK(out.forces[i][k] == ref.forces[i][k]);
            }
        }
    }
}

TEST(forward_argument_errors) {
    AtomicSystem s = make_supercell(quartz_cell(), {2, 2, 2});
    Distributed d = Distributed::create_distributed(s, 4.0, std::nullopt, 1, 1);
    CHECK_THROWS(forward_distributed(d, ToyPotentialParams::init(1, 16, 8, 2, 5.0)));
    CHECK_THROWS(forward_distributed(d, ToyPotentialParams::init(1, 16, 8, 2, 4.0, 3.0)));
}

// md.cpp run_md / velocity_verlet_step through the drop-in header, against
// the oracle's restatement (orc_md_run, pinned to the reference's run_md)
TEST(md_run_vs_oracle) {
    AtomicSystem s = random_perturb(make_supercell(quartz_cell(), {3, 3, 3}), 0.05, 1);
    ToyPotentialParams prm = ToyPotentialParams::init(12345, 16, 8, 2, 5.0);
    MDOptions o;
    o.dt = 1.0;
    o.steps = 10;
    o.partitions = 2;
    o.allow_narrow = true;
    o.seed = 9;
    o.init_temperature = 300.0;
    MDResult res = run_md(s, prm, o);
    const int64_t n = (int64_t)s.size();
    std::vector<double> pos(3 * n), lat(9), blob = prm.blob();
    std::vector<int32_t> z(s.species.begin(), s.species.end());
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) pos[3 * i + k] = s.positions[i][k];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) lat[3 * r + k] = s.lattice[r][k];
    uint8_t pbc[3] = {1, 1, 1};
    std::vector<double> op(3 * n), ov(3 * n), of(3 * n), rec(4 * 11);
    CHECK(orc_md_run(n, pos.data(), z.data(), lat.data(), pbc, 16, 8, 2, 5.0, 0.0, blob.data(),
                     1.0, 10, 300.0, 9, op.data(), ov.data(), of.data(), rec.data()) == 0);
    CHECK(res.records.size() == 11);
    double dx = 0, dv = 0, de = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            dx = std::max(dx, std::abs(res.state.system.positions[i][k] - op[3 * i + k]));
            dv = std::max(dv, std::abs(res.state.velocities[i][k] - ov[3 * i + k]));
        }
    for (int st = 0; st <= 10; ++st) de = std::max(de, std::abs(res.records[st].potential - rec[4 * st]));
    CHECK(dx < 1e-5 && dv < 1e-5 && de / n < 2e-6);
    CHECK(std::abs(res.state.kinetic_energy() - rec[4 * 10 + 1]) / n < 1e-6);
    // one more step through velocity_verlet_step continues the trajectory
    MDState st = res.state;
    StepTiming t;
    velocity_verlet_step(st, prm, o, &t);
    CHECK(st.step == 11 && t.graph_creation > 0);
    MDState fresh = init_md_state(s, o);
    CHECK_THROWS(velocity_verlet_step(fresh, prm, o));  // no forces yet
}

// dump formats through the header (compared with the reference's own dumps
// by tests/test_dumps.py): test_cpp_api --dump DIR P
static int dump_mode(const std::string& dir, int p) {
    AtomicSystem s = random_perturb(make_supercell(quartz_cell(), {3, 3, 3}), 0.05, 1);
    Distributed d = Distributed::create_distributed(s, 5.0, 3.0, p, 1, true);
    d.graph().dump_csv(dir + "/g.csv");
    d.line_parts().dump_csv(dir + "/l.csv");
    std::FILE* f = std::fopen((dir + "/plan.json").c_str(), "w");
    if (!f) return 2;
    const std::string js = partition_plan_to_json(d.atom_parts());
    std::fwrite(js.data(), 1, js.size(), f);
    std::fclose(f);
    return 0;
}

// parameter files, CPU only (tests/test_cli.py): --params-save PATH SEED L R3
// writes ToyPotentialParams::init(...).save(PATH); --params-copy IN OUT loads
// IN and saves it to OUT; errors print "error: <text>" and exit 3
static int params_mode(int argc, char** argv) {
    try {
        const std::string m = argv[1];
        if (m == "--params-save" && argc > 5) {
            ToyPotentialParams::init(std::strtoull(argv[3], nullptr, 10), 16, 8, std::atoi(argv[4]), 5.0,
                                     std::atof(argv[5]))
                .save(argv[2]);
            return 0;
        }
        if (m == "--params-copy" && argc > 3) {
            ToyPotentialParams::load(argv[2]).save(argv[3]);
            return 0;
        }
        return 2;
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 3;
    }
}

int main(int argc, char** argv) {
    if (argc > 3 && std::string(argv[1]) == "--dump") return dump_mode(argv[2], std::atoi(argv[3]));
    if (argc > 1 && std::string(argv[1]).rfind("--params-", 0) == 0) return params_mode(argc, argv);
    std::string only = argc > 1 ? argv[1] : "";
    for (auto& [name, fn] : registry()) {
        if (!only.empty() && name != only) continue;
        int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("  exception: %s\n", e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name.c_str());
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
