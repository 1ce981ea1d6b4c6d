// C ABI + host orchestration of the graphmd B200 path.
//
// gmd_build   == Distributed::create_distributed (proj/src/engine.cpp:44-65)
// gmd_forward == forward_distributed             (proj/src/potential.cpp:563-985)
//
// All per-atom / per-edge work runs in the kernels of gmd_graph.cu,
// gmd_partition.cu, gmd_linegraph.cu and gmd_model.cu; the host only does
// O(1)/O(p) scalar geometry (3x3 lattice algebra, slab walls), sizes buffers
// and -- for the parity views only -- reshapes device results into the
// reference's per-partition containers.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <random>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/graphmd_b200.h"
#include "gmd_builders.cuh"
#include "gmd_comm.cuh"
#include "gmd_common.cuh"
#include "gmd_generic.cuh"
#include "gmd_graph.cuh"
#include "gmd_md.cuh"
#include "gmd_model.cuh"
#include "gmd_partition.cuh"
#include "gmd_wide.cuh"

namespace gmd {
void launch_bond_owner(int64_t n, const int32_t* brow, const int32_t* owner, int32_t* bown,
                       cudaStream_t s);
void launch_bond_req(int64_t n, const int32_t* brow, const int32_t* bedge, const int32_t* esrc,
                     const int32_t* owner, unsigned long long* breq, cudaStream_t s);
void launch_line_count(int64_t nb, const int32_t* bedge, const int32_t* esrc, const int32_t* brow,
                       int32_t* cnt, cudaStream_t s);
void launch_line_fill(int64_t nb, const int32_t* bedge, const int32_t* esrc, const int32_t* brow,
                      const int32_t* brev, const int32_t* lpos, int32_t* pairs, cudaStream_t s);
int tb_grid_size(int64_t n);
void launch_bond_halo_flag(int64_t nb, const int32_t* bedge, const int32_t* esrc,
                           const int32_t* owner, int j, int32_t* flag, cudaStream_t s);
void launch_bond_halo_assign(int64_t nb, const int32_t* bedge, const int32_t* esrc,
                             const int32_t* owner, int j, const int32_t* pos, int32_t base,
                             int32_t* brev, cudaStream_t s);
void launch_bond_send_plan(int64_t n_own, const int32_t* nodes, const int32_t* brow, int64_t nb,
                           const int32_t* bedge, const int32_t* esrc, const uint32_t* img,
                           const int32_t* owner, int r, const int32_t* crow, int32_t from0,
                           int phase, const int32_t* offs, int32_t* cnt_or_fill, int32_t* bcen,
                           int32_t* xs, int32_t nrows, cudaStream_t s);
}  // namespace gmd

using namespace gmd;

namespace {

// ---------------------------------------------------------------------------
// device buffer arena: grow-only, reused across builds / steps
// ---------------------------------------------------------------------------
struct DBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <typename T>
    T* get(size_t count) {
        size_t bytes = std::max<size_t>(count * sizeof(T), 16);
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            size_t nc = std::max(bytes, cap + cap / 4);
            GMD_CUDA(cudaMalloc(&p, nc));
            cap = nc;
        }
        return static_cast<T*>(p);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// ---- host fp64 lattice algebra with the reference's operand order -------
struct V3 {
    double x, y, z;
};
inline V3 vmul(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 vdiv(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 vcross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double vnorm(V3 a) { return std::sqrt(vdot(a, a)); }
inline V3 row3(const double* L, int k) { return {L[3 * k], L[3 * k + 1], L[3 * k + 2]}; }
inline double det3(const double* L) { return vdot(row3(L, 0), vcross(row3(L, 1), row3(L, 2))); }
// Mat3::inverse (system.cpp:55-70)
void inverse3(const double* L, double* inv) {
    double d = det3(L);
    if (std::abs(d) < 1e-10) raise(kConfig, "lattice is singular (|det| < 1e-10)");
    V3 bc = vdiv(vcross(row3(L, 1), row3(L, 2)), d);
    V3 ca = vdiv(vcross(row3(L, 2), row3(L, 0)), d);
    V3 ab = vdiv(vcross(row3(L, 0), row3(L, 1)), d);
    double r[9] = {bc.x, ca.x, ab.x, bc.y, ca.y, ab.y, bc.z, ca.z, ab.z};
    std::memcpy(inv, r, sizeof r);
}
// perpendicular_width (system.cpp:87-93)
double perp_width(const double* L, int axis) {
    double area = vnorm(vcross(row3(L, (axis + 1) % 3), row3(L, (axis + 2) % 3)));
    if (area <= 0.0) raise(kConfig, "degenerate cell");
    return std::abs(det3(L)) / area;
}

double dec_ordered(unsigned long long u) {
    u = (u & 0x8000000000000000ull) ? (u & ~0x8000000000000000ull) : ~u;
    double d;
    std::memcpy(&d, &u, 8);
    return d;
}

// ---- small generic kernels for the feature API --------------------------
__global__ void k_copy_rows(int64_t nr, const int32_t* __restrict__ dst_rows,
                            const int32_t* __restrict__ src_rows, uint32_t* buf, int wwords) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nr * wwords) return;
    int64_t k = t / wwords;
    int c = (int)(t - k * wwords);
    buf[(int64_t)dst_rows[k] * wwords + c] = buf[(int64_t)src_rows[k] * wwords + c];
}

template <typename T>
__global__ void k_transpose_add(int64_t nr, const int32_t* __restrict__ to_rows,
                                const int32_t* __restrict__ from_rows, T* buf, int width) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nr * width) return;
    int64_t k = t / width;
    int c = (int)(t - k * width);
    T* a = buf + (int64_t)to_rows[k] * width + c;
    T* b = buf + (int64_t)from_rows[k] * width + c;
    *a += *b;
    *b = T(0);
}

// duplicates grouped by canonical row, dups in ascending row order
template <typename T>
__global__ void k_dup_fold(int64_t ng, const int32_t* __restrict__ gcanon,
                           const int32_t* __restrict__ gstart, const int32_t* __restrict__ dups,
                           T* buf, int width) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ng * width) return;
    int64_t g = t / width;
    int c = (int)(t - g * width);
    T* cr = buf + (int64_t)gcanon[g] * width + c;
    for (int k = gstart[g]; k < gstart[g + 1]; ++k) {
        T* d = buf + (int64_t)dups[k] * width + c;
        *cr += *d;
        *d = T(0);
    }
}

__global__ void k_gather_rows(int64_t nr, const int32_t* __restrict__ idx,
                              const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                              int wwords) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nr * wwords) return;
    int64_t k = t / wwords;
    int c = (int)(t - k * wwords);
    int64_t r = idx ? idx[k] : k;
    dst[k * wwords + c] = src[r * wwords + c];
}

// for every FROM row: the row of the same id inside the sender's TO span
// (engine.cpp:122-143 copies TO_j[i] -> FROM_i[j] row by row)
__global__ void k_api_src(int64_t nfrom, const int32_t* __restrict__ xdst,
                          const int32_t* __restrict__ list_off, int p, int corrupt,
                          int32_t* __restrict__ out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nfrom) return;
    const int r = xdst[k], stride = 1 + 2 * p;
    int lo = 0, hi = p - 1;  // partition: last i with list_off[i*stride] <= r
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (list_off[mid * stride] <= r) lo = mid; else hi = mid - 1;
    }
    const int i = lo;
    int j = 0;
    for (; j < p; ++j)
        if (r < list_off[i * stride + 2 + p + j]) break;
    const int fb = list_off[i * stride + 1 + p + j];
    out[k] = corrupt ? list_off[j * stride] + (r - fb) : list_off[j * stride + 1 + i] + (r - fb);
}

__global__ void k_to_f32(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = (float)a[i];
}

// --------------------------------------------------------------------------
// host RNG of the reference (system.hpp:121-149): mt19937_64 + Box-Muller
struct HostRng {
    std::mt19937_64 gen;
    bool have = false;
    double spare = 0.0;
    explicit HostRng(uint64_t s) : gen(s) {}
    double uniform() { return (double)(gen() >> 11) * 0x1.0p-53; }
    double normal() {
        if (have) {
            have = false;
            return spare;
        }
        double u1 = 0.0;
        while (u1 == 0.0) u1 = uniform();
        double u2 = uniform();
        double r = std::sqrt(-2.0 * std::log(u1));
        double a = 2.0 * 3.14159265358979323846 * u2;
        spare = r * std::sin(a);
        have = true;
        return r * std::cos(a);
    }
};

// one layout (atoms or bonds): lists in super-row space
struct LayoutState {
    bool ready = false;
    int p = 1;
    int64_t nid = 0;
    std::vector<int32_t> list_off;  // p(1+2p)+1
    int64_t rows = 0;
    int64_t nfrom = 0;
    DBuf node_array, crow, list_off_d, xdst, xsrc, xapi, owner, req;
    bool api_ready = false;
    bool api_corrupt = false;
    // duplicates (host + device groups)
    bool dups_ready = false;
    std::vector<int32_t> h_nodes;  // host copy of node_array (lazy)
    DBuf g_canon, g_start, g_dups, d_canon, d_dup;
    int64_t ngroups = 0, ndups = 0;
    int64_t base(int i) const { return list_off[(size_t)i * (1 + 2 * p)]; }
};

}  // namespace

struct gmd_handle {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;

    bool built = false;
    int64_t n = 0, ne = 0, nb = 0;
    int p = 1;
    double rc = 0, r3 = 0, tau = 0;
    bool has_lg = false, allow_narrow = false, corrupted = false;
    bool z_pending = false;  // species upload on the side stream (ev[6])
    Geom geom{};
    double lat[9]{};
    int axis = 0;
    std::vector<double> bounds;
    double t_graph = 0.0;

    LayoutState atoms, bonds;

    DBuf pos, Z, cell, fw, bin, bin_cnt, bin_start, fill, s_id, s_w, s_p, s_c, deg, bcnt, flags;
    DBuf pos4, cell4;  // per-atom records of the neighbour-list emit
    DBuf zs, zmask;    // per-row species byte, species presence mask (layer-0 conv)
    // the free builders' own wrap buffers (a built graph's pos / cell / fw /
    // flags stay intact: its export re-runs the emit from them)
    DBuf fr_pos, fr_cell, fr_fw, fr_bin, fr_cnt, fr_flags;
    DBuf row, src, img, vd, ed, ebond, edst, lsrc, counts, scan_tmp, sel_ws, sel_out, small;
    DBuf brow, bedge, brev, lcnt, lpairs, slab, feat_tmp, flagtmp, ebid;
    int nl_cap = 0;
    int emit_cap = 0;     // slab row capacity of the current build
    bool img_ok = false;  // per-edge packed images written (else derived on export)

    // model
    bool params_set = false;
    ModelConst mc{};
    uint64_t mc_ver = 0;  // globally unique id of the current parameter set
    bool generic = false;  // widths other than the tuned F = 16, K = 8 (gmd_generic.cu)
    GenModel gm{};
    DBuf gpar;             // fp32 parameter tables of the generic kernels
    DBuf TT, SMR;          // generic three-body scratch rows (t per bond, m_bar_3 per slot)
    int F = 16, K = 8, L = 0;
    double p_r_atom = 0, p_r3 = 0;
    std::vector<DBuf> H;
    bool ctab_ok = false;  // chunk records of the tcgen05 backward (per build)
    int max_bonds = 0;     // max in-bonds of a center (three-body), per build
    int ctab_grid = 0;
    DBuf ccnt, cstart, ctab, ccta;
    DBuf TH, MB, HB, GRAD, TP, TH3, TH4, QB, VIN, VOUT, e_part, v_part, v_grp, v3_part, red, per_atom,
        forces, conv_tmp, exp_tmp, nonfin;
    DBuf md_part, md_out, md_bad;  // on-device MD observables / non-finite flag
    DBuf md_pos, md_vel, md_frc, md_mass, md_z;  // device state of gmd_md_run
    cudaEvent_t ev[8] = {};
    cudaStream_t side = nullptr;  // D2H of per-atom energies during the backward
    void* ipc_window = nullptr;   // exported, not yet attached IPC window
    int ipc_rank = 0, ipc_world = 1;
    int64_t ipc_rows = 0;

    // one rank per GPU: transport + this rank's plan
    std::unique_ptr<Transport> comm;
    int64_t n_own = 0;
    // partitions of a caller-supplied graph (gmd_build_partitions): no positions
    // or per-edge geometry on the device, so no model evaluation / graph export
    bool graph_only = false;
    DBuf cmask, bmask;  // two-hop closure masks per node / edge-table masks per bond
    bool closure_ready = false;
    DBuf nodes, xsend, sendbuf;
    // the same atoms as evaluated: interior (no halo in-edge) first, then border
    DBuf nodes_x;
    int64_t n_int = 0;
    std::vector<int64_t> soff, scnt, roff, rcnt;
    // ... and its bond halo plan (three-body): rows nb .. nb + nb_halo of the
    // per-bond arrays are received, b_* as above in bond rows
    int64_t nb_halo = 0;
    DBuf bxsend, bsendbuf, bcen;
    std::vector<int64_t> b_soff, b_scnt, b_roff, b_rcnt;

    // profiler: event pairs recorded on `stream` around every launch
    bool prof = false;
    std::vector<cudaEvent_t> pev;
    int pidx = 0;
    std::vector<std::pair<const char*, int>> precs;

    // host caches for views (invalidated per build)
    bool hc_ready = false;
    std::vector<int32_t> h_owner, h_row, h_src, h_lsrc, h_crow;
    bool hcb_ready = false;
    bool line_dev_ready = false;  // line edges built on the device (lcnt / lpairs)
    int64_t nline = 0;
    std::vector<int32_t> h_bedge, h_bown, h_pairs;
};

namespace {

struct Prof {
    gmd_handle* h;
    const char* name;
    int a = -1;
    Prof(gmd_handle* h_, const char* n) : h(h_), name(n) {
        if (h->prof && h->pidx + 2 <= (int)h->pev.size()) {
            a = h->pidx;
            h->pidx += 2;
            cudaEventRecord(h->pev[a], h->stream);
        }
    }
    ~Prof() {
        if (a >= 0) {
            cudaEventRecord(h->pev[a + 1], h->stream);
            h->precs.emplace_back(name, a);
        }
    }
};
#define GMD_PROF_CAT2(a, b) a##b
#define GMD_PROF_CAT(a, b) GMD_PROF_CAT2(a, b)
#define PROF(name) Prof GMD_PROF_CAT(prof_, __LINE__)(h, name)

void sync(gmd_handle* h) { GMD_CUDA(cudaStreamSynchronize(h->stream)); }

void check_flags(int e);

void read_flags(gmd_handle* h, int32_t out[2]) {
    GMD_CUDA(cudaMemcpyAsync(out, h->flags.as<int32_t>(), 8, cudaMemcpyDeviceToHost, h->stream));
    sync(h);
    check_flags(out[1]);
}

// error bits of the device flag word (flags[1])
void check_flags(int e) {
    if (e & kErrImgRange)
        raise(kConfig, "periodic image offset exceeds the packed range (+-511 cells)");
    if (e & kErrQRange) raise(kConfig, "neighbour stencil exceeds 127 cell images per axis");
    if (e & kErrCap) raise(kRuntime, "internal: neighbour buffer overflow");
    if (e & 8) raise(kRuntime, "internal: edge endpoint missing from partition layout");
    if (e & 16) raise(kConfig, "an atom has more than 64 three-body bonds (unsupported)");
    if (e & 32) raise(kRuntime, "internal: reverse bond not found (graph not symmetric)");
}

void scan_i32(gmd_handle* h, const int32_t* in, int32_t* out, int64_t n) {
    size_t tb = scan_tmp_bytes(n);
    void* tmp = h->scan_tmp.get<char>(tb);
    exclusive_scan_i32(in, out, n, tmp, tb, h->stream);
}

template <typename T>
void d2h(gmd_handle* h, std::vector<T>& v, const void* d, size_t count) {
    v.resize(count);
    if (count)
        GMD_CUDA(cudaMemcpyAsync(v.data(), d, count * sizeof(T), cudaMemcpyDeviceToHost, h->stream));
}

// ensure_periodic (system.cpp:242-270) with the per-atom projections on the GPU
void ensure_periodic_dev(gmd_handle* h, const uint8_t* pbc, double cutoff) {
    if (!pbc || (pbc[0] && pbc[1] && pbc[2])) return;
    if (cutoff <= 0.0) raise(kConfig, "cutoff must be positive");
    double* d = h->small.get<double>(4);
    for (int k = 0; k < 3; ++k) {
        if (pbc[k]) continue;
        V3 dir = row3(h->lat, k);
        double len = vnorm(dir);
        if (len == 0.0)
            dir = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
        else
            dir = vdiv(dir, len);
        double dv[3] = {dir.x, dir.y, dir.z};
        double lo = 0.0, hi = 0.0;
        if (h->n > 0) {
            launch_minmax_proj(h->pos.as<double>(), h->n, dv, d, h->stream);
            unsigned long long mm[2];
            GMD_CUDA(cudaMemcpyAsync(mm, d, 16, cudaMemcpyDeviceToHost, h->stream));
            sync(h);
            lo = dec_ordered(mm[0]);
            hi = dec_ordered(mm[1]);
        }
        double extent = hi - lo + 2.0 * cutoff;
        V3 nr = vmul(dir, extent);
        h->lat[3 * k] = nr.x;
        h->lat[3 * k + 1] = nr.y;
        h->lat[3 * k + 2] = nr.z;
        V3 sh = vmul(dir, cutoff - lo);
        double add[3] = {sh.x, sh.y, sh.z};
        launch_shift(h->pos.as<double>(), h->n, add, h->stream);
    }
}

// PURE/TO/FROM layout of an id space (atoms or bonds) on the GPU
void build_layout(gmd_handle* h, LayoutState& ls, const int32_t* owner,
                  const unsigned long long* req, int64_t nid, int p, int only = -1) {
    cudaStream_t s = h->stream;
    ls.p = p;
    ls.nid = nid;
    ls.api_ready = false;
    ls.dups_ready = false;
    ls.h_nodes.clear();
    const int64_t nl = layout_nlists(p), nch = layout_chunks(nid);
    LayoutWs lw{};
    lw.counts = h->counts.get<int32_t>(nl * nch + 1);
    lw.scan_tmp_bytes = scan_tmp_bytes(nl * nch);
    lw.scan_tmp = h->scan_tmp.get<char>(lw.scan_tmp_bytes);
    int32_t* lo_d = ls.list_off_d.get<int32_t>(nl + 1);
    { PROF("part_layout_plan"); launch_layout_plan(owner, req, nid, p, lw, lo_d, only, s); }
    d2h(h, ls.list_off, lo_d, nl + 1);
    sync(h);
    ls.rows = ls.list_off[nl];
    int32_t* na = ls.node_array.get<int32_t>(ls.rows);
    int32_t* cr = ls.crow.get<int32_t>(nid);
    { PROF("part_layout_fill"); launch_layout_fill(owner, req, nid, p, lw, na, cr, only, s); }
    const int stride = 1 + 2 * p;
    std::vector<int32_t> rp(3 * p + 1);
    int32_t* ranges = rp.data();
    int32_t* prefix = rp.data() + 2 * p;
    prefix[0] = 0;
    for (int i = 0; i < p; ++i) {
        ranges[2 * i] = ls.list_off[i * stride + 1 + p];
        ranges[2 * i + 1] = ls.list_off[(i + 1) * stride];
        prefix[i + 1] = prefix[i] + ranges[2 * i + 1] - ranges[2 * i];
    }
    ls.nfrom = only >= 0 ? 0 : prefix[p];  // rank mode exchanges through the transport
    int32_t* sm = h->small.get<int32_t>(3 * p + 1);
    GMD_CUDA(cudaMemcpyAsync(sm, rp.data(), sizeof(int32_t) * rp.size(), cudaMemcpyHostToDevice, s));
    PROF("part_from_src");
    launch_from_src(na, cr, sm, p, ls.nfrom, sm + 2 * p, ls.xdst.get<int32_t>(ls.nfrom),
                    ls.xsrc.get<int32_t>(ls.nfrom), s);
    sync(h);  // rp is a host temporary
    ls.ready = true;
}

// one rank per GPU: this rank's atoms (ascending), the canonical rows of its
// TO blocks packed per peer, and the FROM spans peers fill; checked against
// the peers' plans (engine.cpp:132-133 "transfer plan misalignment")
void build_rank_plan(gmd_handle* h, const int32_t* ownp, int r) {
    cudaStream_t s = h->stream;
    LayoutState& A = h->atoms;
    const int W = h->p, stride = 1 + 2 * W;
    const int64_t n = h->n;
    int32_t* flag = h->flagtmp.get<int32_t>(n + 1);
    launch_owned_flags(ownp, n, r, flag, s);
    scan_i32(h, flag, flag, n);
    int32_t nown = 0;
    GMD_CUDA(cudaMemcpyAsync(&nown, flag + n, 4, cudaMemcpyDeviceToHost, s));
    sync(h);
    h->n_own = nown;
    launch_owned_compact(ownp, n, r, flag, h->nodes.get<int32_t>(nown), s);
    {  // interior atoms first: their layer updates overlap the halo exchange
        int32_t* pos = h->counts.get<int32_t>(nown + 1);
        launch_flag_interior(nown, h->nodes.as<int32_t>(), h->row.as<int32_t>(), h->src.as<int32_t>(),
                             ownp, r, pos, s);
        scan_i32(h, pos, pos, nown);
        launch_split_nodes(nown, h->nodes.as<int32_t>(), pos, h->nodes_x.get<int32_t>(std::max(1, nown)),
                           s);
        int32_t ni = 0;
        GMD_CUDA(cudaMemcpyAsync(&ni, pos + nown, 4, cudaMemcpyDeviceToHost, s));
        sync(h);
        h->n_int = ni;
    }
    const int32_t t0 = A.list_off[(size_t)r * stride + 1], t1 = A.list_off[(size_t)r * stride + 1 + W];
    launch_send_rows(t0, t1, A.node_array.as<int32_t>(), A.crow.as<int32_t>(),
                     h->xsend.get<int32_t>(std::max(1, t1 - t0)), s);
    h->soff.assign(W, 0);
    h->scnt.assign(W, 0);
    h->roff.assign(W, 0);
    h->rcnt.assign(W, 0);
    for (int j = 0; j < W; ++j) {
        h->soff[j] = A.list_off[(size_t)r * stride + 1 + j] - t0;
        h->scnt[j] = A.list_off[(size_t)r * stride + 2 + j] - A.list_off[(size_t)r * stride + 1 + j];
        h->roff[j] = A.list_off[(size_t)r * stride + 1 + W + j];
        h->rcnt[j] = A.list_off[(size_t)r * stride + 2 + W + j] - h->roff[j];
    }
    std::vector<int64_t> all((size_t)W * W);
    h->comm->allgather_i64(s, h->scnt.data(), W, all.data());
    for (int j = 0; j < W; ++j)
        if (j != r && all[(size_t)j * W + r] != h->rcnt[j])
            raise(kRuntime, "transfer plan misalignment");
    sync(h);
}

// one rank per GPU, three-body: halo bond rows (see gmd_linegraph.cu)
void build_bond_rank_plan(gmd_handle* h, const int32_t* ownp, int r) {
    cudaStream_t s = h->stream;
    LayoutState& A = h->atoms;
    const int W = h->p, stride = 1 + 2 * W;
    const int64_t nb = h->nb;
    const int32_t* be = h->bedge.as<int32_t>();
    const int32_t* es = h->src.as<int32_t>();
    int32_t* bv = h->brev.as<int32_t>();
    h->b_soff.assign(W, 0);
    h->b_scnt.assign(W, 0);
    h->b_roff.assign(W, 0);
    h->b_rcnt.assign(W, 0);
    // receive rows: per source rank j, bonds (w -> u) with owner(w) = j in (u, row) order
    int32_t* flag = h->flagtmp.get<int32_t>(nb + 1);
    int64_t base = nb;
    for (int j = 0; j < W; ++j) {
        if (j == r) continue;
        launch_bond_halo_flag(nb, be, es, ownp, j, flag, s);
        scan_i32(h, flag, flag, nb + 1);
        int32_t c = 0;
        GMD_CUDA(cudaMemcpyAsync(&c, flag + nb, 4, cudaMemcpyDeviceToHost, s));
        sync(h);
        launch_bond_halo_assign(nb, be, es, ownp, j, flag, (int32_t)base, bv, s);
        h->b_roff[j] = base;
        h->b_rcnt[j] = c;
        base += c;
    }
    h->nb_halo = base - nb;
    // send rows: per FROM row x (grouped by owner, ascending id), the slots
    // (x -> w) at centers owned here, in x's canonical row order
    const int32_t from0 = A.list_off[(size_t)r * stride + 1 + W];
    const int32_t from1 = A.list_off[(size_t)r * stride + 1 + 2 * W];
    const int32_t nfr = from1 - from0;
    int32_t* cnt = h->counts.get<int32_t>(nfr + 1);
    GMD_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nfr + 1), s));
    int32_t* bcen = h->bcen.get<int32_t>(std::max<int64_t>(1, nb));
    const int32_t* crow = A.crow.as<int32_t>();
    const uint32_t* img = h->img.as<uint32_t>();
    launch_bond_send_plan(h->n_own, h->nodes.as<int32_t>(), h->brow.as<int32_t>(), nb, be, es, img,
                          ownp, r, crow, from0, 0, nullptr, cnt, bcen, nullptr, nfr, s);
    int32_t* offs = h->feat_tmp.get<int32_t>(nfr + 1);
    scan_i32(h, cnt, offs, nfr + 1);
    std::vector<int32_t> hoffs;
    d2h(h, hoffs, offs, nfr + 1);
    sync(h);
    const int32_t nsend = hoffs[nfr];
    int32_t* xs = h->bxsend.get<int32_t>(std::max(1, nsend));
    GMD_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nfr + 1), s));
    launch_bond_send_plan(h->n_own, h->nodes.as<int32_t>(), h->brow.as<int32_t>(), nb, be, es, img,
                          ownp, r, crow, from0, 1, offs, cnt, bcen, xs, nfr, s);
    for (int j = 0; j < W; ++j) {
        if (j == r) continue;
        const int32_t a0 = A.list_off[(size_t)r * stride + 1 + W + j] - from0;
        const int32_t a1 = A.list_off[(size_t)r * stride + 2 + W + j] - from0;
        h->b_soff[j] = hoffs[a0];
        h->b_scnt[j] = hoffs[a1] - hoffs[a0];
    }
    std::vector<int64_t> all((size_t)W * W);
    h->comm->allgather_i64(s, h->b_scnt.data(), W, all.data());
    for (int j = 0; j < W; ++j)
        if (j != r && all[(size_t)j * W + r] != h->b_rcnt[j])
            raise(kRuntime, "bond transfer plan misalignment");
    sync(h);
}

// host copies queued on the side stream never outlive the API call that
// queued them (also on error paths): the caller may reuse its buffers
struct DrainSide {
    cudaStream_t side;
    ~DrainSide() { cudaStreamSynchronize(side); }
};

// equal-count walls b_k = (s[c-1] + s[c]) / 2, c = n k / p, over the sorted
// wrapped fractions (partitioner.cpp:77-85): radix select of the needed order
// statistics on the device
void quantile_walls(gmd_handle* h, const double* fw, int64_t n, int p, double* bounds) {
    cudaStream_t s = h->stream;
    std::vector<int64_t> ranks;
    for (int k = 1; k < p; ++k) {
        int64_t c = n * k / p;
        if (c >= 1 && c < n) {
            ranks.push_back(c - 1);
            ranks.push_back(c);
        }
    }
    std::sort(ranks.begin(), ranks.end());
    ranks.erase(std::unique(ranks.begin(), ranks.end()), ranks.end());
    std::vector<double> vals(ranks.size());
    if (!ranks.empty()) {
        void* ws = h->sel_ws.get<char>(select_ws_bytes((int)ranks.size()));
        double* so = h->sel_out.get<double>(ranks.size());
        { PROF("part_select"); launch_select(fw, n, ranks.data(), (int)ranks.size(), ws, so, s); }
        GMD_CUDA(cudaMemcpyAsync(vals.data(), so, sizeof(double) * vals.size(),
                                 cudaMemcpyDeviceToHost, s));
        sync(h);
    }
    auto at = [&](int64_t r) {
        size_t i = std::lower_bound(ranks.begin(), ranks.end(), r) - ranks.begin();
        return vals[i];
    };
    for (int k = 1; k < p; ++k) {
        int64_t c = n * k / p;
        bounds[k] = (c >= 1 && c < n) ? 0.5 * (at(c - 1) + at(c)) : (double)k / p;
    }
}

void ensure_bond_layout(gmd_handle* h);

// line edges (e', e) of every partition on the device (linegraph.cpp:124-171,
// count -> scan -> fill in (e', e) order); lcnt / lpairs
void build_line_edges_dev(gmd_handle* h) {
    ensure_bond_layout(h);
    if (h->line_dev_ready) return;
    cudaStream_t s = h->stream;
    const int64_t nb = h->nb;
    int32_t* cnt = h->lcnt.get<int32_t>(nb + 1);
    launch_line_count(nb, h->bedge.as<int32_t>(), h->src.as<int32_t>(), h->brow.as<int32_t>(), cnt,
                      s);
    scan_i32(h, cnt, cnt, nb);
    int32_t T = 0;
    GMD_CUDA(cudaMemcpyAsync(&T, cnt + nb, 4, cudaMemcpyDeviceToHost, s));
    sync(h);
    h->nline = T;
    int32_t* pairs = h->lpairs.get<int32_t>(2 * (size_t)T);
    launch_line_fill(nb, h->bedge.as<int32_t>(), h->src.as<int32_t>(), h->brow.as<int32_t>(),
                     h->brev.as<int32_t>(), cnt, pairs, s);
    h->line_dev_ready = true;
}

void build_impl(gmd_handle* h, int64_t n, const double* pos, const int32_t* Z, const double* lat,
                const uint8_t* pbc, double rc, double r3, double tau, int p, uint32_t flags) {
    cudaStream_t s = h->stream;
    h->built = false;
    h->graph_only = false;
    h->closure_ready = false;
    h->hc_ready = h->hcb_ready = false;
    h->line_dev_ready = false;
    h->ctab_ok = false;
    h->atoms.ready = h->bonds.ready = false;
    h->corrupted = false;
    if (!pos || !Z || !lat) raise(kArg, "null input pointer");
    if (p < 1) raise(kConfig, "partition count must be >= 1");
    if (rc <= 0.0) raise(kConfig, "cutoff must be positive");
    if (n <= 0) raise(kConfig, "cannot build neighbor list for empty system");
    if (n >= ((int64_t)1 << 31) - 1) raise(kConfig, "atom count exceeds the int32 index range");
    GMD_CUDA(cudaEventRecord(h->ev[0], s));
    h->n = n;
    h->p = p;
    h->rc = rc;
    h->r3 = r3;
    h->tau = tau;
    h->allow_narrow = (flags & GMD_ALLOW_NARROW) != 0;
    std::memcpy(h->lat, lat, sizeof h->lat);

    double* dpos = h->pos.get<double>(3 * n);
    int32_t* dZ = h->Z.get<int32_t>(n);
    cudaMemcpyKind kind =
        (flags & GMD_INPUT_DEVICE) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    GMD_CUDA(cudaMemcpyAsync(dpos, pos, sizeof(double) * 3 * n, kind, s));
    // species are read first by the forward's embedding: a host upload runs
    // on the side stream under the graph build (the forward waits on ev[6];
    // the side stream is drained before gmd_build returns, so the caller may
    // reuse its buffer afterwards)
    DrainSide drain{h->side};
    if (flags & GMD_INPUT_DEVICE) {
        GMD_CUDA(cudaMemcpyAsync(dZ, Z, sizeof(int32_t) * n, kind, s));
        h->z_pending = false;
    } else {
        // after the positions: the two host copies would otherwise share the
        // H2D link while the build waits for the positions
        GMD_CUDA(cudaEventRecord(h->ev[6], s));
        GMD_CUDA(cudaStreamWaitEvent(h->side, h->ev[6], 0));
        GMD_CUDA(cudaMemcpyAsync(dZ, Z, sizeof(int32_t) * n, kind, h->side));
        GMD_CUDA(cudaEventRecord(h->ev[6], h->side));
        h->z_pending = true;
    }
    ensure_periodic_dev(h, pbc, rc);
    if (std::abs(det3(h->lat)) < 1e-10)
        raise(kConfig, "periodic system requires an invertible lattice");

    // ---- scalar geometry (neighborlist.cpp:119-126)
    Geom& g = h->geom;
    std::memcpy(g.L, h->lat, sizeof g.L);
    inverse3(h->lat, g.inv);
    int64_t nbins = 1;
    for (int k = 0; k < 3; ++k) {
        double width = perp_width(h->lat, k);
        double fb = std::floor(width / rc);
        if (fb > 4.0e6) raise(kConfig, "cell is too large relative to the cutoff for binning");
        // neighborlist.cpp:121-126 bins floor(width / rc) and searches
        // floor(rc / bw) + 1 cells each way, i.e. 5 cells per axis when the
        // width is a multiple of rc.  Edge order does not depend on the bins
        // (rows are key-sorted), so take one bin fewer there: bw > rc by a
        // wide margin and the 3-cell stencil is exact.
        if (fb >= 2.0 && width / fb < rc * (1.0 + 1e-6)) fb -= 1.0;
        g.bins[k] = std::max(1, (int)fb);
        double bw = width / g.bins[k];
        g.sten[k] = (int)std::floor(rc / bw) + 1;
        nbins *= g.bins[k];
    }
    if (nbins > ((int64_t)1 << 30)) raise(kConfig, "too many neighbour-search bins");
    g.cutoff2 = rc * rc;
    g.pre2 = g.cutoff2 * 1.000001;
    g.bond_bound = -1.0;
    {  // partition axis: longest lattice vector, first max wins (partitioner.cpp:57-64)
        double best = -1.0;
        for (int k = 0; k < 3; ++k) {
            double len = vnorm(row3(h->lat, k));
            if (len > best) {
                best = len;
                h->axis = k;
            }
        }
        g.axis = h->axis;
    }
    if (p > kMaxParts) raise(kConfig, "partition count limited to 64");
    if ((int64_t)p > n) raise(kConfig, "more partitions than atoms");
    if (r3 > 0.0) {  // check_ranges (linegraph.cpp:10-14)
        if (r3 > rc) raise(kConfig, "three-body range cannot exceed the atom graph cutoff");
        if (tau < 0.0) raise(kConfig, "tolerance tau must be >= 0");
        g.bond_bound = r3 + tau;
    }

    // ---- cell list + neighbour search (neighborlist.cpp:108-197)
    NLBuffers b{};
    b.pos = dpos;
    b.cell = h->cell.get<int32_t>(3 * n);
    b.pos4 = h->pos4.get<double4>(n);
    b.cell4 = h->cell4.get<int4>(n);
    b.fw_axis = h->fw.get<double>(n);
    b.bin = h->bin.get<int32_t>(n);
    b.bin_cnt = h->bin_cnt.get<int32_t>(nbins);
    b.bin_start = h->bin_start.get<int32_t>(nbins + 1);
    b.s_id = h->s_id.get<int32_t>(n);
    b.s_w = h->s_w.get<double>(3 * n);
    b.s_p = h->s_p.get<double>(3 * n);
    b.s_c = h->s_c.get<int32_t>(3 * n);
    b.deg = h->deg.get<int32_t>(n);
    b.bcnt = h->bcnt.get<int32_t>(n);
    b.flags = h->flags.get<int32_t>(4);
    int32_t* fillp = h->fill.get<int32_t>(nbins);
    GMD_CUDA(cudaMemsetAsync(b.bin_cnt, 0, sizeof(int32_t) * nbins, s));
    GMD_CUDA(cudaMemsetAsync(fillp, 0, sizeof(int32_t) * nbins, s));
    GMD_CUDA(cudaMemsetAsync(b.flags, 0, 16, s));
    { PROF("nl_wrap"); launch_wrap(g, n, b, s); }
    { PROF("scan"); scan_i32(h, b.bin_cnt, b.bin_start, nbins); }
    { PROF("nl_bin_scatter"); launch_bin_scatter(g, n, b, fillp, s); }
    // ---- partition rule and owners (partitioner.cpp:46-108).  Owners only
    // depend on the wrapped fractional coordinate, so they are known before
    // the neighbour search -- one rank per GPU then builds only its rows.
    const bool rank_mode = h->comm && h->comm->world > 1;
    const int myrank = rank_mode ? h->comm->rank : -1;
    if (rank_mode && p != h->comm->world)
        raise(kConfig, "one-rank-per-GPU mode needs p == world size");
    h->bounds.assign(p + 1, 0.0);
    h->bounds[p] = 1.0;
    int32_t* ownp = h->atoms.owner.get<int32_t>(n);
    LayoutState& A = h->atoms;
    if (p == 1) {
        GMD_CUDA(cudaMemsetAsync(ownp, 0, sizeof(int32_t) * n, s));
    } else {
        if (flags & GMD_EQUAL_WIDTH) {
            for (int k = 1; k < p; ++k) h->bounds[k] = (double)k / p;
        } else {
            quantile_walls(h, b.fw_axis, n, p, h->bounds.data());
        }
        for (int k = 1; k <= p; ++k)
            if (h->bounds[k] <= h->bounds[k - 1])
                raise(kConfig,
                      "cannot place distinct partition boundaries; coordinates along the axis "
                      "are degenerate");
        if (!h->allow_narrow) {  // check_slab_widths (partitioner.cpp:21-33)
            double perp = perp_width(h->lat, h->axis);
            for (int i = 0; i < p; ++i) {
                double width = (h->bounds[i + 1] - h->bounds[i]) * perp;
                if (width < rc)
                    raise(kConfig, "partition-width error: slab " + std::to_string(i) + " is " +
                                       std::to_string(width) + " A wide, below the cutoff " +
                                       std::to_string(rc) + " A");
            }
        }
        Bounds bd{};
        bd.p = p;
        for (int k = 0; k <= p; ++k) bd.b[k] = h->bounds[k];
        { PROF("part_owner"); launch_owner(b.fw_axis, n, bd, ownp, s); }
    }
    if (rank_mode) GMD_CUDA(cudaMemsetAsync(b.deg, 0, sizeof(int32_t) * n, s));

    // fp32 prefilter threshold: keeps every pair the fp64 prefilter keeps.
    // Coordinates are taken relative to the destination bin origin, so each
    // component is bounded by B = max_k sum_r |L_rk| (s_r + 1) / bins_r; fp32
    // rounding moves each component of v by at most delta = 4 B 2^-24.
    float thr32, acc32, zero32, pos_gate;
    {
        double B = 0.0;
        for (int k = 0; k < 3; ++k) {
            double bk = 0.0;
            for (int r = 0; r < 3; ++r)
                bk += std::abs(g.L[3 * r + k]) * (double)(g.sten[r] + 1) / g.bins[r];
            B = std::max(B, bk);
        }
        B *= 1.01;
        const double u = std::ldexp(1.0, -24);
        const double delta = 4.0 * B * u;
        const double r = std::sqrt(g.pre2) * (1.0 + 1e-9) + std::sqrt(3.0) * delta;
        const double thr = r * r * (1.0 + 8.0 * u);
        thr32 = std::nextafter((float)thr, INFINITY);
        // fast-accept band: |v32|^2 <= acc32 puts the true vector within
        // rc (1 - 1e-9) (|v - v32| <= sqrt(3) delta, fp32 |.|^2 relative error
        // <= 4u), i.e. inside both fp64 tests with a margin far above fp64
        // rounding (wrapped vs raw vectors differ by ~1e-12 A); |v32|^2 >
        // zero32 keeps the true vector away from 0 (d2 != 0).
        const double ra = std::sqrt(g.cutoff2) * (1.0 - 1e-9) - std::sqrt(3.0) * delta;
        const double acc = ra > 0.0 ? ra * ra / (1.0 + 8.0 * u) : 0.0;
        acc32 = std::nextafter((float)acc, 0.0f);
        const double rz = 2.0 * std::sqrt(3.0) * delta + 1e-6;
        zero32 = std::nextafter((float)(rz * rz * (1.0 + 8.0 * u)), INFINITY);
        if (!(acc32 > zero32)) acc32 = -1.0f;  // no fast path: every survivor in fp64
        // The band's margin (rc * 1e-9) must dwarf the fp64 disagreement between
        // the wrapped vector (fractional -> floor -> lattice) and the reference's
        // raw one ((p_j - p_i) + off L).  Both are a few dozen roundings of
        // magnitudes <= kappa (M + S), M = max |input coordinate| (k_wrap, on
        // the device), S = sum |L|, kappa = conditioning of the fractional map:
        // fast accept is kept only while 64 u64 kappa (M + S) <= rc 1e-9 / 2.
        double S = 0.0, imax = 0.0;
        for (int k = 0; k < 9; ++k) {
            S += std::abs(g.L[k]);
            imax = std::max(imax, std::abs(g.inv[k]));
        }
        const double kappa = 3.0 * S * imax + 1.0;
        const double mgate = 0.5e-9 * std::sqrt(g.cutoff2) / (64.0 * std::ldexp(1.0, -53) * kappa) - S;
        pos_gate = mgate > 0.0 ? std::nextafter((float)mgate, 0.0f) : -1.0f;
        if (!(pos_gate > 0.0f)) acc32 = -1.0f;
    }
    int cap = h->nl_cap;
    if (cap <= 0) {  // first build: density estimate of the mean degree
        const double mean = (double)n * 4.18879020478639 * rc * rc * rc / std::abs(det3(h->lat));
        cap = ((int)(1.2 * mean + 16) + 7) & ~7;
    }
    int32_t* rowp = h->row.get<int32_t>(n + 1);
    int32_t hdr[2];
    int32_t ne32 = 0;
    // p = 1: the edge arrays are sized n x cap, so the emit follows the search
    // without a host round trip; the edge count and the slab-overflow check
    // ride on the build's final flag read (an overflowing row, rare with the
    // carried capacity, rebuilds at the larger capacity)
    const bool defer = p == 1 && !rank_mode && (int64_t)n * cap < INT32_MAX;
    for (int attempt = 0; attempt < 2; ++attempt) {
        auto* slab = h->slab.get<unsigned long long>((size_t)n * cap);
        { PROF("nl_search"); launch_nl_search(g, thr32, acc32, zero32, pos_gate, nbins, n, cap, b, slab, ownp, myrank, s); }
        { PROF("scan"); scan_i32(h, b.deg, rowp, n); }
        if (defer) break;
        GMD_CUDA(cudaMemcpyAsync(&ne32, rowp + n, 4, cudaMemcpyDeviceToHost, s));
        read_flags(h, hdr);
        if (hdr[0] <= cap) break;
        cap = (hdr[0] + 7) & ~7;  // rare: an atom exceeded the slab row
        GMD_CUDA(cudaMemsetAsync(b.flags, 0, 8, s));  // keeps k_wrap's flags[3]
    }
    if (!defer) {
        h->nl_cap = (hdr[0] + hdr[0] / 8 + 4 + 7) & ~7;  // next build: this one's max degree
        if (ne32 < 0) raise(kConfig, "edge count exceeds the int32 index range");
        h->ne = ne32;
    }
    const int64_t ecap = std::max<int64_t>(1, defer ? (int64_t)n * cap : (int64_t)ne32);
    GraphDev gd;
    gd.n = n;
    gd.ne = defer ? -1 : h->ne;  // (the emit and the bond kernels read row[], not ne)
    gd.row = rowp;
    gd.src = h->src.get<int32_t>(ecap);
    // packed image offsets: the three-body stage needs them; otherwise they
    // are only read by the graph export, which re-derives them from the slab
    // (4 B per edge not written per step)
    h->emit_cap = cap;
    h->img_ok = r3 > 0.0;
    gd.img = h->img_ok ? h->img.get<uint32_t>(ecap) : nullptr;
    gd.vd = h->vd.get<float4>(ecap);
    gd.d = h->ed.get<float>(ecap);
    gd.bond = r3 > 0.0 ? h->ebond.get<uint8_t>(ecap) : nullptr;  // three-body bonds only
    // p > 1 in one process: the requirement masks are OR-ed in by the emit
    unsigned long long* req_emit = nullptr;
    if (p > 1 && !rank_mode) {
        req_emit = A.req.get<unsigned long long>(n);
        GMD_CUDA(cudaMemsetAsync(req_emit, 0, sizeof(unsigned long long) * n, s));
    }
    { PROF("nl_emit"); launch_nl_emit(g, n, cap, h->slab.as<unsigned long long>(), b, gd, s, ownp, req_emit); }

    // ---- requirement masks, span layouts, local edge ends (partitioner.cpp:110-218)
    h->n_own = n;
    if (p == 1) {
        A.p = 1;
        A.nid = n;
        A.list_off = {0, (int32_t)n, (int32_t)n, (int32_t)n};
        A.rows = n;
        A.nfrom = 0;
        A.ready = true;
        A.api_ready = A.dups_ready = false;
        A.h_nodes.clear();
    } else {
        auto* reqp = A.req.get<unsigned long long>(n);
        if (rank_mode) {
            GMD_CUDA(cudaMemsetAsync(reqp, 0, sizeof(unsigned long long) * n, s));
            PROF("part_required");
            launch_required_rank(rowp, gd.src, n, ownp, myrank, reqp, s);
        }  // else: written by the emit
        build_layout(h, A, ownp, reqp, n, p, myrank);
        {
            PROF("part_edge_lsrc");
            launch_edge_lsrc(rowp, gd.src, n, ownp, A.crow.as<int32_t>(), A.node_array.as<int32_t>(),
                             A.list_off_d.as<int32_t>(), p, h->lsrc.get<int32_t>(ecap), b.flags, s);
        }
        if (rank_mode) build_rank_plan(h, ownp, myrank);
    }

    // ---- three-body bonds (linegraph.cpp:25-43) + reverse-bond index
    h->has_lg = r3 > 0.0;
    h->nb = 0;
    if (h->has_lg) {
        int32_t* br = h->brow.get<int32_t>(n + 1);
        { PROF("scan"); scan_i32(h, b.bcnt, br, n); }
        // deferred like the edge count: bond arrays sized by the edge
        // capacity, the bond count and max in-bonds read with the final flags
        const bool defer_b = defer && !(flags & GMD_LINE_PARTS);
        int64_t bcap = ecap;
        if (!defer_b) {
            int32_t nb32 = 0, fl[4];
            GMD_CUDA(cudaMemcpyAsync(&nb32, br + n, 4, cudaMemcpyDeviceToHost, s));
            GMD_CUDA(cudaMemcpyAsync(fl, b.flags, 16, cudaMemcpyDeviceToHost, s));
            sync(h);
            h->nb = nb32;
            h->max_bonds = fl[2];
            bcap = std::max<int64_t>(1, h->nb);
        }
        int32_t* be = h->bedge.get<int32_t>(bcap);
        int32_t* bv = h->brev.get<int32_t>(bcap);
        int32_t* ebid = h->ebid.get<int32_t>(ecap);
        { PROF("bond_edges"); launch_bond_edges(rowp, gd.bond, n, br, be, ebid, s); }
        { PROF("bond_rev"); launch_bond_rev(n, gd, br, be, ebid, bv, b.flags, ownp, myrank, s); }
        if (rank_mode) build_bond_rank_plan(h, ownp, myrank);
    }
    h->built = true;
    // create_distributed builds the line-graph partitions eagerly
    // (engine.cpp:57-62); the model never reads them (it works per center on
    // the global bonds), so they are built here only on request
    if ((flags & GMD_LINE_PARTS) && h->has_lg && !rank_mode) build_line_edges_dev(h);
    GMD_CUDA(cudaEventRecord(h->ev[1], s));
    if (defer) {
        int32_t fl[4] = {0, 0, 0, 0}, nb32 = 0;
        GMD_CUDA(cudaMemcpyAsync(&ne32, rowp + n, 4, cudaMemcpyDeviceToHost, s));
        GMD_CUDA(cudaMemcpyAsync(fl, b.flags, 16, cudaMemcpyDeviceToHost, s));
        if (h->has_lg) GMD_CUDA(cudaMemcpyAsync(&nb32, h->brow.as<int32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
        sync(h);
        hdr[0] = fl[0];
        hdr[1] = fl[1];
        if (h->has_lg && !(flags & GMD_LINE_PARTS)) {
            h->nb = nb32;
            h->max_bonds = fl[2];
        }
        if (hdr[0] > cap) {  // truncated slab rows: everything above is void
            h->built = false;
            h->nl_cap = (hdr[0] + hdr[0] / 8 + 4 + 7) & ~7;
            build_impl(h, n, pos, Z, lat, pbc, rc, r3, tau, p, flags);
            return;
        }
        h->nl_cap = (hdr[0] + hdr[0] / 8 + 4 + 7) & ~7;  // next build: this one's max degree
        if (ne32 < 0) raise(kConfig, "edge count exceeds the int32 index range");
        h->ne = ne32;
        check_flags(hdr[1]);
    } else {
        read_flags(h, hdr);
    }
    float ms = 0.f;
    GMD_CUDA(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    h->t_graph = ms * 1e-3;
}

void need_built(const gmd_handle* h) {
    if (!h->built) raise(kConfig, "no graph has been built on this handle");
}

// bond layouts + line graph partitions, lazily (export / bond feature API)
void ensure_bond_layout(gmd_handle* h) {
    need_built(h);
    if (!h->has_lg) raise(kConfig, "no line graph was built");
    if (h->comm && h->comm->world > 1)
        raise(kConfig, "bond partition views are not available in one-rank-per-GPU mode");
    LayoutState& B = h->bonds;
    if (B.ready) return;
    cudaStream_t s = h->stream;
    int32_t* bown = B.owner.get<int32_t>(h->nb);
    launch_bond_owner(h->n, h->brow.as<int32_t>(), h->atoms.owner.as<int32_t>(), bown, s);
    if (h->p == 1) {
        B.p = 1;
        B.nid = h->nb;
        B.list_off = {0, (int32_t)h->nb, (int32_t)h->nb, (int32_t)h->nb};
        B.rows = h->nb;
        B.nfrom = 0;
        B.ready = true;
        B.api_ready = B.dups_ready = false;
        B.h_nodes.clear();
        return;
    }
    auto* breq = B.req.get<unsigned long long>(h->nb);
    launch_bond_req(h->n, h->brow.as<int32_t>(), h->bedge.as<int32_t>(), h->src.as<int32_t>(),
                    h->atoms.owner.as<int32_t>(), breq, s);
    build_layout(h, B, bown, breq, h->nb, h->p);
}

void ensure_host_cache(gmd_handle* h) {
    need_built(h);
    if (h->hc_ready) return;
    d2h(h, h->h_owner, h->atoms.owner.as<int32_t>(), h->n);
    d2h(h, h->h_row, h->row.as<int32_t>(), h->n + 1);
    d2h(h, h->h_src, h->src.as<int32_t>(), h->ne);
    if (h->p > 1) {
        d2h(h, h->h_lsrc, h->lsrc.as<int32_t>(), h->ne);
        d2h(h, h->h_crow, h->atoms.crow.as<int32_t>(), h->n);
    }
    sync(h);
    h->hc_ready = true;
}

const std::vector<int32_t>& host_nodes(gmd_handle* h, LayoutState& ls) {
    if (ls.h_nodes.empty() && ls.rows > 0) {
        if (ls.p == 1) {
            ls.h_nodes.resize(ls.rows);
            for (int64_t i = 0; i < ls.rows; ++i) ls.h_nodes[i] = (int32_t)i;
        } else {
            d2h(h, ls.h_nodes, ls.node_array.as<int32_t>(), ls.rows);
            sync(h);
        }
    }
    return ls.h_nodes;
}

LayoutState& layout_of(gmd_handle* h, int bonds) {
    need_built(h);
    if (bonds) {
        ensure_bond_layout(h);
        return h->bonds;
    }
    return h->atoms;
}

void check_part(gmd_handle* h, int part) {
    if (part < 0 || part >= h->p) raise(kArg, "partition index out of range");
}

// duplicates of one partition in build_span_layout order (partitioner.cpp:159-166)
std::vector<std::pair<int64_t, int64_t>> dup_pairs(gmd_handle* h, LayoutState& ls, int part) {
    const auto& nodes = host_nodes(h, ls);
    const int stride = 1 + 2 * ls.p;
    const int64_t b0 = ls.list_off[(size_t)part * stride], b1 = ls.list_off[(size_t)(part + 1) * stride];
    std::unordered_map<int32_t, int64_t> first;
    first.reserve((size_t)(b1 - b0) * 2);
    std::vector<std::pair<int64_t, int64_t>> out;
    for (int64_t r = b0; r < b1; ++r) {
        auto it = first.emplace(nodes[r], r - b0);
        if (!it.second) out.emplace_back(it.first->second, r - b0);
    }
    return out;
}

void ensure_dup_groups(gmd_handle* h, LayoutState& ls) {
    if (ls.dups_ready) return;
    std::vector<int32_t> gc, gs, dd, dc, du;
    for (int i = 0; i < ls.p; ++i) {
        auto pairs = dup_pairs(h, ls, i);
        const int64_t base = ls.base(i);
        std::stable_sort(pairs.begin(), pairs.end(),
                         [](auto& a, auto& b) { return a.first < b.first; });
        for (size_t k = 0; k < pairs.size(); ++k) {
            if (k == 0 || pairs[k].first != pairs[k - 1].first) {  // new canonical group
                gs.push_back((int32_t)dd.size());
                gc.push_back((int32_t)(pairs[k].first + base));
            }
            dd.push_back((int32_t)(pairs[k].second + base));
            dc.push_back((int32_t)(pairs[k].first + base));
            du.push_back((int32_t)(pairs[k].second + base));
        }
    }
    gs.push_back((int32_t)dd.size());
    ls.ngroups = (int64_t)gc.size();
    ls.ndups = (int64_t)dd.size();
    cudaStream_t s = h->stream;
    auto up = [&](DBuf& bf, const std::vector<int32_t>& v) {
        int32_t* d = bf.get<int32_t>(v.size());
        if (!v.empty())
            GMD_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice, s));
    };
    up(ls.g_canon, gc);
    up(ls.g_start, gs);
    up(ls.g_dups, dd);
    up(ls.d_canon, dc);
    up(ls.d_dup, du);
    sync(h);
    ls.dups_ready = true;
}

void ensure_api_plan(gmd_handle* h, LayoutState& ls, bool corrupt) {
    if (ls.api_ready && ls.api_corrupt == corrupt) return;
    if (ls.nfrom > 0) {
        int32_t* out = ls.xapi.get<int32_t>(ls.nfrom);
        k_api_src<<<div_up(ls.nfrom, 256), 256, 0, h->stream>>>(
            ls.nfrom, ls.xdst.as<int32_t>(), ls.list_off_d.as<int32_t>(), ls.p, corrupt ? 1 : 0, out);
        GMD_LAUNCH_CHECK();
    }
    ls.api_ready = true;
    ls.api_corrupt = corrupt;
}

// feature-API buffers may be host memory (GMD_HOST_MEMORY): stage them
struct Staged {
    gmd_handle* h;
    void* user;
    void* dev;
    size_t bytes;
    bool host;
    Staged(gmd_handle* h_, void* buf, size_t b, bool host_, bool copy_in)
        : h(h_), user(buf), dev(buf), bytes(b), host(host_) {
        if (host) {
            dev = h->feat_tmp.get<char>(bytes);
            if (copy_in && bytes)
                GMD_CUDA(cudaMemcpyAsync(dev, user, bytes, cudaMemcpyHostToDevice, h->stream));
        }
    }
    void copy_out() {
        if (host && bytes)
            GMD_CUDA(cudaMemcpyAsync(user, dev, bytes, cudaMemcpyDeviceToHost, h->stream));
    }
};

int elem_size(int dtype) {
    dtype &= 0xff;
    if (dtype == GMD_F32) return 4;
    if (dtype == GMD_F64) return 8;
    raise(kArg, "dtype must be GMD_F32 or GMD_F64");
}

// chunk records for the tcgen05 backward edge pass (once per graph build)
void ensure_chunk_table(gmd_handle* h, const ConvArgs& a) {
    if (h->ctab_ok) return;
    cudaStream_t s = h->stream;
    const int grid = bwd_tc_grid(a.n);
    int32_t* cnt = h->ccnt.get<int32_t>(a.n + 1);
    int32_t* cst = h->cstart.get<int32_t>(a.n + 1);
    launch_chunk_count(a, cnt, s);
    scan_i32(h, cnt, cst, a.n + 1);
    int32_t T = 0;
    GMD_CUDA(cudaMemcpyAsync(&T, cst + a.n, 4, cudaMemcpyDeviceToHost, s));
    GMD_CUDA(cudaStreamSynchronize(s));
    int4* tab = h->ctab.get<int4>(std::max<int64_t>(1, T));
    launch_chunk_fill(a, cst, tab, grid, h->ccta.get<int32_t>(grid + 1), s);
    h->ctab_grid = grid;
    h->ctab_ok = true;
}

// ---------------------------------------------------------------------------
// forward_distributed (potential.cpp:563-985)
// ---------------------------------------------------------------------------
void forward_impl(gmd_handle* h, double* energy, void* per_atom, void* forces, double* stress,
                  double* timing, uint32_t flags) {
    need_built(h);
    if (h->graph_only)
        raise(kConfig, "this handle holds partitions of a caller-supplied graph (no model evaluation)");
    if (!h->params_set) raise(kConfig, "no parameters have been set on this handle");
    const bool tb = h->p_r3 > 0.0;
    if (tb && !h->has_lg)
        raise(kConfig,
              "three-body parameters require a line graph in the distributed handle");
    if (std::abs(h->rc - h->p_r_atom) > 1e-12)
        raise(kConfig, "distributed handle cutoff does not match the parameters");
    cudaStream_t s = h->stream;
    DrainSide drain{h->side};
    const int64_t n_all = h->n;
    const bool rank_mode = h->comm && h->comm->world > 1;
    const int64_t n = rank_mode ? h->n_own : n_all;  // nodes this handle updates
    const int L = h->L;
    LayoutState& A = h->atoms;
    const int64_t R = A.rows;
    const bool part = h->p > 1;
    const bool gen = h->generic;  // widths other than F = 16, K = 8 (gmd_generic.cu)
    const int F = gen ? h->F : kF;
    // F = 64, K = 8: the feature-major / tcgen05 kernels of gmd_wide.cu
    // (GMD_WIDE=0 selects the width-generic kernels instead)
    const char* wide_env = std::getenv("GMD_WIDE");
    const bool wide = gen && wide_model(h->gm) && !(wide_env && wide_env[0] == '0');
    // tuned widths, but a center with more in-bonds than the tuned three-body
    // kernels stage: the three-body stage runs on the width-generic kernels
    // (any in-bond count, linegraph.cpp:144-160)
    const bool tbg = tb && !gen && h->max_bonds > kMaxBondsPerAtom;
    const bool tgen = gen || tbg;  // generic three-body kernels

    {   // the __constant__ model copy is per device: upload only when another
        // parameter set was resident (saves a blocking pageable copy per step)
        static std::mutex mu;
        static uint64_t resident[64] = {};
        std::lock_guard<std::mutex> lock(mu);
        const int dv = h->device & 63;
        if (!gen && resident[dv] != h->mc_ver) {
            upload_model(h->mc, s);
            resident[dv] = h->mc_ver;
        }
    }

    GMD_CUDA(cudaEventRecord(h->ev[2], s));
    if ((int)h->H.size() < L + 1) h->H.resize(L + 1);
    std::vector<float*> H(L + 1);
    for (int l = 0; l <= L; ++l) H[l] = h->H[l].get<float>(R * F);
    float* TH = h->TH.get<float>((size_t)L * n * F);
    float* MB = h->MB.get<float>(R * F);
    float* HB = h->HB.get<float>(n * F);
    double4* GRAD = h->GRAD.get<double4>(n);  // fp64: exact per-node sums of antisymmetric edge terms
    const int grid = model_grid(n);
    // backward edge pass: FFMA kernel, or the tcgen05 kernel with GMD_BWD_TC=1
    const char* tc_env = std::getenv("GMD_BWD_TC");
    const bool use_tc = !gen && tc_env && tc_env[0] == '1';
    const int vgrid = wide ? wide_bwd_grid(n) : gen ? gen_grid(n) * 8 : use_tc ? bwd_tc_grid(n) : bwd_edge_grid(n);
    // host forces (e2e): the last layer's edge pass runs in node chunks; a
    // chunk's forces are final once it finishes (GRAD[v] gathers only v's
    // in-edges; the three-body terms came at l = L - 1), so they go to the
    // host on the side stream while the next chunk computes
    constexpr int kForceChunks = 4;
    auto pinned = [](const void* p) {  // a pageable copy would block the launching thread
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return at.type == cudaMemoryTypeHost;
    };
    const int nchunk = (!gen && !rank_mode && forces && !(flags & GMD_OUTPUT_DEVICE) && pinned(forces) &&
                        !(flags & GMD_OUTPUT_F32) && !use_tc && bwd_edge_ranges() &&
                        !(tb && L == 1) && bwd_edge_grid(n / 10) == vgrid)
                           ? kForceChunks
                           : 1;
    // one rank per GPU: interior atoms (h->nodes_x[0, n_int)) compute while
    // the halo rows are in flight, the border atoms after they landed; the
    // two launches have their own energy / virial partial slots
    const char* ov_env = std::getenv("GMD_OVERLAP");
    const bool overlap = rank_mode && !use_tc && h->n_int > 0 && h->n_int < n &&
                         !(ov_env && ov_env[0] == '0');
    const int halves = overlap ? 2 : 1;
    double* e_part = h->e_part.get<double>((size_t)grid * halves);
    double* v_part = h->v_part.get<double>((size_t)L * halves * vgrid * 6);
    if (overlap) {
        GMD_CUDA(cudaMemsetAsync(e_part, 0, sizeof(double) * grid * halves, s));
        GMD_CUDA(cudaMemsetAsync(v_part, 0, sizeof(double) * L * halves * vgrid * 6, s));
    }
    const int tgrid = wide ? wide_tb_grid(n) : tgen ? gen_grid(n) * 8 : tb_grid_size(n);
    double* v3_part = h->v3_part.get<double>((size_t)tgrid * 9);
    double* red = h->red.get<double>(16);
    double* pa = h->per_atom.get<double>(n_all);
    if (rank_mode) GMD_CUDA(cudaMemsetAsync(pa, 0, sizeof(double) * n_all, s));

    ConvArgs a{n,
               rank_mode ? h->nodes_x.as<int32_t>() : nullptr,
               part ? A.crow.as<int32_t>() : nullptr,
               h->row.as<int32_t>(),
               part ? h->lsrc.as<int32_t>() : h->src.as<int32_t>(),
               h->vd.as<float4>(),
               h->ed.as<float>()};
    if (use_tc) ensure_chunk_table(h, a);
    // per-layer non-finite feature check (potential.cpp:107-115, :772)
    auto* nonfin = h->nonfin.get<unsigned long long>(1);
    GMD_CUDA(cudaMemsetAsync(nonfin, 0xff, 8, s));
    a.nonfinite = nonfin;
    BondArgs ba{n,
                a.nodes,
                a.crow,
                h->brow.as<int32_t>(),
                h->bedge.as<int32_t>(),
                h->brev.as<int32_t>(),
                h->src.as<int32_t>(),
                h->vd.as<float4>()};
    float *TP = nullptr, *TH3 = nullptr, *TH4 = nullptr;
    const int64_t nbr = h->nb + (rank_mode ? h->nb_halo : 0);  // bond rows incl. received
    if (tb) {
        TP = h->TP.get<float>((size_t)nbr * F);
        TH3 = h->TH3.get<float>((size_t)nbr * F);
        TH4 = h->TH4.get<float>(n * F);
    }
    const int32_t* xd = A.xdst.as<int32_t>();
    const int32_t* xs = A.xsrc.as<int32_t>();
    // corrupt_transfer_plan_for_test: the forward atom transfers read the
    // wrong span, as the reference's transfer_impl does (engine.cpp:136-137)
    const int32_t* xs_fwd = xs;
    if (h->corrupted && !rank_mode && A.nfrom > 0) {
        ensure_api_plan(h, A, true);
        xs_fwd = A.xapi.as<int32_t>();
    }
    // halo exchange of a row buffer: FROM rows <- owners' canonical rows
    // (engine.cpp:122-143); one rank per GPU packs its TO rows and goes
    // through the transport
    const int64_t nsend = rank_mode ? std::accumulate(h->scnt.begin(), h->scnt.end(), (int64_t)0) : 0;
    float* sendbuf = rank_mode ? h->sendbuf.get<float>(std::max<int64_t>(1, nsend) * F) : nullptr;
    auto exchange = [&](float* buf, bool fwd = false) {
        if (rank_mode && h->comm->fused_gather()) {
            PROF("halo_exchange");  // gather + P2P store + flags in the transport's kernels
            h->comm->exchange_gather(s, buf, h->xsend.as<int32_t>(), h->soff.data(), h->scnt.data(), buf,
                                     h->roff.data(), h->rcnt.data(), F);
        } else if (rank_mode) {
            {
                PROF("halo_pack");
                if (nsend > 0) {
                    k_gather_rows<<<div_up(nsend * F, 256), 256, 0, s>>>(
                        nsend, h->xsend.as<int32_t>(), reinterpret_cast<const uint32_t*>(buf),
                        reinterpret_cast<uint32_t*>(sendbuf), F);
                    GMD_LAUNCH_CHECK();
                }
            }
            PROF("halo_exchange");
            h->comm->exchange(s, sendbuf, h->soff.data(), h->scnt.data(), buf, h->roff.data(),
                              h->rcnt.data(), F);
        } else if (A.nfrom > 0) {
            PROF("exchange");
            if (gen) {  // any row width: 32-bit words
                k_copy_rows<<<div_up(A.nfrom * F, 256), 256, 0, s>>>(
                    A.nfrom, xd, fwd ? xs_fwd : xs, reinterpret_cast<uint32_t*>(buf), F);
                GMD_LAUNCH_CHECK();
            } else {
                launch_exchange(A.nfrom, xd, fwd ? xs_fwd : xs, buf, kF, s);
            }
        }
    };

    // split exchange (overlap): sends now, receives at exchange_end
    auto exchange_begin = [&](float* buf) {
        if (h->comm->fused_gather()) {
            PROF("halo_send");
            h->comm->exchange_gather_begin(s, buf, h->xsend.as<int32_t>(), h->soff.data(), h->scnt.data(),
                                           buf, h->roff.data(), h->rcnt.data(), F);
        } else {
            exchange(buf);
        }
    };
    auto exchange_end = [&]() {
        if (h->comm->fused_gather()) {
            PROF("halo_recv");
            h->comm->exchange_gather_end(s);
        }
    };

    // bond halo rows (three-body, one rank per GPU): t' and v_bar of the
    // reverse bonds computed at centers owned by peers
    const int64_t nbsend =
        rank_mode && tb ? std::accumulate(h->b_scnt.begin(), h->b_scnt.end(), (int64_t)0) : 0;
    float* bsend = rank_mode && tb ? h->bsendbuf.get<float>(std::max<int64_t>(1, nbsend) * F)
                                   : nullptr;
    auto bond_exchange = [&](float* buf, int width) {
        if (!(rank_mode && tb)) return;
        if (h->comm->fused_gather()) {
            PROF("halo_exchange");
            h->comm->exchange_gather(s, buf, h->bxsend.as<int32_t>(), h->b_soff.data(), h->b_scnt.data(),
                                     buf, h->b_roff.data(), h->b_rcnt.data(), width);
            return;
        }
        {
            PROF("halo_pack");
            if (nbsend > 0) {
                k_gather_rows<<<div_up(nbsend * width, 256), 256, 0, s>>>(
                    nbsend, h->bxsend.as<int32_t>(), reinterpret_cast<const uint32_t*>(buf),
                    reinterpret_cast<uint32_t*>(bsend), width);
                GMD_LAUNCH_CHECK();
            }
        }
        PROF("halo_exchange");
        h->comm->exchange(s, bsend, h->b_soff.data(), h->b_scnt.data(), buf, h->b_roff.data(),
                          h->b_rcnt.data(), width);
    };

    // ---- feature calculation: embeddings for every layout row (:597-602)
    if (h->z_pending) {
        GMD_CUDA(cudaStreamWaitEvent(s, h->ev[6], 0));
        h->z_pending = false;
    }
    {
        PROF("embed");
        if (gen)
            launch_gen_embed(h->gm, R, part ? A.node_array.as<int32_t>() : nullptr, h->Z.as<int32_t>(), H[0], s,
                             wide ? h->zs.get<uint8_t>(std::max<int64_t>(1, R)) : nullptr,
                             wide ? h->zmask.get<unsigned>(4) : nullptr);
        else
            launch_embed(R, part ? A.node_array.as<int32_t>() : nullptr, h->Z.as<int32_t>(), H[0], s,
                         h->zs.get<uint8_t>(std::max<int64_t>(1, R)), h->zmask.get<unsigned>(4));
    }
    GMD_CUDA(cudaEventRecord(h->ev[3], s));

    // ---- forward (:657-793)
    for (int l = 0; l < L; ++l) {
        const bool tbl = tb && l == L - 1;
        if (tbl) {
            if (wide) {
                float* TT = h->TT.get<float>((size_t)std::max<int64_t>(1, nbr) * F);
                { PROF("tb_t"); launch_wide_tb_t(h->gm, ba, TT, s); }
                { PROF("tb_forward"); launch_wide_tb_forward(h->gm, ba, TT, TP, TH3, s); }
            } else if (tgen) {
                float* TT = h->TT.get<float>((size_t)std::max<int64_t>(1, nbr) * F);
                { PROF("tb_t"); launch_gen_tb_t(h->gm, ba, nbr, TT, s); }
                { PROF("tb_forward"); launch_gen_tb_forward(h->gm, ba, TT, TP, TH3, h->flags.as<int32_t>(), s); }
            } else {
                PROF("tb_forward");
                launch_tb_forward(ba, TP, TH3, h->flags.as<int32_t>(), h->max_bonds, s);
            }
            bond_exchange(TP, F);
            {
                PROF("tb_inject");
                if (wide)
                    launch_wide_tb_inject(h->gm, ba, TP, H[l], TH4, s);
                else if (tgen)
                    launch_gen_tb_inject(h->gm, ba, TP, H[l], TH4, s);
                else
                    launch_tb_inject(ba, TP, H[l], TH4, s);
            }
        }
        // nodes [k0, k1) of the evaluation order; energy partials in half `hf`
        auto conv = [&](int64_t k0, int64_t k1, int hf) {
            if (k1 <= k0) return;
            PROF("conv");
            ConvArgs ar = a;
            ar.n = k1 - k0;
            if (ar.nodes) ar.nodes += k0;
            float* th = TH + ((size_t)l * n + k0) * F;
            double* pl = l == L - 1 ? pa : nullptr;
            if (wide)
                launch_wide_conv(h->gm, ar, l, H[l], H[l + 1], th, pl, s,
                                 l == 0 && !tbl ? h->zs.as<uint8_t>() : nullptr,
                                 l == 0 && !tbl ? h->zmask.as<unsigned>() : nullptr);
            else if (gen)
                launch_gen_conv(h->gm, ar, l, H[l], H[l + 1], th, pl, s);
            else
                launch_conv(ar, l, H[l], H[l + 1], th, pl, l == L - 1 ? e_part + (size_t)hf * grid : nullptr,
                            s, l == 0 && !tbl ? h->zs.as<uint8_t>() : nullptr,
                            l == 0 && !tbl ? h->zmask.as<unsigned>() : nullptr);
        };
        const bool halo = l > 0 || tbl;
        if (halo && overlap) {
            exchange_begin(H[l]);
            conv(0, h->n_int, 0);
            exchange_end();
            conv(h->n_int, n, 1);
        } else {
            if (halo) exchange(H[l], true);
            conv(0, n, 0);
        }
    }
    GMD_CUDA(cudaEventRecord(h->ev[4], s));
    // per-atom energies are final after the forward: copy them to the host
    // while the backward runs (e2e use with host buffers)
    const bool pa_early = per_atom && !(flags & GMD_OUTPUT_DEVICE) && !(flags & GMD_OUTPUT_F32);
    if (pa_early) {
        GMD_CUDA(cudaStreamWaitEvent(h->side, h->ev[4], 0));
        GMD_CUDA(cudaMemcpyAsync(per_atom, pa, 8 * n_all, cudaMemcpyDeviceToHost, h->side));
    }

    // ---- backward (:796-984)
    if (gen && !wide) launch_gen_init_hbar(h->gm, n, HB, s);  // (tuned, wide: fused into the first bwd_node)
    GMD_CUDA(cudaMemsetAsync(GRAD, 0, sizeof(double4) * n, s));
    for (int l = L - 1; l >= 0; --l) {
        // layer 0's h_bar is the embedding gradient (no position dependence,
        // never read) unless the three-body backward follows it (L = 1)
        const bool need_hbar = l > 0 || (tb && l == L - 1);
        // layer 0 reads h0 = emb[Z] (no three-body injection before it)
        const bool h0_emb = l == 0 && !(tb && L == 1) && !gen && !wide;
        const uint8_t* zs_l = h0_emb ? h->zs.as<uint8_t>() : nullptr;
        const unsigned* zm_l = h0_emb ? h->zmask.as<unsigned>() : nullptr;

        {
            PROF("bwd_node");
            if (wide)
                launch_wide_bwd_node(h->gm, n, a.nodes, a.crow, l, HB, TH + (size_t)l * n * F, MB,
                                     l == L - 1, s);
            else if (gen)
                launch_gen_bwd_node(h->gm, n, a.nodes, a.crow, l, HB, TH + (size_t)l * n * F, MB, s);
            else
                launch_bwd_node(n, a.nodes, a.crow, l, HB, TH + (size_t)l * n * kF, MB, l == L - 1, s);
        }
        if (overlap) {
            auto edge = [&](int64_t k0, int64_t k1, int hf) {
                if (k1 <= k0) return;
                PROF("bwd_edge");
                ConvArgs ar = a;
                ar.n = k1 - k0;
                ar.nodes += k0;
                double* vp = v_part + ((size_t)l * 2 + hf) * vgrid * 6;
                if (wide)
                    launch_wide_bwd_edge(h->gm, ar, MB, H[l], HB + k0 * F, GRAD + k0, vp, s, need_hbar);
                else if (gen)
                    launch_gen_bwd_edge(h->gm, ar, MB, H[l], HB + k0 * F, GRAD + k0, vp, s);
                else
                    launch_bwd_edge(ar, MB, H[l], HB + k0 * F, GRAD + k0, vp, s, nullptr, 0, need_hbar, zs_l, zm_l);
            };
            exchange_begin(MB);
            edge(0, h->n_int, 0);
            exchange_end();
            edge(h->n_int, n, 1);
        } else {
            exchange(MB);
            PROF("bwd_edge");
            if (wide)
                launch_wide_bwd_edge(h->gm, a, MB, H[l], HB, GRAD, v_part + (size_t)l * vgrid * 6, s, need_hbar);
            else if (gen)
                launch_gen_bwd_edge(h->gm, a, MB, H[l], HB, GRAD, v_part + (size_t)l * vgrid * 6, s);
            else if (use_tc)
                launch_bwd_edge_tc(a, h->ctab.as<int4>(), h->ccta.as<int32_t>(), vgrid, MB, H[l], HB,
                                   GRAD, v_part + (size_t)l * vgrid * 6, s);
            else if (l > 0 || nchunk == 1)
                launch_bwd_edge(a, MB, H[l], HB, GRAD, v_part + (size_t)l * vgrid * 6, s, nullptr, 0, need_hbar, zs_l,
                                zm_l);
            else {  // l = 0 in node chunks, forces streamed out per chunk
                double* fd = h->forces.get<double>(3 * n_all);
                // chunk starts on multiples of the grid's node stride and one
                // carried per-group virial: bitwise the unchunked launch
                const int64_t stride = bwd_edge_stride(vgrid);
                double* vg = h->v_grp.get<double>((size_t)stride * 6);
                // shrinking chunks (40/30/20/10 %): each chunk's force copy
                // hides under the next chunk's edge pass, and the last one,
                // exposed after the pass, is the smallest
                static const int cum[kForceChunks + 1] = {0, 4, 7, 9, 10};
                for (int c = 0; c < nchunk; ++c) {
                    ConvArgs ac = a;
                    ac.k0 = (n * cum[c] / 10) / stride * stride;
                    ac.n = c + 1 == nchunk ? n : (n * cum[c + 1] / 10) / stride * stride;
                    if (ac.n <= ac.k0) continue;
                    launch_bwd_edge(ac, MB, H[l], HB, GRAD, v_part, s, vg, vgrid, need_hbar, zs_l, zm_l);
                    launch_forces_out(ac.n - ac.k0, nullptr, GRAD + ac.k0, fd + 3 * ac.k0, nullptr, s);
                    GMD_CUDA(cudaEventRecord(h->ev[7], s));
                    GMD_CUDA(cudaStreamWaitEvent(h->side, h->ev[7], 0));
                    GMD_CUDA(cudaMemcpyAsync(static_cast<double*>(forces) + 3 * ac.k0, fd + 3 * ac.k0,
                                             24 * (ac.n - ac.k0), cudaMemcpyDeviceToHost, h->side));
                }
            }
        }
        if (tb && l == L - 1) {
            float* QB = h->QB.get<float>(R * F);
            float4* VIN = h->VIN.get<float4>(nbr);
            float4* VOUT = h->VOUT.get<float4>(nbr);
            {
                PROF("tb_bwd_q");
                if (wide)
                    launch_wide_tb_bwd_q(h->gm, n, a.nodes, a.crow, HB, TH4, QB, s);
                else if (tgen)
                    launch_gen_tb_bwd_q(h->gm, n, a.nodes, a.crow, HB, TH4, QB, s);
                else
                    launch_tb_bwd_q(n, a.nodes, a.crow, HB, TH4, QB, s);
            }
            if (rank_mode) exchange(QB);  // q_bar of halo atoms (bond sources)
            {
                PROF("tb_backward");
                if (wide)
                    launch_wide_tb_backward(h->gm, ba, QB, TH3, h->TT.as<float>(),
                                            h->SMR.get<float>((size_t)std::max<int64_t>(1, nbr) * F),
                                            VIN, VOUT, v3_part, s);
                else if (tgen)
                    launch_gen_tb_backward(h->gm, ba, QB, TH3, h->TT.as<float>(),
                                           h->SMR.get<float>((size_t)std::max<int64_t>(1, nbr) * F),
                                           VIN, VOUT, v3_part, s);
                else
                    launch_tb_backward(ba, QB, TH3, VIN, VOUT, v3_part, h->max_bonds, s);
            }
            bond_exchange(reinterpret_cast<float*>(VIN), 4);
            bond_exchange(reinterpret_cast<float*>(VOUT), 4);
            { PROF("tb_grad"); launch_tb_grad(ba, VIN, VOUT, GRAD, s); }
        }
    }
    const bool out_dev = flags & GMD_OUTPUT_DEVICE;
    const bool out_f32 = flags & GMD_OUTPUT_F32;
    double* fd = nullptr;
    float* ff = nullptr;
    if (forces) {
        if (out_f32)
            ff = out_dev ? static_cast<float*>(forces) : h->forces.get<float>(3 * n_all);
        else
            fd = out_dev ? static_cast<double*>(forces) : h->forces.get<double>(3 * n_all);
        if (rank_mode) {  // only this rank's atoms are written
            if (ff) GMD_CUDA(cudaMemsetAsync(ff, 0, 12 * n_all, s));
            if (fd) GMD_CUDA(cudaMemsetAsync(fd, 0, 24 * n_all, s));
        }
        if (nchunk == 1) {  // else written per chunk above
            PROF("forces_out");
            launch_forces_out(n, a.nodes, GRAD, fd, ff, s);
        }
    }
    {
        PROF("reduce");
        // generic kernels: the energy is the fixed-order sum of the per-atom energies
        const double* ps[3] = {gen ? pa : e_part, v_part, v3_part};
        const int np[3] = {gen ? (int)n_all : grid * halves, L * halves * vgrid, tgrid},
                  w[3] = {1, 6, 9};
        if (!tb) GMD_CUDA(cudaMemsetAsync(red + 7, 0, 9 * sizeof(double), s));
        launch_reduce_sets(tb ? 3 : 2, ps, np, w, red, s);
    }
    GMD_CUDA(cudaEventRecord(h->ev[5], s));

    double hred[16];
    GMD_CUDA(cudaMemcpyAsync(hred, red, sizeof hred, cudaMemcpyDeviceToHost, s));
    if (per_atom) {
        if (out_f32) {
            float* dst = out_dev ? static_cast<float*>(per_atom) : h->conv_tmp.get<float>(n_all);
            k_to_f32<<<div_up(n_all, 256), 256, 0, s>>>(n_all, pa, dst);
            GMD_LAUNCH_CHECK();
            if (!out_dev)
                GMD_CUDA(cudaMemcpyAsync(per_atom, dst, 4 * n_all, cudaMemcpyDeviceToHost, s));
        } else if (out_dev) {
            GMD_CUDA(cudaMemcpyAsync(per_atom, pa, 8 * n_all, cudaMemcpyDeviceToDevice, s));
        } else {
            GMD_CUDA(cudaStreamSynchronize(h->side));  // pa_early copy
        }
    }
    if (forces && !out_dev && nchunk == 1) {
        if (out_f32)
            GMD_CUDA(cudaMemcpyAsync(forces, ff, 12 * n_all, cudaMemcpyDeviceToHost, s));
        else
            GMD_CUDA(cudaMemcpyAsync(forces, fd, 24 * n_all, cudaMemcpyDeviceToHost, s));
    }
    unsigned long long nfkey = ~0ull;
    GMD_CUDA(cudaMemcpyAsync(&nfkey, nonfin, 8, cudaMemcpyDeviceToHost, s));
    int32_t hdr[2];
    read_flags(h, hdr);  // synchronizes the stream
    if (nchunk > 1) GMD_CUDA(cudaStreamSynchronize(h->side));  // streamed force chunks
    // first non-finite feature: (layer, partition, layout row) -> global atom id
    int64_t nf_layer = -1, nf_part = -1, nf_atom = -1;
    if (nfkey != ~0ull) {
        nf_layer = (int64_t)(nfkey >> 40);
        const int64_t row = (int64_t)(nfkey & ((1ull << 40) - 1));
        nf_atom = row;
        if (part) {
            int32_t gid = 0;
            GMD_CUDA(cudaMemcpy(&gid, A.node_array.as<int32_t>() + row, 4, cudaMemcpyDeviceToHost));
            nf_atom = gid;
        }
        if (rank_mode) {
            nf_part = h->comm->rank;
        } else if (part) {
            int32_t ow = 0;
            GMD_CUDA(cudaMemcpy(&ow, h->atoms.owner.as<int32_t>() + nf_atom, 4, cudaMemcpyDeviceToHost));
            nf_part = ow;
        } else {
            nf_part = 0;
        }
    }
    if (rank_mode) {  // energy + virial: rank-ordered sum of the per-rank sums
        constexpr int kW = 19;  // 16 sums + first non-finite (layer, partition, atom)
        double mine[kW];
        std::copy(hred, hred + 16, mine);
        mine[16] = (double)nf_layer;
        mine[17] = (double)nf_part;
        mine[18] = (double)nf_atom;
        std::vector<double> all((size_t)h->comm->world * kW);
        h->comm->allgather_f64(s, mine, kW, all.data());
        for (int c = 0; c < 16; ++c) {
            double acc = 0.0;
            for (int j = 0; j < h->comm->world; ++j) acc += all[(size_t)j * kW + c];
            hred[c] = acc;
        }
        nf_layer = -1;  // every rank reports the same offender: lowest layer, then rank
        for (int j = 0; j < h->comm->world; ++j) {
            const double* o = all.data() + (size_t)j * kW;
            if (o[16] >= 0 && (nf_layer < 0 || o[16] < nf_layer)) {
                nf_layer = (int64_t)o[16];
                nf_part = (int64_t)o[17];
                nf_atom = (int64_t)o[18];
            }
        }
    }
    if (nf_layer >= 0)  // parallel_for_partitions' wrapper (engine.cpp:278-283)
        raise(kRuntime, "worker for partition " + std::to_string(nf_part) +
                            " failed: non-finite feature at layer " + std::to_string(nf_layer) +
                            ", atom " + std::to_string(nf_atom));
    if (!std::isfinite(hred[0])) raise(kRuntime, "non-finite energy (non-finite features)");
    if (energy) *energy = hred[0];
    if (stress) {  // stress = sym(virial) / V (potential.cpp:978-982)
        const double* v6 = hred + 1;
        const double* v9 = hred + 7;
        double V[9] = {v6[0], v6[3], v6[4], v6[3], v6[1], v6[5], v6[4], v6[5], v6[2]};
        for (int k = 0; k < 9; ++k) V[k] += v9[k];
        double vol = std::abs(det3(h->lat));
        for (int a2 = 0; a2 < 3; ++a2)
            for (int b2 = 0; b2 < 3; ++b2)
                stress[3 * a2 + b2] = 0.5 * (V[3 * a2 + b2] + V[3 * b2 + a2]) / vol;
    }
    if (timing) {
        float f1 = 0, f2 = 0, f3 = 0;
        GMD_CUDA(cudaEventElapsedTime(&f1, h->ev[2], h->ev[3]));
        GMD_CUDA(cudaEventElapsedTime(&f2, h->ev[3], h->ev[4]));
        GMD_CUDA(cudaEventElapsedTime(&f3, h->ev[4], h->ev[5]));
        timing[0] = h->t_graph;
        timing[1] = f1 * 1e-3;
        timing[2] = f2 * 1e-3;
        timing[3] = f3 * 1e-3;
    }
}

}  // namespace

// ===========================================================================
// extern "C"
// ===========================================================================

namespace {
int run(gmd_handle* h, const std::function<void()>& fn) {
    if (!h) return GMD_ERR_ARG;
    try {
        GMD_CUDA(cudaSetDevice(h->device));
        fn();
        h->err.clear();
        return GMD_OK;
    } catch (const Status& e) {
        h->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        h->err = e.what();
        return GMD_ERR_RUNTIME;
    }
}
thread_local std::string g_err;
}  // namespace

extern "C" {

const char* gmd_version(void) { return "graphmd_b200 0.1 (sm_100a)"; }

const char* gmd_last_error(const gmd_handle* h) { return h ? h->err.c_str() : g_err.c_str(); }

int gmd_create(int device, gmd_handle** out) {
    if (!out) return GMD_ERR_ARG;
    *out = nullptr;
    auto* h = new gmd_handle();
    h->device = device;
    try {
        int ndev = 0;
        GMD_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) raise(kArg, "device ordinal out of range");
        GMD_CUDA(cudaSetDevice(device));
        GMD_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        GMD_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
        for (auto& e : h->ev) GMD_CUDA(cudaEventCreate(&e));
    } catch (const Status& e) {
        g_err = e.what();
        delete h;
        return e.code;
    }
    *out = h;
    return GMD_OK;
}

void gmd_destroy(gmd_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    DBuf* bufs[] = {&h->pos, &h->pos4, &h->cell4, &h->zs, &h->zmask, &h->fr_pos, &h->fr_cell, &h->fr_fw, &h->fr_bin,
                    &h->fr_cnt, &h->fr_flags, &h->Z, &h->cell, &h->fw, &h->bin, &h->bin_cnt, &h->bin_start,
                    &h->fill, &h->s_id, &h->s_w, &h->s_p, &h->s_c, &h->deg, &h->bcnt, &h->flags,
                    &h->row, &h->src, &h->img, &h->vd, &h->ed, &h->ebond, &h->edst, &h->lsrc, &h->counts,
                    &h->scan_tmp, &h->sel_ws, &h->sel_out, &h->small, &h->brow, &h->bedge, &h->ebid,
                    &h->brev, &h->lcnt, &h->lpairs, &h->slab, &h->feat_tmp, &h->flagtmp, &h->nodes, &h->nodes_x, &h->xsend, &h->sendbuf, &h->TH, &h->MB, &h->HB, &h->GRAD, &h->TP,
                    &h->TH3, &h->TH4, &h->QB, &h->VIN, &h->VOUT, &h->e_part, &h->v_part,
                    &h->v3_part, &h->red, &h->per_atom, &h->forces, &h->conv_tmp, &h->exp_tmp,
                    &h->md_part, &h->md_out, &h->md_bad, &h->md_pos, &h->md_vel, &h->md_frc,
                    &h->md_mass, &h->md_z, &h->gpar, &h->TT, &h->SMR};
    for (DBuf* b : bufs) b->release();
    for (LayoutState* ls : {&h->atoms, &h->bonds}) {
        DBuf* lb[] = {&ls->node_array, &ls->crow, &ls->list_off_d, &ls->xdst, &ls->xsrc,
                      &ls->xapi, &ls->owner, &ls->req, &ls->g_canon, &ls->g_start, &ls->g_dups,
                      &ls->d_canon, &ls->d_dup};
        for (DBuf* b : lb) b->release();
    }
    for (auto& b : h->H) b.release();
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : h->pev) cudaEventDestroy(e);
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->side) cudaStreamDestroy(h->side);
    h->comm.reset();
    if (h->ipc_window) cudaFree(h->ipc_window);
    delete h;
}

int gmd_build(gmd_handle* h, int64_t n, const double* pos, const int32_t* Z,
              const double lattice[9], const uint8_t pbc[3], double rc, double r3, double tau,
              int p, int n_threads, uint32_t flags) {
    (void)n_threads;
    return run(h, [&] { build_impl(h, n, pos, Z, lattice, pbc, rc, r3, tau, p, flags); });
}

int64_t gmd_params_size(int F, int K, int L) {
    return 119LL * F + (int64_t)L * F * F + (int64_t)L * F + 2LL * F * K + 2LL * F * F + F;
}

int gmd_params_init(uint64_t seed, int F, int K, int L, double r_atom, double r3, double* blob) {
    (void)r_atom;
    (void)r3;
    if (!blob || F < 1 || K < 1 || L < 1) return GMD_ERR_ARG;
    HostRng rng(seed ^ 0x9e3779b97f4a7c15ull);  // potential.cpp:132-145
    const struct {
        int64_t n;
        double scale;
    } seg[8] = {{119LL * F, 0.5},
                {(int64_t)L * F * F, 1.0 / std::sqrt((double)F)},
                {(int64_t)L * F, 0.1},
                {(int64_t)F * K, 1.0 / std::sqrt((double)K)},
                {(int64_t)F * K, 0.5 / std::sqrt((double)K)},
                {(int64_t)F * F, 1.0 / std::sqrt((double)F)},
                {(int64_t)F * F, 0.5 / std::sqrt((double)F)},
                {(int64_t)F, 0.5}};
    double* q = blob;
    for (const auto& sg : seg)
        for (int64_t i = 0; i < sg.n; ++i) *q++ = sg.scale * rng.normal();
    return GMD_OK;
}

namespace {
void build_gen_tables(gmd_handle* h, int F, int K, int L, double r_atom, double r3, const double* blob) {
    const size_t nemb = 119 * (size_t)F, nW = (size_t)L * F * F, nb = (size_t)L * F,
                 nP = (size_t)F * K, nFF = (size_t)F * F;
    std::vector<float> t(nemb + nW + nb + 3 * nP + 2 * nFF + F + nW + 2 * nFF + nP);
    const double* q = blob;
    size_t o = 0;
    for (size_t i = 0; i < nemb + nW + nb + nP; ++i) t[o++] = (float)*q++;  // emb, W, b, P
    const double* Pd = blob + nemb + nW + nb;
    for (size_t i = 0; i < nP; ++i) t[o++] = (float)(Pd[i] * (double)(i % K));  // k P
    for (size_t i = 0; i < nP + 2 * nFF + F; ++i) t[o++] = (float)*q++;  // P3 W3 W4 ro
    // transposed W (per layer), W3, W4
    const float* Wf = t.data() + nemb;
    const float* W3f = t.data() + nemb + nW + nb + 2 * nP + nP;
    const float* W4f = W3f + nFF;
    for (int l = 0; l < L; ++l)
        for (int f = 0; f < F; ++f)
            for (int gg = 0; gg < F; ++gg)
                t[o + (size_t)l * nFF + (size_t)gg * F + f] = Wf[(size_t)l * nFF + (size_t)f * F + gg];
    o += nW;
    for (int f = 0; f < F; ++f)
        for (int gg = 0; gg < F; ++gg) {
            t[o + (size_t)gg * F + f] = W3f[(size_t)f * F + gg];
            t[o + nFF + (size_t)gg * F + f] = W4f[(size_t)f * F + gg];
        }
    o += 2 * nFF;
    const float* P3f = t.data() + nemb + nW + nb + 2 * nP;
    for (int f = 0; f < F; ++f)
        for (int kk = 0; kk < K; ++kk) t[o + (size_t)kk * F + f] = P3f[(size_t)f * K + kk];
    o += nP;
    float* d = h->gpar.get<float>(t.size());
    GMD_CUDA(cudaMemcpy(d, t.data(), sizeof(float) * t.size(), cudaMemcpyHostToDevice));
    GenModel& g = h->gm;
    g.F = F;
    g.K = K;
    g.L = L;
    g.emb = d;
    g.W = d + nemb;
    g.b = g.W + nW;
    g.P = g.b + nb;
    g.Pk = g.P + nP;
    g.P3 = g.Pk + nP;
    g.W3 = g.P3 + nP;
    g.W4 = g.W3 + nFF;
    g.ro = g.W4 + nFF;
    g.WT = g.ro + F;
    g.W3T = g.WT + nW;
    g.W4T = g.W3T + nFF;
    g.P3T = g.W4T + nFF;
    const double r3e = r3 > 0.0 ? r3 : 1.0;
    g.r3 = (float)r3e;
    g.inv_r3 = (float)(1.0 / r3e);
    g.inv_sigma3 = (float)(K / r3e);
    g.mu_step3 = K > 1 ? (float)(r3e / (K - 1)) : 0.f;
    g.rc = (float)r_atom;
    g.inv_rc = (float)(1.0 / r_atom);
    g.inv_sigma = (float)(K / r_atom);  // sigma = rc / K (potential.cpp:34)
    g.mu_step = K > 1 ? (float)(r_atom / (K - 1)) : 0.f;
}

}  // namespace

int gmd_set_params(gmd_handle* h, int F, int K, int L, double r_atom, double r3,
                   const double* blob) {
    return run(h, [&] {
        if (!blob) raise(kArg, "null parameter blob");
        if (L < 1) raise(kConfig, "layer count must be >= 1");
        if (F < 1 || K < 1) raise(kConfig, "feature and basis widths must be >= 1");
        if (r_atom <= 0.0) raise(kConfig, "atom cutoff must be positive");
        if (r3 > 0.0 && r3 > r_atom)
            raise(kConfig, "three-body cutoff cannot exceed the atom cutoff");
        const int64_t total = gmd_params_size(F, K, L);
        {   // ToyPotentialParams::validate (potential.cpp:150-176), blob order
            const int64_t f = F, k = K, l = L;
            const std::pair<const char*, int64_t> arrays[] = {
                {"embedding", 119 * f}, {"layer_w", l * f * f}, {"layer_b", l * f},
                {"basis_proj", f * k}, {"basis3_proj", f * k}, {"w3", f * f}, {"w4", f * f},
                {"readout", f}};
            int64_t off = 0;
            for (const auto& a : arrays) {
                for (int64_t i = 0; i < a.second; ++i)
                    if (!std::isfinite(blob[off + i]))
                        raise(kConfig, std::string("parameter array ") + a.first +
                                           " contains a non-finite value");
                off += a.second;
            }
            if (off != total) raise(kRuntime, "internal: parameter blob layout");
        }
        h->generic = F != kF || K != kK || L > kMaxLayers;
        if (h->generic && (F > kGenMaxF || K > kGenMaxK))
            raise(kConfig, "feature_width <= 128 and basis_count <= 32 are supported");
        // fp32 tables of the width-generic kernels: the whole model for other
        // widths; for F = 16, K = 8 the three-body fallback for centers with
        // more in-bonds than the tuned kernels stage (kMaxBondsPerAtom)
        build_gen_tables(h, F, K, L, r_atom, r3, blob);
        if (h->generic) {
            h->F = F;
            h->K = K;
            h->L = L;
            h->p_r_atom = r_atom;
            h->p_r3 = r3;
            h->params_set = true;
            static std::atomic<uint64_t> gen_ver{1ull << 62};
            h->mc_ver = gen_ver++;
            return;
        }
        ModelConst& m = h->mc;
        std::memset(&m, 0, sizeof m);
        const double* q = blob;
        for (int i = 0; i < 119 * F; ++i) m.emb[i] = (float)*q++;
        for (int l = 0; l < L; ++l)
            for (int i = 0; i < F * F; ++i) m.W[l][i] = (float)*q++;
        for (int l = 0; l < L; ++l)
            for (int i = 0; i < F; ++i) m.b[l][i] = (float)*q++;
        for (int i = 0; i < F * K; ++i) m.P[i] = (float)*q++;
        for (int f = 0; f < F; ++f)
            for (int k = 0; k < K; ++k) m.PT[k * F + f] = m.P[f * K + k];
        {
            const double* Pd = blob + 119 * F + (size_t)L * F * F + (size_t)L * F;
            for (int i = 0; i < F * K; ++i) m.Pk[i] = (float)(Pd[i] * (double)(i % K));
        }
        for (int i = 0; i < F * K; ++i) m.P3[i] = (float)*q++;
        for (int i = 0; i < F * F; ++i) m.W3[i] = (float)*q++;
        for (int i = 0; i < F * F; ++i) m.W4[i] = (float)*q++;
        for (int f = 0; f < F; ++f) {
            for (int k = 0; k < K; ++k) m.P3T[k * F + f] = m.P3[f * K + k];
            for (int g = 0; g < F; ++g) {
                m.W3T[g * F + f] = m.W3[f * F + g];
                m.W4T[g * F + f] = m.W4[f * F + g];
            }
        }
        {   // B3 = W3 P3 in fp64 from the blob (three-body backward, E = B3^T y)
            const double* W3d = blob + 119 * F + (size_t)L * F * F + (size_t)L * F + (size_t)F * K + (size_t)F * K;
            const double* P3d = blob + 119 * F + (size_t)L * F * F + (size_t)L * F + (size_t)F * K;
            for (int f = 0; f < F; ++f)
                for (int k = 0; k < K; ++k) {
                    double acc = 0.0;
                    for (int g = 0; g < F; ++g) acc += W3d[f * F + g] * P3d[g * K + k];
                    m.B3[f * K + k] = (float)acc;
                }
        }
        for (int i = 0; i < F; ++i) m.ro[i] = (float)*q++;
        m.rc = (float)r_atom;
        m.inv_rc = (float)(1.0 / r_atom);
        m.inv_sigma = (float)(K / r_atom);  // sigma = rc / K (potential.cpp:34)
        m.mu_step = K > 1 ? (float)(r_atom / (K - 1)) : 0.f;
        {
            const double sl2e = std::sqrt(1.4426950408889634);  // sqrt(log2 e)
            m.a2 = (float)(sl2e * K / r_atom);
            m.pi_rc = (float)(3.14159265358979323846 / r_atom);
            for (int k = 0; k < K; ++k)
                m.bx[k] = (float)((K > 1 ? r_atom * k / (K - 1) : 0.0) * sl2e * K / r_atom);
        }
        const double r3e = r3 > 0.0 ? r3 : 1.0;
        m.r3 = (float)r3e;
        m.inv_r3 = (float)(1.0 / r3e);
        m.inv_sigma3 = (float)(K / r3e);
        m.mu_step3 = K > 1 ? (float)(r3e / (K - 1)) : 0.f;
        m.L = L;
        h->F = F;
        h->K = K;
        h->L = L;
        h->p_r_atom = r_atom;
        h->p_r3 = r3;
        h->params_set = true;
        static std::atomic<uint64_t> next_ver{1};
        h->mc_ver = next_ver++;
    });
}

int gmd_forward(gmd_handle* h, double* energy, void* per_atom, void* forces, double* stress,
                double* timing, uint32_t flags) {
    return run(h, [&] { forward_impl(h, energy, per_atom, forces, stress, timing, flags); });
}

int gmd_num_nodes(const gmd_handle* h, int64_t* n) {
    if (!h || !n) return GMD_ERR_ARG;
    *n = h->built ? h->n : 0;
    return GMD_OK;
}
int gmd_num_edges(const gmd_handle* h, int64_t* ne) {
    if (!h || !ne) return GMD_ERR_ARG;
    *ne = h->built ? h->ne : 0;
    return GMD_OK;
}
int gmd_num_partitions(const gmd_handle* h, int* p) {
    if (!h || !p) return GMD_ERR_ARG;
    *p = h->p;
    return GMD_OK;
}

int gmd_get_graph(gmd_handle* h, int64_t* src, int64_t* dst, int32_t* off, double* dist,
                  double* vec) {
    return run(h, [&] {
        need_built(h);
        if (h->graph_only) raise(kConfig, "this handle holds partitions of a caller-supplied graph");
        const int64_t ne = h->ne;
        if (ne == 0) return;
        cudaStream_t s = h->stream;
        int32_t* edst = h->edst.get<int32_t>(ne);
        launch_edge_dst(h->row.as<int32_t>(), h->n, edst, s);
        // staging: src, dst (i64), off (3 x i32), dist, vec (3 x f64)
        char* tmp = h->exp_tmp.get<char>((size_t)ne * (8 + 8 + 12 + 8 + 24));
        int64_t* t_src = reinterpret_cast<int64_t*>(tmp);
        int64_t* t_dst = t_src + ne;
        double* t_dist = reinterpret_cast<double*>(t_dst + ne);
        double* t_vec = t_dist + ne;
        int32_t* t_off = reinterpret_cast<int32_t*>(t_vec + 3 * ne);
        if (!h->img_ok) {  // re-run the (deterministic) emit once with image output
            NLBuffers b{};
            b.pos = h->pos.as<double>();
            b.cell = h->cell.as<int32_t>();
            b.pos4 = h->pos4.as<double4>();
            b.cell4 = h->cell4.as<int4>();
            b.bcnt = h->bcnt.as<int32_t>();
            b.flags = h->flags.as<int32_t>();
            GraphDev ge;
            ge.n = h->n;
            ge.ne = ne;
            ge.row = h->row.as<int32_t>();
            ge.src = h->src.as<int32_t>();
            ge.img = h->img.get<uint32_t>(std::max<int64_t>(1, ne));
            ge.vd = h->vd.as<float4>();
            ge.d = h->ed.as<float>();
            ge.bond = h->has_lg ? h->ebond.as<uint8_t>() : nullptr;
            launch_nl_emit(h->geom, h->n, h->emit_cap, h->slab.as<unsigned long long>(), b, ge, s);
            h->img_ok = true;
        }
        GraphDev gd;
        gd.n = h->n;
        gd.ne = ne;
        gd.row = h->row.as<int32_t>();
        gd.src = h->src.as<int32_t>();
        gd.img = h->img.as<uint32_t>();
        launch_export_graph(h->geom, h->pos.as<double>(), gd, edst, t_src, t_dst, t_off, t_dist,
                            t_vec, s);
        if (src) GMD_CUDA(cudaMemcpyAsync(src, t_src, 8 * ne, cudaMemcpyDeviceToHost, s));
        if (dst) GMD_CUDA(cudaMemcpyAsync(dst, t_dst, 8 * ne, cudaMemcpyDeviceToHost, s));
        if (off) GMD_CUDA(cudaMemcpyAsync(off, t_off, 12 * ne, cudaMemcpyDeviceToHost, s));
        if (dist) GMD_CUDA(cudaMemcpyAsync(dist, t_dist, 8 * ne, cudaMemcpyDeviceToHost, s));
        if (vec) GMD_CUDA(cudaMemcpyAsync(vec, t_vec, 24 * ne, cudaMemcpyDeviceToHost, s));
        sync(h);
    });
}

int gmd_get_system(gmd_handle* h, double* pos, double* lattice) {
    return run(h, [&] {
        need_built(h);
        if (pos)
            GMD_CUDA(cudaMemcpyAsync(pos, h->pos.as<double>(), 24 * h->n, cudaMemcpyDeviceToHost,
                                     h->stream));
        if (lattice) std::memcpy(lattice, h->lat, sizeof h->lat);
        sync(h);
    });
}

namespace {

// ---------------------------------------------------------------------------
// Free builder API (partitioner.hpp:66-106, linegraph.hpp:26-78): the same
// partition / bond / line-graph kernels as gmd_build, on a caller's graph
// ---------------------------------------------------------------------------
// wrapped fractional coordinate along `axis` of every atom (fractional_along_axis,
// partitioner.cpp:38-44) into h->fw; positions as given (no ensure_periodic)
const double* wrapped_fracs(gmd_handle* h, int64_t n, const double* pos, const double* lat, int axis) {
    cudaStream_t s = h->stream;
    if (std::abs(det3(lat)) < 1e-10) raise(kConfig, "degenerate cell");
    double* dpos = h->fr_pos.get<double>(3 * n);
    GMD_CUDA(cudaMemcpyAsync(dpos, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    Geom g{};
    std::memcpy(g.L, lat, sizeof g.L);
    inverse3(lat, g.inv);
    g.bins[0] = g.bins[1] = g.bins[2] = 1;
    g.axis = axis;
    NLBuffers b{};
    b.pos = dpos;
    b.cell = h->fr_cell.get<int32_t>(3 * n);
    b.fw_axis = h->fr_fw.get<double>(n);
    b.bin = h->fr_bin.get<int32_t>(n);
    b.bin_cnt = h->fr_cnt.get<int32_t>(1);
    b.flags = h->fr_flags.get<int32_t>(4);
    GMD_CUDA(cudaMemsetAsync(b.bin_cnt, 0, 4, s));
    GMD_CUDA(cudaMemsetAsync(b.flags, 0, 16, s));
    launch_wrap(g, n, b, s);
    return b.fw_axis;
}

void check_rule_args(int64_t n, int p) {  // choose_partition_rule (partitioner.cpp:48-51)
    if (p < 1) raise(kConfig, "partition count must be >= 1");
    if (p > kMaxParts) raise(kConfig, "partition count limited to 64");
    if ((int64_t)p > n) raise(kConfig, "more partitions than atoms");
}

int longest_axis(const double* lat) {  // partitioner.cpp:57-64
    int axis = 0;
    double best = -1.0;
    for (int k = 0; k < 3; ++k) {
        double len = vnorm(row3(lat, k));
        if (len > best) {
            best = len;
            axis = k;
        }
    }
    return axis;
}

void partitions_impl(gmd_handle* h, int64_t n, const double* pos, const double* lat, int64_t ne,
                     const int64_t* src, const int64_t* dst, const int32_t* off, const double* dist,
                     double cutoff, double r3, double tau, int axis, int p, const double* bounds,
                     const int32_t* owner, uint32_t flags) {
    cudaStream_t s = h->stream;
    h->built = false;
    h->graph_only = true;
    h->closure_ready = false;
    h->hc_ready = h->hcb_ready = false;
    h->line_dev_ready = false;
    h->ctab_ok = false;
    h->atoms.ready = h->bonds.ready = false;
    h->corrupted = false;
    if (n <= 0) raise(kConfig, "graph has no nodes");
    if (p < 1) raise(kConfig, "partition count must be >= 1");
    if (p > kMaxParts) raise(kConfig, "partition count limited to 64");
    if (ne < 0 || (ne > 0 && (!src || !dst || !off))) raise(kArg, "null edge arrays");
    if (n >= ((int64_t)1 << 31) - 1 || ne >= ((int64_t)1 << 31) - 1)
        raise(kConfig, "graph exceeds the int32 index range");
    if (r3 > 0.0) {  // check_ranges (linegraph.cpp:10-14)
        if (r3 > cutoff) raise(kConfig, "three-body range cannot exceed the atom graph cutoff");
        if (tau < 0.0) raise(kConfig, "tolerance tau must be >= 0");
        if (ne > 0 && !dist) raise(kArg, "null distance array");
    }
    if (bounds) {
        h->bounds.assign(bounds, bounds + p + 1);
    } else {
        h->bounds.assign(p + 1, 0.0);
        h->bounds[p] = 1.0;
    }
    if (lat) std::memcpy(h->lat, lat, sizeof h->lat);
    // check_slab_widths (partitioner.cpp:21-33), with the graph's cutoff
    if (p > 1 && !(flags & GMD_ALLOW_NARROW)) {
        if (!lat || !bounds) raise(kArg, "slab-width check needs the lattice and the rule");
        const double perp = perp_width(lat, axis);
        for (int i = 0; i < p; ++i) {
            const double width = (bounds[i + 1] - bounds[i]) * perp;
            if (width < cutoff)
                raise(kConfig, "partition-width error: slab " + std::to_string(i) + " is " +
                                   std::to_string(width) + " A wide, below the cutoff " +
                                   std::to_string(cutoff) + " A");
        }
    }
    h->n = n;
    h->ne = ne;
    h->p = p;
    h->rc = cutoff;
    h->r3 = r3;
    h->tau = tau;
    h->axis = axis;
    h->allow_narrow = (flags & GMD_ALLOW_NARROW) != 0;
    h->n_own = n;

    // owners: given, or which_partition of each atom's wrapped fraction
    int32_t* ownp = h->atoms.owner.get<int32_t>(n);
    if (owner) {
        for (int64_t i = 0; i < n; ++i)
            if (owner[i] < 0 || owner[i] >= p) raise(kArg, "owner out of range");
        GMD_CUDA(cudaMemcpyAsync(ownp, owner, 4 * n, cudaMemcpyHostToDevice, s));
    } else if (p == 1) {
        GMD_CUDA(cudaMemsetAsync(ownp, 0, 4 * n, s));
    } else {
        if (!pos || !lat || !bounds) raise(kArg, "owners need positions, lattice and rule");
        const double* fw = wrapped_fracs(h, n, pos, lat, axis);
        Bounds bd{};
        bd.p = p;
        for (int k = 0; k <= p; ++k) bd.b[k] = bounds[k];
        launch_owner(fw, n, bd, ownp, s);
    }
    // CSR of the caller's edges: canonical order is dst-major (neighborlist.hpp:14-16)
    std::vector<int32_t> row(n + 1, 0), s32(ne);
    for (int64_t e = 0; e < ne; ++e) {
        if (dst[e] < 0 || dst[e] >= n || src[e] < 0 || src[e] >= n)
            raise(kArg, "edge endpoint out of range");
        if (e > 0 && dst[e] < dst[e - 1]) raise(kConfig, "graph edges are not in dst-major order");
        ++row[dst[e] + 1];
        s32[e] = (int32_t)src[e];
    }
    for (int64_t v = 0; v < n; ++v) row[v + 1] += row[v];
    int32_t* rowp = h->row.get<int32_t>(n + 1);
    int32_t* srcp = h->src.get<int32_t>(std::max<int64_t>(1, ne));
    GMD_CUDA(cudaMemcpyAsync(rowp, row.data(), 4 * (n + 1), cudaMemcpyHostToDevice, s));
    if (ne) GMD_CUDA(cudaMemcpyAsync(srcp, s32.data(), 4 * ne, cudaMemcpyHostToDevice, s));
    int32_t* fl = h->flags.get<int32_t>(4);
    GMD_CUDA(cudaMemsetAsync(fl, 0, 16, s));
    GraphDev gd;
    gd.n = n;
    gd.ne = ne;
    gd.row = rowp;
    gd.src = srcp;
    gd.img = h->img.get<uint32_t>(std::max<int64_t>(1, ne));
    gd.bond = r3 > 0.0 ? h->ebond.get<uint8_t>(std::max<int64_t>(1, ne)) : nullptr;
    if (ne) {
        int32_t* off_d = reinterpret_cast<int32_t*>(h->exp_tmp.get<char>((size_t)ne * 20));
        double* dist_d = reinterpret_cast<double*>(off_d + 3 * ne + (ne & 1));
        GMD_CUDA(cudaMemcpyAsync(off_d, off, 12 * ne, cudaMemcpyHostToDevice, s));
        if (r3 > 0.0) GMD_CUDA(cudaMemcpyAsync(dist_d, dist, 8 * ne, cudaMemcpyHostToDevice, s));
        launch_graph_import(ne, off_d, dist_d, r3 > 0.0 ? r3 + tau : -1.0, gd.img, gd.bond, fl, s);
    }
    h->img_ok = true;
    LayoutState& A = h->atoms;
    if (p == 1) {
        A.p = 1;
        A.nid = n;
        A.list_off = {0, (int32_t)n, (int32_t)n, (int32_t)n};
        A.rows = n;
        A.nfrom = 0;
        A.ready = true;
        A.api_ready = A.dups_ready = false;
        A.h_nodes.clear();
    } else {
        auto* reqp = A.req.get<unsigned long long>(n);
        GMD_CUDA(cudaMemsetAsync(reqp, 0, sizeof(unsigned long long) * n, s));
        launch_required(rowp, srcp, n, ownp, reqp, s);
        build_layout(h, A, ownp, reqp, n, p);
        launch_edge_lsrc(rowp, srcp, n, ownp, A.crow.as<int32_t>(), A.node_array.as<int32_t>(),
                         A.list_off_d.as<int32_t>(), p, h->lsrc.get<int32_t>(std::max<int64_t>(1, ne)),
                         fl, s);
    }
    h->has_lg = r3 > 0.0;
    h->nb = 0;
    if (h->has_lg) {
        int32_t* bc = h->bcnt.get<int32_t>(n);
        launch_row_bond_count(rowp, gd.bond, n, bc, s);
        int32_t* br = h->brow.get<int32_t>(n + 1);
        scan_i32(h, bc, br, n);
        int32_t nb32 = 0;
        GMD_CUDA(cudaMemcpyAsync(&nb32, br + n, 4, cudaMemcpyDeviceToHost, s));
        sync(h);
        h->nb = nb32;
        int32_t* be = h->bedge.get<int32_t>(std::max<int64_t>(1, h->nb));
        int32_t* bv = h->brev.get<int32_t>(std::max<int64_t>(1, h->nb));
        int32_t* ebid = h->ebid.get<int32_t>(std::max<int64_t>(1, ne));
        launch_bond_edges(rowp, gd.bond, n, br, be, ebid, s);
        launch_bond_rev(n, gd, br, be, ebid, bv, fl, ownp, -1, s);
    }
    int32_t hf[4];
    GMD_CUDA(cudaMemcpyAsync(hf, fl, 16, cudaMemcpyDeviceToHost, s));
    sync(h);
    // a caller's graph need not be closed under reversal: a bond without a
    // reverse (flag 32) simply has none to skip (is_reverse_pair, linegraph.cpp:16-21)
    if (hf[1] & kErrImgRange)
        raise(kConfig, "periodic image offset exceeds the packed range (+-511 cells)");
    if (hf[1] & 8) raise(kRuntime, "internal: edge endpoint missing from partition layout");
    h->built = true;
}

// two-hop closures of every partition at once (linegraph.cpp:45-65)
void ensure_closure(gmd_handle* h) {
    need_built(h);
    if (h->closure_ready) return;
    cudaStream_t s = h->stream;
    const int64_t n = h->n;
    auto* m0 = h->cmask.get<unsigned long long>(2 * n);
    auto* m1 = m0 + n;
    launch_closure_init(h->atoms.owner.as<int32_t>(), n, m0, s);
    launch_closure_hop(h->row.as<int32_t>(), h->src.as<int32_t>(), n, m0, m1, s);
    launch_closure_hop(h->row.as<int32_t>(), h->src.as<int32_t>(), n, m1, m0, s);
    h->closure_ready = true;
}
}  // namespace

// ---- free builders ----------------------------------------------------------
int gmd_partition_rule(gmd_handle* h, int64_t n, const double* pos, const double* lattice, int p,
                       int equal_width, int* axis, double* boundaries) {
    return run(h, [&] {
        if (!lattice || !axis || !boundaries || (n > 0 && !pos)) raise(kArg, "null argument");
        check_rule_args(n, p);
        if (std::abs(det3(lattice)) < 1e-10) raise(kConfig, "degenerate cell");
        *axis = longest_axis(lattice);
        boundaries[0] = 0.0;
        boundaries[p] = 1.0;
        if (p == 1) return;
        if (equal_width) {
            for (int k = 1; k < p; ++k) boundaries[k] = (double)k / p;
            return;
        }
        const double* fw = wrapped_fracs(h, n, pos, lattice, *axis);
        quantile_walls(h, fw, n, p, boundaries);
        for (int k = 1; k <= p; ++k)
            if (boundaries[k] <= boundaries[k - 1])
                raise(kConfig,
                      "cannot place distinct partition boundaries; coordinates along the axis "
                      "are degenerate");
    });
}

int gmd_assign_owners(gmd_handle* h, int64_t n, const double* pos, const double* lattice, int axis,
                      int p, const double* boundaries, double* fracs, int32_t* owner) {
    return run(h, [&] {
        if (n <= 0) return;
        if (!pos || !lattice) raise(kArg, "null argument");
        if (axis < 0 || axis > 2) raise(kArg, "axis out of range");
        const double* fw = wrapped_fracs(h, n, pos, lattice, axis);
        cudaStream_t s = h->stream;
        if (owner) {
            if (!boundaries || p < 1 || p > kMaxParts) raise(kArg, "bad partition rule");
            Bounds bd{};
            bd.p = p;
            for (int k = 0; k <= p; ++k) bd.b[k] = boundaries[k];
            int32_t* o = h->flagtmp.get<int32_t>(n + 1);
            launch_owner(fw, n, bd, o, s);
            GMD_CUDA(cudaMemcpyAsync(owner, o, 4 * n, cudaMemcpyDeviceToHost, s));
        }
        if (fracs) GMD_CUDA(cudaMemcpyAsync(fracs, fw, 8 * n, cudaMemcpyDeviceToHost, s));
        sync(h);
    });
}

int gmd_build_partitions(gmd_handle* h, int64_t n, const double* pos, const double* lattice,
                         int64_t ne, const int64_t* src, const int64_t* dst, const int32_t* off,
                         const double* dist, double cutoff, double r3, double tau, int axis, int p,
                         const double* boundaries, const int32_t* owner, uint32_t flags) {
    return run(h, [&] {
        partitions_impl(h, n, pos, lattice, ne, src, dst, off, dist, cutoff, r3, tau, axis, p,
                        boundaries, owner, flags);
    });
}

int gmd_get_closure(gmd_handle* h, int part, int64_t* count, int64_t* ids) {
    return run(h, [&] {
        ensure_closure(h);
        check_part(h, part);
        std::vector<unsigned long long> m;
        d2h(h, m, h->cmask.as<unsigned long long>(), h->n);
        sync(h);
        int64_t c = 0;
        for (int64_t v = 0; v < h->n; ++v)
            if (m[v] >> part & 1ull) {
                if (ids) ids[c] = v;
                ++c;
            }
        if (count) *count = c;
    });
}

int gmd_get_bond_tables(gmd_handle* h, uint64_t* mask) {
    return run(h, [&] {
        need_built(h);
        if (!h->has_lg) raise(kConfig, "no line graph was built");
        ensure_closure(h);
        cudaStream_t s = h->stream;
        const int64_t nb = h->nb;
        int32_t* edst = h->edst.get<int32_t>(std::max<int64_t>(1, h->ne));
        launch_edge_dst(h->row.as<int32_t>(), h->n, edst, s);
        auto* bm = h->bmask.get<unsigned long long>(std::max<int64_t>(1, nb));
        launch_bond_tables(nb, h->bedge.as<int32_t>(), edst, h->src.as<int32_t>(),
                           h->cmask.as<unsigned long long>(), bm, s);
        if (nb) GMD_CUDA(cudaMemcpyAsync(mask, bm, 8 * nb, cudaMemcpyDeviceToHost, s));
        sync(h);
    });
}

int gmd_brute_force_line_graph(gmd_handle* h, int64_t* count, int64_t* pairs) {
    return run(h, [&] {
        need_built(h);
        if (!h->has_lg) raise(kConfig, "no line graph was built");
        cudaStream_t s = h->stream;
        const int64_t n = h->n, nb = h->nb;
        int32_t* edst = h->edst.get<int32_t>(std::max<int64_t>(1, h->ne));
        launch_edge_dst(h->row.as<int32_t>(), h->n, edst, s);
        // by_dst = the bond CSR (brow / bond ids in order); by_src built here
        std::vector<int32_t> be, es;
        d2h(h, be, h->bedge.as<int32_t>(), nb);
        d2h(h, es, h->src.as<int32_t>(), h->ne);
        sync(h);
        std::vector<int32_t> orow(n + 1, 0), obond(std::max<int64_t>(1, nb)), inb(std::max<int64_t>(1, nb));
        for (int64_t b = 0; b < nb; ++b) ++orow[es[be[b]] + 1];
        for (int64_t v = 0; v < n; ++v) orow[v + 1] += orow[v];
        std::vector<int32_t> fill(orow.begin(), orow.end() - 1);
        for (int64_t b = 0; b < nb; ++b) obond[fill[es[be[b]]]++] = (int32_t)b;
        for (int64_t b = 0; b < nb; ++b) inb[b] = (int32_t)b;
        int32_t* d_orow = h->lcnt.get<int32_t>(3 * (n + 1) + 2 * std::max<int64_t>(1, nb));
        int32_t* d_obond = d_orow + (n + 1);
        int32_t* d_inb = d_obond + std::max<int64_t>(1, nb);
        int32_t* d_cnt = d_inb + std::max<int64_t>(1, nb);
        int32_t* d_off = d_cnt + (n + 1);
        GMD_CUDA(cudaMemcpyAsync(d_orow, orow.data(), 4 * (n + 1), cudaMemcpyHostToDevice, s));
        if (nb) {
            GMD_CUDA(cudaMemcpyAsync(d_obond, obond.data(), 4 * nb, cudaMemcpyHostToDevice, s));
            GMD_CUDA(cudaMemcpyAsync(d_inb, inb.data(), 4 * nb, cudaMemcpyHostToDevice, s));
        }
        launch_brute_line(n, h->brow.as<int32_t>(), d_inb, d_orow, d_obond, h->bedge.as<int32_t>(),
                          h->src.as<int32_t>(), edst, h->img.as<uint32_t>(), d_cnt, nullptr, nullptr, s);
        scan_i32(h, d_cnt, d_off, n);
        int32_t T = 0;
        GMD_CUDA(cudaMemcpyAsync(&T, d_off + n, 4, cudaMemcpyDeviceToHost, s));
        sync(h);
        int32_t* d_pairs = h->lpairs.get<int32_t>(2 * std::max<int64_t>(1, T));
        launch_brute_line(n, h->brow.as<int32_t>(), d_inb, d_orow, d_obond, h->bedge.as<int32_t>(),
                          h->src.as<int32_t>(), edst, h->img.as<uint32_t>(), d_cnt, d_off, d_pairs, s);
        std::vector<int32_t> hp;
        d2h(h, hp, d_pairs, 2 * (size_t)T);
        sync(h);
        h->hcb_ready = false;  // lpairs / lcnt are shared with the line-graph cache
        h->line_dev_ready = false;
        if (count) *count = T;
        if (pairs) {
            std::vector<std::pair<int64_t, int64_t>> v((size_t)T);
            for (int64_t t = 0; t < T; ++t) v[t] = {hp[2 * t], hp[2 * t + 1]};
            std::sort(v.begin(), v.end());
            for (int64_t t = 0; t < T; ++t) {
                pairs[2 * t] = v[t].first;
                pairs[2 * t + 1] = v[t].second;
            }
        }
    });
}

int gmd_brute_force_neighbor_list(gmd_handle* h, int64_t n, const double* pos,
                                  const double* lattice, const uint8_t* pbc, double cutoff,
                                  int64_t* ne_out, int64_t* src, int64_t* dst, int32_t* off,
                                  double* dist, double* vec) {
    return run(h, [&] {
        if (cutoff <= 0.0) raise(kConfig, "cutoff must be positive");
        if (n == 0) raise(kConfig, "cannot build neighbor list for empty system");
        if (n > 5000) raise(kConfig, "brute force guard: N > 5000");
        if (!pos || !lattice || !ne_out) raise(kArg, "null argument");
        cudaStream_t s = h->stream;
        h->built = false;
        h->n = n;
        double* dpos = h->pos.get<double>(3 * n);
        GMD_CUDA(cudaMemcpyAsync(dpos, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
        std::memcpy(h->lat, lattice, sizeof h->lat);
        ensure_periodic_dev(h, pbc, cutoff);  // pads non-periodic axes (system.cpp:242-270)
        if (std::abs(det3(h->lat)) < 1e-10)
            raise(kConfig, "periodic system requires an invertible lattice");
        Geom g{};
        std::memcpy(g.L, h->lat, sizeof g.L);
        inverse3(h->lat, g.inv);
        g.bins[0] = g.bins[1] = g.bins[2] = 1;
        NLBuffers b{};
        b.pos = dpos;
        b.cell = h->cell.get<int32_t>(3 * n);
        b.fw_axis = h->fw.get<double>(n);
        b.bin = h->bin.get<int32_t>(n);
        b.bin_cnt = h->bin_cnt.get<int32_t>(1);
        b.flags = h->flags.get<int32_t>(4);
        GMD_CUDA(cudaMemsetAsync(b.bin_cnt, 0, 4, s));
        GMD_CUDA(cudaMemsetAsync(b.flags, 0, 16, s));
        launch_wrap(g, n, b, s);  // cell_of of wrap_for_search (neighborlist.cpp:42-50)
        BruteNL bn{};
        std::memcpy(bn.L, h->lat, sizeof bn.L);
        bn.cutoff2 = cutoff * cutoff;
        for (int k = 0; k < 3; ++k)  // neighborlist.cpp:211-214
            bn.span[k] = (int)std::ceil(cutoff / perp_width(h->lat, k)) + 1;
        int32_t* cnt = h->deg.get<int32_t>(n + 1);
        int32_t* rowoff = h->row.get<int32_t>(n + 1);
        launch_brute_nl(bn, n, dpos, b.cell, cnt, nullptr, nullptr, nullptr, s);
        scan_i32(h, cnt, rowoff, n);
        int32_t ne32 = 0;
        GMD_CUDA(cudaMemcpyAsync(&ne32, rowoff + n, 4, cudaMemcpyDeviceToHost, s));
        sync(h);
        const int64_t ne = ne32;
        *ne_out = ne;
        if (!src && !dst && !off && !dist && !vec) return;
        int32_t* d_src = h->src.get<int32_t>(std::max<int64_t>(1, ne));
        int32_t* d_off = reinterpret_cast<int32_t*>(h->exp_tmp.get<char>(std::max<int64_t>(1, ne) * 12));
        launch_brute_nl(bn, n, dpos, b.cell, cnt, rowoff, d_src, d_off, s);
        std::vector<int32_t> hs, ho, hr;
        d2h(h, hs, d_src, ne);
        d2h(h, ho, d_off, 3 * ne);
        d2h(h, hr, rowoff, n + 1);
        sync(h);
        // assemble (neighborlist.cpp:60-85): rows in (src, ox, oy, oz) order
        std::vector<int32_t> order(ne), ssrc(ne), sdst(ne), soff(3 * ne);
        for (int64_t i = 0; i < n; ++i) {
            const int32_t a = hr[i], z = hr[i + 1];
            for (int32_t k = a; k < z; ++k) order[k] = k;
            std::sort(order.begin() + a, order.begin() + z, [&](int32_t x, int32_t y) {
                if (hs[x] != hs[y]) return hs[x] < hs[y];
                for (int c = 0; c < 3; ++c)
                    if (ho[3 * x + c] != ho[3 * y + c]) return ho[3 * x + c] < ho[3 * y + c];
                return false;
            });
            for (int32_t k = a; k < z; ++k) {
                ssrc[k] = hs[order[k]];
                sdst[k] = (int32_t)i;
                for (int c = 0; c < 3; ++c) soff[3 * k + c] = ho[3 * order[k] + c];
            }
        }
        if (src) for (int64_t e = 0; e < ne; ++e) src[e] = ssrc[e];
        if (dst) for (int64_t e = 0; e < ne; ++e) dst[e] = sdst[e];
        if (off) std::copy(soff.begin(), soff.end(), off);
        if (dist || vec) {  // exact fp64 geometry on the device
            int32_t* d_dst = h->edst.get<int32_t>(std::max<int64_t>(1, ne));
            double* d_dist = h->fw.get<double>(std::max<int64_t>(1, 4 * ne));
            GMD_CUDA(cudaMemcpyAsync(d_src, ssrc.data(), 4 * ne, cudaMemcpyHostToDevice, s));
            GMD_CUDA(cudaMemcpyAsync(d_dst, sdst.data(), 4 * ne, cudaMemcpyHostToDevice, s));
            GMD_CUDA(cudaMemcpyAsync(d_off, soff.data(), 12 * ne, cudaMemcpyHostToDevice, s));
            launch_edge_geometry(bn, ne, dpos, d_src, d_dst, d_off, d_dist, d_dist + ne, s);
            std::vector<double> hd;
            d2h(h, hd, d_dist, 4 * ne);
            sync(h);
            if (dist) std::copy(hd.begin(), hd.begin() + ne, dist);
            if (vec) std::copy(hd.begin() + ne, hd.end(), vec);
        }
    });
}

int gmd_get_csr(gmd_handle* h, int32_t* row, int32_t* src) {
    return run(h, [&] {
        need_built(h);
        cudaStream_t s = h->stream;
        if (row) GMD_CUDA(cudaMemcpyAsync(row, h->row.as<int32_t>(), 4 * (h->n + 1), cudaMemcpyDeviceToHost, s));
        if (src && h->ne) GMD_CUDA(cudaMemcpyAsync(src, h->src.as<int32_t>(), 4 * h->ne, cudaMemcpyDeviceToHost, s));
        sync(h);
    });
}

int gmd_util_ensure_periodic(gmd_handle* h, int64_t n, const double* pos, const double* lattice,
                             const uint8_t* pbc, double cutoff, double* out_pos, double* out_lat) {
    return run(h, [&] {
        if (!lattice || !pbc || !out_lat || (n > 0 && (!pos || !out_pos))) raise(kArg, "null argument");
        h->built = false;
        h->n = n;
        std::memcpy(h->lat, lattice, sizeof h->lat);
        if (n > 0) {
            double* d = h->pos.get<double>(3 * n);
            GMD_CUDA(cudaMemcpyAsync(d, pos, 24 * n, cudaMemcpyHostToDevice, h->stream));
            ensure_periodic_dev(h, pbc, cutoff);
            GMD_CUDA(cudaMemcpyAsync(out_pos, d, 24 * n, cudaMemcpyDeviceToHost, h->stream));
            sync(h);
        } else if (!(pbc[0] && pbc[1] && pbc[2])) {
            if (cutoff <= 0.0) raise(kConfig, "cutoff must be positive");
            raise(kConfig, "cannot pad the cell of an empty system");
        }
        std::memcpy(out_lat, h->lat, sizeof h->lat);
    });
}

int gmd_get_rule(gmd_handle* h, int* axis, double* boundaries) {
    return run(h, [&] {
        need_built(h);
        if (axis) *axis = h->axis;
        if (boundaries) std::copy(h->bounds.begin(), h->bounds.end(), boundaries);
    });
}

int gmd_get_owner(gmd_handle* h, int32_t* owner) {
    return run(h, [&] {
        need_built(h);
        GMD_CUDA(cudaMemcpyAsync(owner, h->atoms.owner.as<int32_t>(), 4 * h->n,
                                 cudaMemcpyDeviceToHost, h->stream));
        sync(h);
    });
}

int gmd_get_layout_size(gmd_handle* h, int part, int bonds, int64_t* size) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        check_part(h, part);
        const int stride = 1 + 2 * ls.p;
        *size = ls.list_off[(size_t)(part + 1) * stride] - ls.list_off[(size_t)part * stride];
    });
}

int gmd_get_layout(gmd_handle* h, int part, int bonds, int64_t* node_array, int64_t* markers) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        check_part(h, part);
        const int p = ls.p, stride = 1 + 2 * p;
        const int64_t b0 = ls.list_off[(size_t)part * stride];
        const int64_t b1 = ls.list_off[(size_t)(part + 1) * stride];
        if (node_array) {
            const auto& nodes = host_nodes(h, ls);
            for (int64_t r = b0; r < b1; ++r) node_array[r - b0] = nodes[r];
        }
        if (markers) {
            markers[0] = 0;
            for (int bb = 0; bb < 1 + 2 * p; ++bb)
                markers[bb + 1] = ls.list_off[(size_t)part * stride + bb + 1] - b0;
        }
    });
}

int gmd_get_num_duplicates(gmd_handle* h, int part, int bonds, int64_t* count) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        check_part(h, part);
        *count = (int64_t)dup_pairs(h, ls, part).size();
    });
}

int gmd_get_duplicates(gmd_handle* h, int part, int bonds, int64_t* pairs) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        check_part(h, part);
        auto v = dup_pairs(h, ls, part);
        for (size_t k = 0; k < v.size(); ++k) {
            pairs[2 * k] = v[k].first;
            pairs[2 * k + 1] = v[k].second;
        }
    });
}

namespace {
// owned edges of a partition in ascending global id (partitioner.cpp:200-216)
void owned_edges(gmd_handle* h, int part, std::vector<int64_t>* owned, std::vector<int64_t>* ls,
                 std::vector<int64_t>* ld, std::vector<int64_t>* border) {
    ensure_host_cache(h);
    check_part(h, part);
    const int64_t base = h->atoms.base(part);
    int64_t k = 0;
    for (int64_t v = 0; v < h->n; ++v) {
        if (h->h_owner[v] != part) continue;
        for (int32_t e = h->h_row[v]; e < h->h_row[v + 1]; ++e, ++k) {
            const int32_t u = h->h_src[e];
            if (owned) owned->push_back(e);
            if (ls) ls->push_back((h->p > 1 ? h->h_lsrc[e] : u) - base);
            if (ld) ld->push_back((h->p > 1 ? h->h_crow[v] : v) - base);
            if (border && h->h_owner[u] != part) border->push_back(k);
        }
    }
}
}  // namespace

int gmd_get_num_owned_edges(gmd_handle* h, int part, int64_t* count) {
    return run(h, [&] {
        ensure_host_cache(h);
        check_part(h, part);
        int64_t c = 0;
        for (int64_t v = 0; v < h->n; ++v)
            if (h->h_owner[v] == part) c += h->h_row[v + 1] - h->h_row[v];
        *count = c;
    });
}

int gmd_get_owned_edges(gmd_handle* h, int part, int64_t* owned, int64_t* local_src,
                        int64_t* local_dst) {
    return run(h, [&] {
        std::vector<int64_t> a, b, c;
        owned_edges(h, part, &a, &b, &c, nullptr);
        if (owned) std::copy(a.begin(), a.end(), owned);
        if (local_src) std::copy(b.begin(), b.end(), local_src);
        if (local_dst) std::copy(c.begin(), c.end(), local_dst);
    });
}

int gmd_get_num_border_edges(gmd_handle* h, int part, int64_t* count) {
    return run(h, [&] {
        std::vector<int64_t> b;
        owned_edges(h, part, nullptr, nullptr, nullptr, &b);
        *count = (int64_t)b.size();
    });
}

int gmd_get_border_edges(gmd_handle* h, int part, int64_t* border) {
    return run(h, [&] {
        std::vector<int64_t> b;
        owned_edges(h, part, nullptr, nullptr, nullptr, &b);
        std::copy(b.begin(), b.end(), border);
    });
}

int gmd_has_line_graph(const gmd_handle* h, int* yes) {
    if (!h || !yes) return GMD_ERR_ARG;
    *yes = h->built && h->has_lg ? 1 : 0;
    return GMD_OK;
}

namespace {
void ensure_line_cache(gmd_handle* h) {
    build_line_edges_dev(h);
    if (h->hcb_ready) return;
    const int64_t nb = h->nb;
    d2h(h, h->h_pairs, h->lpairs.as<int32_t>(), 2 * (size_t)h->nline);
    d2h(h, h->h_bedge, h->bedge.as<int32_t>(), nb);
    d2h(h, h->h_bown, h->bonds.owner.as<int32_t>(), nb);
    sync(h);
    h->hcb_ready = true;
}

// bond global id -> local row of partition `part` (canonical, first occurrence)
std::unordered_map<int32_t, int64_t> bond_g2l(gmd_handle* h, int part) {
    LayoutState& B = h->bonds;
    const auto& nodes = host_nodes(h, B);
    const int stride = 1 + 2 * B.p;
    const int64_t b0 = B.list_off[(size_t)part * stride], b1 = B.list_off[(size_t)(part + 1) * stride];
    std::unordered_map<int32_t, int64_t> m;
    m.reserve((size_t)(b1 - b0) * 2);
    for (int64_t r = b0; r < b1; ++r) m.emplace(nodes[r], r - b0);
    return m;
}
}  // namespace

int gmd_get_num_bonds(gmd_handle* h, int64_t* nb) {
    return run(h, [&] {
        need_built(h);
        *nb = h->has_lg ? h->nb : 0;
    });
}

int gmd_get_bonds(gmd_handle* h, int64_t* edge_of_bond, int32_t* bond_owner) {
    return run(h, [&] {
        ensure_line_cache(h);
        for (int64_t b = 0; b < h->nb; ++b) {
            if (edge_of_bond) edge_of_bond[b] = h->h_bedge[b];
            if (bond_owner) bond_owner[b] = h->h_bown[b];
        }
    });
}

int gmd_get_num_line_edges(gmd_handle* h, int part, int64_t* count) {
    return run(h, [&] {
        ensure_line_cache(h);
        check_part(h, part);
        int64_t c = 0;
        const size_t T = h->h_pairs.size() / 2;
        for (size_t t = 0; t < T; ++t)
            if (h->h_bown[h->h_pairs[2 * t + 1]] == part) ++c;
        *count = c;
    });
}

int gmd_get_line_edges(gmd_handle* h, int part, int64_t* pairs) {
    return run(h, [&] {
        ensure_line_cache(h);
        check_part(h, part);
        auto g2l = bond_g2l(h, part);
        const size_t T = h->h_pairs.size() / 2;
        int64_t k = 0;
        for (size_t t = 0; t < T; ++t) {
            const int32_t e = h->h_pairs[2 * t], ep = h->h_pairs[2 * t + 1];
            if (h->h_bown[ep] != part) continue;
            auto a = g2l.find(e), b = g2l.find(ep);
            if (a == g2l.end() || b == g2l.end())
                raise(kRuntime, "dangling bond reference in line graph");
            pairs[2 * k] = a->second;
            pairs[2 * k + 1] = b->second;
            ++k;
        }
    });
}

// ---- feature API --------------------------------------------------------
int gmd_block_rows(gmd_handle* h, int bonds, int64_t* total_rows) {
    return run(h, [&] { *total_rows = layout_of(h, bonds).rows; });
}

int gmd_block_offset(gmd_handle* h, int part, int bonds, int64_t* row0) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        check_part(h, part);
        *row0 = ls.base(part);
    });
}

int gmd_transfer(gmd_handle* h, int bonds, void* dev_buf, int width, int dtype) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        const int es = elem_size(dtype);
        if (width < 1) raise(kArg, "width must be >= 1");
        if (ls.nfrom == 0) return;
        Staged st(h, dev_buf, (size_t)ls.rows * width * es, dtype & GMD_HOST_MEMORY, true);
        ensure_api_plan(h, ls, h->corrupted && !bonds);
        const int ww = width * es / 4;
        k_copy_rows<<<div_up(ls.nfrom * ww, 256), 256, 0, h->stream>>>(
            ls.nfrom, ls.xdst.as<int32_t>(), ls.xapi.as<int32_t>(), static_cast<uint32_t*>(st.dev),
            ww);
        GMD_LAUNCH_CHECK();
        st.copy_out();
        sync(h);
    });
}

int gmd_transfer_transpose(gmd_handle* h, int bonds, void* dev_buf, int width, int dtype) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        const int es = elem_size(dtype);
        if (width < 1) raise(kArg, "width must be >= 1");
        cudaStream_t s = h->stream;
        Staged st(h, dev_buf, (size_t)ls.rows * width * es, dtype & GMD_HOST_MEMORY, true);
        dev_buf = st.dev;
        if (ls.nfrom > 0) {
            ensure_api_plan(h, ls, false);
            const int64_t tot = ls.nfrom * width;
            if (es == 8)
                k_transpose_add<double><<<div_up(tot, 256), 256, 0, s>>>(
                    ls.nfrom, ls.xapi.as<int32_t>(), ls.xdst.as<int32_t>(),
                    static_cast<double*>(dev_buf), width);
            else
                k_transpose_add<float><<<div_up(tot, 256), 256, 0, s>>>(
                    ls.nfrom, ls.xapi.as<int32_t>(), ls.xdst.as<int32_t>(),
                    static_cast<float*>(dev_buf), width);
            GMD_LAUNCH_CHECK();
        }
        ensure_dup_groups(h, ls);
        if (ls.ngroups > 0) {
            const int64_t tot = ls.ngroups * width;
            if (es == 8)
                k_dup_fold<double><<<div_up(tot, 256), 256, 0, s>>>(
                    ls.ngroups, ls.g_canon.as<int32_t>(), ls.g_start.as<int32_t>(),
                    ls.g_dups.as<int32_t>(), static_cast<double*>(dev_buf), width);
            else
                k_dup_fold<float><<<div_up(tot, 256), 256, 0, s>>>(
                    ls.ngroups, ls.g_canon.as<int32_t>(), ls.g_start.as<int32_t>(),
                    ls.g_dups.as<int32_t>(), static_cast<float*>(dev_buf), width);
            GMD_LAUNCH_CHECK();
        }
        st.copy_out();
        sync(h);
    });
}

int gmd_sync_duplicates(gmd_handle* h, int bonds, void* dev_buf, int width, int dtype) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        const int es = elem_size(dtype);
        ensure_dup_groups(h, ls);
        if (ls.ndups == 0) return;
        Staged st(h, dev_buf, (size_t)ls.rows * width * es, dtype & GMD_HOST_MEMORY, true);
        const int ww = width * es / 4;
        k_copy_rows<<<div_up(ls.ndups * ww, 256), 256, 0, h->stream>>>(
            ls.ndups, ls.d_dup.as<int32_t>(), ls.d_canon.as<int32_t>(),
            static_cast<uint32_t*>(st.dev), ww);
        GMD_LAUNCH_CHECK();
        st.copy_out();
        sync(h);
    });
}

int gmd_distribute(gmd_handle* h, int bonds, const void* host_global, void* dev_buf, int width,
                   int dtype) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        const int es = elem_size(dtype);
        const int ww = width * es / 4;
        cudaStream_t s = h->stream;
        uint32_t* tmp = h->conv_tmp.get<uint32_t>((size_t)ls.nid * ww);
        GMD_CUDA(cudaMemcpyAsync(tmp, host_global, (size_t)ls.nid * ww * 4, cudaMemcpyHostToDevice,
                                 s));
        Staged st(h, dev_buf, (size_t)ls.rows * ww * 4, dtype & GMD_HOST_MEMORY, false);
        if (ls.rows > 0) {
            k_gather_rows<<<div_up(ls.rows * ww, 256), 256, 0, s>>>(
                ls.rows, ls.p > 1 ? ls.node_array.as<int32_t>() : nullptr, tmp,
                static_cast<uint32_t*>(st.dev), ww);
            GMD_LAUNCH_CHECK();
        }
        st.copy_out();
        sync(h);
    });
}

int gmd_aggregate(gmd_handle* h, int bonds, const void* dev_buf, void* host_global, int width,
                  int dtype) {
    return run(h, [&] {
        LayoutState& ls = layout_of(h, bonds);
        const int es = elem_size(dtype);
        const int ww = width * es / 4;
        cudaStream_t s = h->stream;
        uint32_t* tmp = h->conv_tmp.get<uint32_t>((size_t)ls.nid * ww);
        Staged st(h, const_cast<void*>(dev_buf), (size_t)ls.rows * ww * 4, dtype & GMD_HOST_MEMORY, true);
        if (ls.nid > 0) {  // canonical owned row of every id (engine.cpp:214-229)
            k_gather_rows<<<div_up(ls.nid * ww, 256), 256, 0, s>>>(
                ls.nid, ls.p > 1 ? ls.crow.as<int32_t>() : nullptr,
                static_cast<const uint32_t*>(st.dev), tmp, ww);
            GMD_LAUNCH_CHECK();
        }
        GMD_CUDA(cudaMemcpyAsync(host_global, tmp, (size_t)ls.nid * ww * 4, cudaMemcpyDeviceToHost,
                                 s));
        sync(h);
    });
}

int gmd_corrupt_transfer_plan_for_test(gmd_handle* h) {
    return run(h, [&] {
        need_built(h);
        h->corrupted = true;
    });
}

int gmd_comm_nccl_id(uint8_t id[128]) {
    if (!id) return GMD_ERR_ARG;
    std::string err;
    if (!nccl_unique_id(id, &err)) {
        g_err = err;
        return GMD_ERR_CUDA;
    }
    return GMD_OK;
}

int gmd_comm_init_nccl(gmd_handle* h, int rank, int world, const uint8_t id[128]) {
    return run(h, [&] {
        if (!id || world < 1 || rank < 0 || rank >= world) raise(kArg, "bad rank/world");
        h->comm.reset(make_nccl_transport(rank, world, id, h->device));
        h->built = false;
    });
}

int gmd_comm_ipc_export(gmd_handle* h, int rank, int world, int64_t slot_rows,
                        uint8_t handle[64]) {
    return run(h, [&] {
        if (!handle || world < 1 || rank < 0 || rank >= world || slot_rows < 1)
            raise(kArg, "bad rank/world/slot_rows");
        if (h->ipc_window) cudaFree(h->ipc_window);
        h->ipc_window = ipc_window_create(world, slot_rows, handle);
        h->ipc_rank = rank;
        h->ipc_world = world;
        h->ipc_rows = slot_rows;
    });
}

int gmd_comm_init_ipc(gmd_handle* h, const uint8_t* handles) {
    return run(h, [&] {
        if (!handles || !h->ipc_window) raise(kArg, "gmd_comm_ipc_export first");
        h->comm.reset(make_ipc_transport(h->ipc_rank, h->ipc_world, h->device, h->ipc_rows,
                                         h->ipc_window, handles));
        h->ipc_window = nullptr;  // owned by the transport now
        h->built = false;
    });
}

int gmd_comm_init_local(gmd_handle** hs, int world) {
    if (!hs || world < 1) return GMD_ERR_ARG;
    for (int r = 0; r < world; ++r)
        if (!hs[r]) return GMD_ERR_ARG;
    LocalGroup* g = local_group_create(world);
    for (int r = 0; r < world; ++r) {
        hs[r]->comm.reset(make_local_transport(g, r));
        hs[r]->built = false;
    }
    return GMD_OK;
}

int gmd_comm_info(const gmd_handle* h, int* rank, int* world) {
    if (!h) return GMD_ERR_ARG;
    if (rank) *rank = h->comm ? h->comm->rank : 0;
    if (world) *world = h->comm ? h->comm->world : 1;
    return GMD_OK;
}

int gmd_num_owned(const gmd_handle* h, int64_t* n) {
    if (!h || !n) return GMD_ERR_ARG;
    *n = h->built ? (h->comm && h->comm->world > 1 ? h->n_own : h->n) : 0;
    return GMD_OK;
}

int gmd_num_interior(const gmd_handle* h, int64_t* n) {
    if (!h || !n) return GMD_ERR_ARG;
    *n = h->built && h->comm && h->comm->world > 1 ? h->n_int : 0;
    return GMD_OK;
}

int gmd_get_owned_ids(gmd_handle* h, int64_t* ids) {
    return run(h, [&] {
        need_built(h);
        if (h->comm && h->comm->world > 1) {
            std::vector<int32_t> v;
            d2h(h, v, h->nodes.as<int32_t>(), h->n_own);
            sync(h);
            std::copy(v.begin(), v.end(), ids);
        } else {
            for (int64_t i = 0; i < h->n; ++i) ids[i] = i;
        }
    });
}

// ---- on-device MD (md.cpp:20-160) ------------------------------------------
// standard atomic weights up to Xe, linear estimate beyond (system.cpp:28-37,
// :289-293)
static const double kMassTable[55] = {
    0.0,    1.008,  4.0026, 6.94,   9.0122, 10.81,  12.011, 14.007, 15.999, 18.998, 20.180,
    22.990, 24.305, 26.982, 28.085, 30.974, 32.06,  35.45,  39.948, 39.098, 40.078, 44.956,
    47.867, 50.942, 51.996, 54.938, 55.845, 58.933, 58.693, 63.546, 65.38,  69.723, 72.630,
    74.922, 78.971, 79.904, 83.798, 85.468, 87.62,  88.906, 91.224, 92.906, 95.95,  97.0,
    101.07, 102.91, 106.42, 107.87, 112.41, 114.82, 118.71, 121.76, 127.60, 126.90, 131.29};

int gmd_md_masses(int64_t n, const int32_t* Z, double* masses) {
    if ((n > 0 && (!Z || !masses)) || n < 0) return GMD_ERR_ARG;
    for (int64_t i = 0; i < n; ++i) {
        const int z = Z[i];
        if (z < 1 || z > 118) {
            g_err = "atomic number out of range";
            return GMD_ERR_CONFIG;
        }
        masses[i] = z < 55 ? kMassTable[z] : 2.5 * z;
    }
    return GMD_OK;
}

int gmd_md_maxwell_boltzmann(int64_t n, const int32_t* Z, double temperature, uint64_t seed,
                             double* vel) {
    if ((n > 0 && (!Z || !vel)) || n < 0) return GMD_ERR_ARG;
    std::fill(vel, vel + 3 * n, 0.0);
    if (temperature <= 0.0 || n == 0) return GMD_OK;
    std::vector<double> m(n);
    if (int rc = gmd_md_masses(n, Z, m.data())) return rc;
    HostRng rng(seed ^ 0xd1b54a32d192ed03ull);  // md.cpp:28
    for (int64_t i = 0; i < n; ++i) {
        const double sigma = std::sqrt(gmd::kBoltzmann * temperature / (m[i] * gmd::kKinetic));
        for (int k = 0; k < 3; ++k) vel[3 * i + k] = sigma * rng.normal();
    }
    double p[3] = {0.0, 0.0, 0.0}, mtot = 0.0;  // remove the centre-of-mass momentum
    for (int64_t i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) p[k] += vel[3 * i + k] * m[i];
        mtot += m[i];
    }
    const double vcm[3] = {p[0] / mtot, p[1] / mtot, p[2] / mtot};
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) vel[3 * i + k] -= vcm[k];
    return GMD_OK;
}

int gmd_md_evaluate(gmd_handle* h, int64_t n, const double* pos, const int32_t* Z,
                    const double lattice[9], const uint8_t pbc[3], double rc, double r3, double tau,
                    int p, uint32_t flags, double* forces, double* energy, double* timing) {
    return run(h, [&] {
        if (!pos || !Z || !lattice || !forces) raise(kArg, "null pointer");
        build_impl(h, n, pos, Z, lattice, pbc, rc, r3, tau, p, flags | GMD_INPUT_DEVICE);
        forward_impl(h, energy, nullptr, forces, nullptr, timing, GMD_OUTPUT_DEVICE);
    });
}

int gmd_md_step(gmd_handle* h, int64_t n, double* pos, double* vel, double* forces,
                const double* masses, const int32_t* Z, const double lattice[9],
                const uint8_t pbc[3], double dt, double rc, double r3, double tau, int p,
                uint32_t flags, double* energy, double* timing) {
    return run(h, [&] {
        if (!pos || !vel || !forces || !masses || !Z || !lattice) raise(kArg, "null pointer");
        if (dt < 0.0) raise(kConfig, "time step must be >= 0");
        if (h->comm && h->comm->world > 1)
            raise(kConfig, "gmd_md_step integrates all atoms on one handle (rank groups: "
                           "gather forces with gmd_md_evaluate on each rank)");
        cudaStream_t s = h->stream;
        Mat9 L, inv;
        for (int k = 0; k < 9; ++k) L.m[k] = lattice[k];
        inverse3(lattice, inv.m);
        launch_md_kick_drift(n, pos, vel, forces, masses, dt, s);
        launch_md_wrap(n, pos, L, inv, s);
        build_impl(h, n, pos, Z, lattice, pbc, rc, r3, tau, p, flags | GMD_INPUT_DEVICE);
        forward_impl(h, energy, nullptr, forces, nullptr, timing, GMD_OUTPUT_DEVICE);
        auto* bad = h->md_bad.get<unsigned long long>(1);
        GMD_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
        launch_md_kick(n, vel, forces, masses, dt, bad, s);
        unsigned long long hb = 0;
        GMD_CUDA(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, s));
        GMD_CUDA(cudaStreamSynchronize(s));
        if (hb != ~0ull) raise(kRuntime, "non-finite force on atom " + std::to_string(hb));
    });
}

int gmd_md_observe(gmd_handle* h, int64_t n, const double* vel, const double* masses,
                   const double* forces, double* kinetic, double* max_force) {
    return run(h, [&] {
        if (!vel || !masses) raise(kArg, "null pointer");
        cudaStream_t s = h->stream;
        double* part = h->md_part.get<double>(2 * (size_t)md_observe_parts());
        double* out = h->md_out.get<double>(2);
        launch_md_observe(n, vel, masses, forces, part, out, s);
        double ho[2];
        GMD_CUDA(cudaMemcpyAsync(ho, out, sizeof ho, cudaMemcpyDeviceToHost, s));
        GMD_CUDA(cudaStreamSynchronize(s));
        if (kinetic) *kinetic = ho[0];
        if (max_force) *max_force = ho[1];
    });
}

int gmd_md_run(gmd_handle* h, int64_t n, double* pos, double* vel, double* forces,
               const int32_t* Z, const double lattice[9], const uint8_t pbc[3], double dt,
               int64_t steps, double rc, double r3, double tau, int p, uint32_t flags,
               double* records) {
    if (!h || !pos || !vel || !Z || !lattice || n < 0 || steps < 0) return GMD_ERR_ARG;
    std::vector<double> m(n);
    if (int rc0 = gmd_md_masses(n, Z, m.data())) {
        h->err = g_err;
        return rc0;
    }
    double *dp = nullptr, *dv = nullptr, *df = nullptr, *dm = nullptr;
    int32_t* dz = nullptr;
    int rc1 = run(h, [&] {
        cudaStream_t s = h->stream;
        dp = h->md_pos.get<double>(3 * n);
        dv = h->md_vel.get<double>(3 * n);
        df = h->md_frc.get<double>(3 * n);
        dm = h->md_mass.get<double>(n);
        dz = h->md_z.get<int32_t>(n);
        GMD_CUDA(cudaMemcpyAsync(dp, pos, 24 * n, cudaMemcpyHostToDevice, s));
        GMD_CUDA(cudaMemcpyAsync(dv, vel, 24 * n, cudaMemcpyHostToDevice, s));
        GMD_CUDA(cudaMemcpyAsync(dm, m.data(), 8 * n, cudaMemcpyHostToDevice, s));
        GMD_CUDA(cudaMemcpyAsync(dz, Z, 4 * n, cudaMemcpyHostToDevice, s));
    });
    if (rc1) return rc1;
    auto rec = [&](int64_t step, double pot, const double* tm) -> int {
        double ke = 0.0, fm = 0.0;
        if (int r = gmd_md_observe(h, n, dv, dm, df, &ke, &fm)) return r;
        if (records) {
            double* r = records + 8 * step;
            r[0] = pot;
            r[1] = ke;
            r[2] = pot + ke;
            r[3] = fm;
            for (int k = 0; k < 4; ++k) r[4 + k] = tm[k];
        }
        return GMD_OK;
    };
    double pot = 0.0, tm[4] = {0, 0, 0, 0};
    if (int r = gmd_md_evaluate(h, n, dp, dz, lattice, pbc, rc, r3, tau, p, flags, df, &pot, tm))
        return r;
    if (int r = rec(0, pot, tm)) return r;
    for (int64_t step = 1; step <= steps; ++step) {
        if (int r = gmd_md_step(h, n, dp, dv, df, dm, dz, lattice, pbc, dt, rc, r3, tau, p, flags,
                                &pot, tm)) {
            if (h->err.rfind("non-finite force", 0) == 0)
                h->err += " at step " + std::to_string(step);
            return r;
        }
        if (int r = rec(step, pot, tm)) return r;
    }
    return run(h, [&] {
        cudaStream_t s = h->stream;
        GMD_CUDA(cudaMemcpyAsync(pos, dp, 24 * n, cudaMemcpyDeviceToHost, s));
        GMD_CUDA(cudaMemcpyAsync(vel, dv, 24 * n, cudaMemcpyDeviceToHost, s));
        if (forces) GMD_CUDA(cudaMemcpyAsync(forces, df, 24 * n, cudaMemcpyDeviceToHost, s));
        GMD_CUDA(cudaStreamSynchronize(s));
    });
}

int gmd_util_rng_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out) {
    if (!out || count < 0) return GMD_ERR_ARG;
    HostRng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * r.uniform();
    return GMD_OK;
}

int gmd_util_supercell(int64_t n, const double* pos, const int32_t* Z, const double lattice[9],
                       int rx, int ry, int rz, double amp, uint64_t seed, double* out_pos,
                       int32_t* out_Z, double* out_lattice) {
    if (!pos || !Z || !lattice || !out_pos || !out_Z || !out_lattice) return GMD_ERR_ARG;
    if (rx < 1 || ry < 1 || rz < 1) return GMD_ERR_CONFIG;
    const int reps[3] = {rx, ry, rz};
    for (int k = 0; k < 3; ++k) {  // make_supercell (system.cpp:188-214)
        V3 r = vmul(row3(lattice, k), (double)reps[k]);
        out_lattice[3 * k] = r.x;
        out_lattice[3 * k + 1] = r.y;
        out_lattice[3 * k + 2] = r.z;
    }
    int64_t o = 0;
    for (int a = 0; a < rx; ++a)
        for (int b = 0; b < ry; ++b)
            for (int c = 0; c < rz; ++c) {
                V3 l0 = vmul(row3(lattice, 0), a), l1 = vmul(row3(lattice, 1), b),
                   l2 = vmul(row3(lattice, 2), c);
                V3 sh = {l0.x + l1.x + l2.x, l0.y + l1.y + l2.y, l0.z + l1.z + l2.z};
                for (int64_t i = 0; i < n; ++i, ++o) {
                    out_pos[3 * o] = pos[3 * i] + sh.x;
                    out_pos[3 * o + 1] = pos[3 * i + 1] + sh.y;
                    out_pos[3 * o + 2] = pos[3 * i + 2] + sh.z;
                    out_Z[o] = Z[i];
                }
            }
    if (amp > 0.0) {  // random_perturb (system.cpp:231-240)
        HostRng r(seed);
        for (int64_t i = 0; i < o; ++i)
            for (int k = 0; k < 3; ++k) out_pos[3 * i + k] += -amp + (amp - -amp) * r.uniform();
    } else if (amp < 0.0) {
        return GMD_ERR_CONFIG;
    }
    return GMD_OK;
}

int gmd_profile(gmd_handle* h, int enable) {
    return run(h, [&] {
        h->prof = enable != 0;
        h->pidx = 0;
        h->precs.clear();
        if (h->prof && h->pev.empty()) {
            h->pev.resize(16384);
            for (auto& e : h->pev) GMD_CUDA(cudaEventCreate(&e));
        }
    });
}

int gmd_profile_read(gmd_handle* h, char* names, int names_cap, double* total_ms, int* launches,
                     int* count) {
    return run(h, [&] {
        if (!count) raise(kArg, "null count");
        sync(h);
        std::vector<std::string> order;
        std::unordered_map<std::string, std::pair<double, int>> acc;
        for (auto& r : h->precs) {
            float ms = 0.f;
            GMD_CUDA(cudaEventElapsedTime(&ms, h->pev[r.second], h->pev[r.second + 1]));
            auto it = acc.find(r.first);
            if (it == acc.end()) {
                order.push_back(r.first);
                acc[r.first] = {ms, 1};
            } else {
                it->second.first += ms;
                it->second.second += 1;
            }
        }
        const int cap = *count;
        int k = 0, pos = 0;
        for (const auto& nm : order) {
            if (k >= cap || pos + (int)nm.size() + 1 > names_cap) break;
            std::memcpy(names + pos, nm.c_str(), nm.size() + 1);
            pos += (int)nm.size() + 1;
            total_ms[k] = acc[nm].first;
            launches[k] = acc[nm].second;
            ++k;
        }
        *count = k;
    });
}

int gmd_launch_count(int64_t* count) {
    if (!count) return GMD_ERR_ARG;
    *count = __atomic_load_n(&g_gmd_launches, __ATOMIC_RELAXED);
    return GMD_OK;
}

int gmd_get_stream(gmd_handle* h, void** stream) {
    if (!h || !stream) return GMD_ERR_ARG;
    *stream = (void*)h->stream;
    return GMD_OK;
}

}  // extern "C"
