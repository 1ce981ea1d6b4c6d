// Periodic radius graph on the GPU (north_star 1).  Replaces
// build_neighbor_list (proj/src/neighborlist.cpp:108-197) with a cell-list
// search whose fp64 decisions are bit-identical to the reference.
#pragma once
#include "gmd_common.cuh"

namespace gmd {

// Scalar geometry computed on the host with the reference's operand order
// (system.cpp:55-93, neighborlist.cpp:119-126).
struct Geom {
    double L[9];     // lattice rows (after ensure_periodic)
    double inv[9];   // Mat3::inverse rows
    int bins[3];     // max(1, floor(width_k / rc))
    int sten[3];     // floor(rc / bin_width_k) + 1
    double cutoff2;  // rc * rc
    double pre2;     // rc * rc * 1.000001 (prefilter, neighborlist.cpp:177)
    double bond_bound;  // r3 + tau, < 0 when no three-body graph is needed
    int axis;        // partition axis (longest lattice row)
};

// Device arrays of the built graph (canonical dst-major CSR).
struct GraphDev {
    int64_t n = 0, ne = 0;
    int32_t* row = nullptr;    // n + 1
    int32_t* src = nullptr;    // ne, global source id
    uint32_t* img = nullptr;   // ne, packed image offset
    float4* vd = nullptr;      // ne, (vx, vy, vz, d) rounded from fp64
    float* d = nullptr;        // ne, d (the forward pass reads only this)
    uint8_t* bond = nullptr;   // ne, 1 iff d <= r3 + tau (three-body bond)
};

struct NLBuffers {
    // atom-indexed
    double* pos;       // n x 3 AoS (input, raw Cartesian)
    int32_t* cell;     // n x 3 AoS, floor of fractional coords (neighborlist.cpp:43-49)
    double* fw_axis;   // n, wrapped fractional coordinate along the partition axis
    int32_t* bin;      // n
    // bin-sorted copies
    int32_t* bin_cnt;    // nbins (scratch)
    int32_t* bin_start;  // nbins + 1
    int32_t* s_id;       // n
    double* s_w;         // 3 x n SoA: wrapped Cartesian
    double* s_p;         // 3 x n SoA: raw Cartesian
    int32_t* s_c;        // 3 x n SoA: cell_of
    int32_t* deg;        // n (per-dst degree)
    int32_t* bcnt;       // n (per-dst bond count)
    int32_t* flags;      // [0] max degree, [1] error bits, [2] max in-bonds,
                         // [3] max |input coordinate| (fp32 bits, k_wrap)
    // optional 32-byte / 16-byte per-atom records (raw position, cell_of)
    // written by k_wrap: the emit gathers an edge's source with two vector
    // loads instead of six scalar ones (required by launch_nl_emit)
    double4* pos4 = nullptr;
    int4* cell4 = nullptr;
};

enum : int { kErrImgRange = 1, kErrQRange = 2, kErrCap = 4 };

void launch_wrap(const Geom& g, int64_t n, NLBuffers& b, cudaStream_t s);
void launch_bin_scatter(const Geom& g, int64_t n, NLBuffers& b, int32_t* fill, cudaStream_t s);
// search: per-destination sorted (src, image) keys into slab[n x cap], stored
// row lengths min(degree, cap) into deg, the true max degree into flags[0]
// (slab rows truncated at cap; a build whose max exceeds cap is redone)
// only >= 0: rows only for destination atoms with owner[i] == only (the
// other rows stay empty; deg must be zeroed by the caller)
// pos_gate: the fast-accept band is disabled on the device when any input
// coordinate exceeds it (wrapped vs raw vectors could then differ by more
// than the band's margin)
void launch_nl_search(const Geom& g, float thr32, float acc32, float zero32, float pos_gate,
                      int64_t nbins, int64_t n, int cap,
                      NLBuffers& b, unsigned long long* slab, const int32_t* owner, int only,
                      cudaStream_t s);
// emit: slab rows -> CSR (row must hold the scanned degrees)
// owner / req (optional): requirement masks of p > 1 partitions in one
// process, OR-ed in from the emitted edges (replaces launch_required)
void launch_nl_emit(const Geom& g, int64_t n, int cap, const unsigned long long* slab,
                    NLBuffers& b, GraphDev& gd, cudaStream_t s, const int32_t* owner = nullptr,
                    unsigned long long* req = nullptr);
void launch_minmax_proj(const double* pos, int64_t n, const double dir[3], double* out2,
                        cudaStream_t s);
void launch_shift(double* pos, int64_t n, const double add[3], cudaStream_t s);
// canonical fp64 export: src/dst int64, off int32x3, dist, vec (exact recompute)
void launch_export_graph(const Geom& g, const double* pos, const GraphDev& gd,
                         const int32_t* edst, int64_t* src, int64_t* dst, int32_t* off,
                         double* dist, double* vec, cudaStream_t s);
// edge -> dst lookup (row expansion)
void launch_edge_dst(const int32_t* row, int64_t n, int32_t* edst, cudaStream_t s);

// bonds (three-body): bedge[brow[v]..brow[v+1]) = bond edges into v in edge
// order; brev[b] = bond id of b's reverse bond
void launch_bond_edges(const int32_t* row, const uint8_t* ebond, int64_t n, const int32_t* brow,
                       int32_t* bedge, int32_t* ebid, cudaStream_t s);
// reverse bond per bond (linegraph.cpp:16-21) via binary search in the
// reverse row + the edge -> bond id map of launch_bond_edges
void launch_bond_rev(int64_t n, const GraphDev& gd, const int32_t* brow, const int32_t* bedge,
                     const int32_t* ebid, int32_t* brev, int32_t* flags, const int32_t* owner,
                     int only, cudaStream_t s);

}  // namespace gmd
