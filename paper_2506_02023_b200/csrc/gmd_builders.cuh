// Device side of the reference's free builder API (partitioner.hpp:66-106,
// linegraph.hpp:26-78, neighborlist.hpp:40-42) on a caller-supplied graph:
// the partition / bond / line-graph kernels of gmd_build run unchanged once
// these kernels have put the caller's edges into the handle's CSR form.
#pragma once
#include "gmd_common.cuh"

namespace gmd {

// caller's canonical (dst-major) edge list -> CSR pieces: packed images (the
// reverse-bond search keys) and three-body bond flags d <= bound with
// per-destination bond counts; kErrImgRange in flags[1] when an offset does
// not fit the packed range
void launch_graph_import(int64_t ne, const int32_t* off3, const double* dist, double bond_bound,
                         uint32_t* img, uint8_t* ebond, int32_t* flags, cudaStream_t s);
void launch_row_bond_count(const int32_t* row, const uint8_t* ebond, int64_t n, int32_t* bcnt,
                           cudaStream_t s);

// two-hop closure (linegraph.cpp:45-65) of all partitions at once: a u64
// partition mask per node, mask'[v] = mask[v] | OR_{e into v} mask[src e]
void launch_closure_init(const int32_t* owner, int64_t n, unsigned long long* mask,
                         cudaStream_t s);
void launch_closure_hop(const int32_t* row, const int32_t* src, int64_t n,
                        const unsigned long long* in, unsigned long long* out, cudaStream_t s);
// edge-table membership (linegraph.cpp:84-93): bond b is in partition i's
// table iff both endpoints of its edge are in closure i
void launch_bond_tables(int64_t nb, const int32_t* bedge, const int32_t* edst,
                        const int32_t* src, const unsigned long long* mask,
                        unsigned long long* bmask, cudaStream_t s);

// brute-force radius graph (neighborlist.cpp:199-239): one warp per
// destination atom, lanes over sources, every image in the span; the
// reference's exact fp64 expressions.  Pass 1 (out == nullptr) counts per
// destination, pass 2 writes (src, ox, oy, oz) at row offsets (unsorted
// within a row; the caller sorts rows into canonical order).
struct BruteNL {
    double L[9];
    double cutoff2;
    int span[3];
};
void launch_brute_nl(const BruteNL& b, int64_t n, const double* pos, const int32_t* cell,
                     int32_t* cnt, const int32_t* rowoff, int32_t* out_src, int32_t* out_off,
                     cudaStream_t s);
// exact fp64 distance and vector of edges (src, dst, off) (neighborlist.cpp:184-191)
void launch_edge_geometry(const BruteNL& b, int64_t ne, const double* pos, const int32_t* src,
                          const int32_t* dst, const int32_t* off, double* dist, double* vec,
                          cudaStream_t s);

// brute-force line graph (linegraph.cpp:201-219): per center u every
// (in-bond e, out-bond e') pair that is not a reverse pair; pass 1 counts
// per center, pass 2 writes (edge e, edge e') pairs at the center's offset
void launch_brute_line(int64_t n, const int32_t* in_row, const int32_t* in_bonds,
                       const int32_t* out_row, const int32_t* out_bonds, const int32_t* bedge,
                       const int32_t* src, const int32_t* edst, const uint32_t* img, int32_t* cnt,
                       const int32_t* off, int32_t* pairs, cudaStream_t s);

}  // namespace gmd
