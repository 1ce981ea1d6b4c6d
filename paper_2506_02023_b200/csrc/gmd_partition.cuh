// Slab partitioning with halo (border-node) sets on the GPU (north_star 2).
// Replaces choose_partition_rule / assign_to_partitions / build_span_layout /
// build_atom_partitions (proj/src/partitioner.cpp:46-218).
#pragma once
#include "gmd_common.cuh"

namespace gmd {

// Radix select (8-bit MSD digits) of the given ascending ranks from n
// non-negative doubles viewed as u64 keys.  out[k] = the rank[k]-th smallest.
// All state lives in `ws` (see select_ws_bytes); results land in out (device).
size_t select_ws_bytes(int nranks);
void launch_select(const double* keys, int64_t n, const int64_t* ranks_host, int nranks,
                   void* ws, double* out_dev, cudaStream_t s);

struct Bounds {
    double b[kMaxParts + 1];
    int p;
};

void launch_owner(const double* fw_axis, int64_t n, const Bounds& bd, int32_t* owner,
                  cudaStream_t s);
// req[src] |= 1 << owner[dst] for every edge crossing partitions
// (partitioner.cpp:124-134); req must be zeroed by the caller.
void launch_required(const int32_t* row, const int32_t* src, int64_t n, const int32_t* owner,
                     unsigned long long* req, cudaStream_t s);

// Stable multi-list compaction that lays out [PURE | TO_0..TO_p-1 |
// FROM_0..FROM_p-1] for every partition of an id space (atoms or bonds).
// List id of (partition i, block b) = i*(1+2p) + b.  Produces:
//   node_array (concatenated over partitions, "super rows"),
//   crow[id]   = canonical super row of id in its owner partition
//                (first occurrence, partitioner.cpp:163-164),
//   list_off   = start of every list in the super array (nlists + 1).
struct LayoutWs {
    int32_t* counts;     // nlists * nchunks (+1) scan buffer
    void* scan_tmp;
    size_t scan_tmp_bytes;
};
int64_t layout_chunks(int64_t nid);
int64_t layout_nlists(int p);
// plan: per-(list, chunk) counts, their scan, and list_off (nlists + 1
// entries, last = total super rows).  fill: node_array + crow.
// only >= 0 restricts the layout to partition `only` (one rank per GPU).
void launch_layout_plan(const int32_t* owner, const unsigned long long* req, int64_t nid, int p,
                        LayoutWs& ws, int32_t* list_off, int only, cudaStream_t s);
void launch_layout_fill(const int32_t* owner, const unsigned long long* req, int64_t nid, int p,
                        LayoutWs& ws, int32_t* node_array, int32_t* crow, int only,
                        cudaStream_t s);

// one rank per GPU (rank r of p): requirement masks from r's own rows,
// the ascending list of r's atoms, and the send plan of its TO rows
void launch_required_rank(const int32_t* row, const int32_t* src, int64_t n, const int32_t* owner,
                          int r, unsigned long long* req, cudaStream_t s);
void launch_owned_flags(const int32_t* owner, int64_t n, int r, int32_t* flag, cudaStream_t s);
void launch_owned_compact(const int32_t* owner, int64_t n, int r, const int32_t* pos,
                          int32_t* nodes, cudaStream_t s);
// interior / border split of r's atoms (flag[k] = 1: no in-edge from a peer's
// atom; out = interior ascending, then border ascending; pos = scan of flag)
void launch_flag_interior(int64_t n_own, const int32_t* nodes, const int32_t* row, const int32_t* src,
                          const int32_t* owner, int r, int32_t* flag, cudaStream_t s);
void launch_split_nodes(int64_t n_own, const int32_t* nodes, const int32_t* pos, int32_t* out,
                        cudaStream_t s);
void launch_send_rows(int32_t t0, int32_t t1, const int32_t* node_array, const int32_t* crow,
                      int32_t* xsend, cudaStream_t s);

// Exchange plan: for every FROM super row, the canonical super row of the
// same id in its owner partition.  from_ranges[i] = (begin, end) super rows.
void launch_from_src(const int32_t* node_array, const int32_t* crow, const int32_t* from_ranges,
                     int p, int64_t nfrom_total, const int32_t* from_prefix, int32_t* xdst,
                     int32_t* xsrc, cudaStream_t s);

// Per-edge source super row in the owner partition of the edge's dst:
// crow[src] when the source is owned there, else its row in the FROM block
// (partitioner.cpp:200-216, local_of through global_to_local).
void launch_edge_lsrc(const int32_t* row, const int32_t* src, int64_t n, const int32_t* owner,
                      const int32_t* crow, const int32_t* node_array, const int32_t* list_off,
                      int p, int32_t* lsrc, int32_t* flags, cudaStream_t s);

}  // namespace gmd
