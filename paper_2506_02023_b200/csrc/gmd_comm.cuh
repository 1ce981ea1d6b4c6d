// Halo-exchange transports for one-rank-per-GPU execution.
//
// The reference exchanges TO_j[i] -> FROM_i[j] spans by memcpy between
// in-process blocks (engine.cpp:122-143).  Here every rank owns one slab;
// before each layer it packs the canonical rows of its TO_r[j] blocks into a
// send buffer (one contiguous run per peer) and receives peer j's run straight
// into its FROM_r[j] span (rows are in ascending global id on both sides, so
// no unpack is needed).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "gmd_common.cuh"

namespace gmd {

struct Transport {
    int rank = 0, world = 1;
    virtual ~Transport() = default;
    virtual const char* name() const = 0;
    // send: rows packed per peer at soff[j] (scnt[j] rows); recv: peer j's
    // rows land at recv + roff[j] * width (rcnt[j] rows).  Offsets in rows.
    virtual void exchange(cudaStream_t s, const float* send, const int64_t* soff,
                          const int64_t* scnt, float* recv, const int64_t* roff,
                          const int64_t* rcnt, int width) = 0;
    // the same exchange with the send rows gathered by the transport from
    // src rows sidx[soff[j] ..) (no separate packing pass); transports that
    // cannot fuse it pack into `scratch` and call exchange
    virtual bool fused_gather() const { return false; }
    virtual void exchange_gather(cudaStream_t s, const float* src, const int32_t* sidx,
                                 const int64_t* soff, const int64_t* scnt, float* recv,
                                 const int64_t* roff, const int64_t* rcnt, int width) {
        (void)s, (void)src, (void)sidx, (void)soff, (void)scnt, (void)recv, (void)roff, (void)rcnt,
            (void)width;
    }
    // split form of exchange_gather: begin issues the sends, end completes the
    // receives; stream work between them that does not touch recv's halo rows
    // (interior atoms) overlaps the transfer.  Transports without a split do
    // the whole exchange in begin.
    virtual void exchange_gather_begin(cudaStream_t s, const float* src, const int32_t* sidx,
                                       const int64_t* soff, const int64_t* scnt, float* recv,
                                       const int64_t* roff, const int64_t* rcnt, int width) {
        exchange_gather(s, src, sidx, soff, scnt, recv, roff, rcnt, width);
    }
    virtual void exchange_gather_end(cudaStream_t s) { (void)s; }
    // rank-ordered all-gathers of small host vectors (out: world * n)
    virtual void allgather_f64(cudaStream_t s, const double* in, int n, double* out) = 0;
    virtual void allgather_i64(cudaStream_t s, const int64_t* in, int n, int64_t* out) = 0;
};

// in-process group: W handles (same or different GPUs) exchanging through
// device-to-device copies; each handle must be driven by its own host thread
struct LocalGroup;
LocalGroup* local_group_create(int world);
void local_group_release(LocalGroup* g);  // refcounted; the last rank frees it
Transport* make_local_transport(LocalGroup* g, int rank);

// NCCL (libnccl.so.2 loaded at run time; torch's bundled copy when present)
bool nccl_unique_id(unsigned char id[128], std::string* err);
Transport* make_nccl_transport(int rank, int world, const unsigned char id[128], int device);

// CUDA-IPC peer transport for ranks on one node (P2P stores over NVLink):
// ipc_window_create allocates this rank's window and returns its IPC handle;
// after all ranks exchanged handles, make_ipc_transport maps the peers'.
size_t ipc_window_bytes(int world, int64_t slot_rows);
void* ipc_window_create(int world, int64_t slot_rows, unsigned char handle[64]);
Transport* make_ipc_transport(int rank, int world, int device, int64_t slot_rows, void* window,
                              const unsigned char* handles /* world x 64 bytes */);

}  // namespace gmd
