// Halo-exchange transports (see gmd_comm.cuh).
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>

#include "gmd_comm.cuh"

namespace gmd {

// ---------------------------------------------------------------------------
// in-process group
// ---------------------------------------------------------------------------
struct LocalGroup {
    int world;
    int refs;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long generation = 0;
    std::vector<const float*> send;
    std::vector<std::vector<int64_t>> soff, scnt;
    std::vector<std::vector<double>> dbuf;
    std::vector<std::vector<int64_t>> ibuf;
    std::vector<int> bad;  // per rank: this exchange failed its plan check

    explicit LocalGroup(int w)
        : world(w), refs(w), send(w), soff(w), scnt(w), dbuf(w), ibuf(w), bad(w, 0) {}

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

LocalGroup* local_group_create(int world) { return new LocalGroup(world); }

void local_group_release(LocalGroup* g) {
    bool last;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        last = --g->refs == 0;
    }
    if (last) delete g;
}

namespace {

struct LocalTransport final : Transport {
    LocalGroup* g;
    LocalTransport(LocalGroup* grp, int r) : g(grp) {
        rank = r;
        world = grp->world;
    }
    ~LocalTransport() override { local_group_release(g); }
    const char* name() const override { return "local"; }

    void exchange(cudaStream_t s, const float* send, const int64_t* soff, const int64_t* scnt,
                  float* recv, const int64_t* roff, const int64_t* rcnt, int width) override {
        GMD_CUDA(cudaStreamSynchronize(s));  // packed rows are complete
        g->send[rank] = send;
        g->soff[rank].assign(soff, soff + world);
        g->scnt[rank].assign(scnt, scnt + world);
        g->barrier();
        // a plan mismatch is recorded, not thrown here: every rank must still
        // reach the second barrier, then all of them raise together (a rank
        // leaving early would leave its peers blocked in barrier())
        bool bad = false;
        for (int j = 0; j < world; ++j) {
            if (j == rank || rcnt[j] == 0) continue;
            if (g->scnt[j][rank] != rcnt[j]) {
                bad = true;
                continue;
            }
            GMD_CUDA(cudaMemcpyAsync(recv + roff[j] * width, g->send[j] + g->soff[j][rank] * width,
                                     sizeof(float) * rcnt[j] * width, cudaMemcpyDefault, s));
        }
        GMD_CUDA(cudaStreamSynchronize(s));
        // each rank writes only its own slot, and only after the first barrier
        // of an exchange, so the reads below never race with the next exchange
        g->bad[rank] = bad;
        g->barrier();  // peers are done reading this rank's send buffer
        if (bad) raise(kRuntime, "transfer plan misalignment");
        for (int j = 0; j < world; ++j)
            if (g->bad[j])
                raise(kRuntime, "transfer plan misalignment (detected by rank " + std::to_string(j) + ")");
    }

    void allgather_f64(cudaStream_t, const double* in, int n, double* out) override {
        g->dbuf[rank].assign(in, in + n);
        g->barrier();
        for (int j = 0; j < world; ++j) std::memcpy(out + (size_t)j * n, g->dbuf[j].data(), 8 * n);
        g->barrier();
    }
    void allgather_i64(cudaStream_t, const int64_t* in, int n, int64_t* out) override {
        g->ibuf[rank].assign(in, in + n);
        g->barrier();
        for (int j = 0; j < world; ++j) std::memcpy(out + (size_t)j * n, g->ibuf[j].data(), 8 * n);
        g->barrier();
    }
};

// ---------------------------------------------------------------------------
// NCCL, resolved at run time so the library loads where NCCL is absent
// ---------------------------------------------------------------------------
typedef int ncclResult_t_;
typedef void* ncclComm_t_;
struct NcclId {  // ncclUniqueId: passed BY VALUE to ncclCommInitRank
    char internal[128];
};
struct NcclApi {
    void* lib = nullptr;
    ncclResult_t_ (*GetUniqueId)(void*) = nullptr;
    ncclResult_t_ (*CommInitRank)(ncclComm_t_*, int, NcclId, int) = nullptr;
    ncclResult_t_ (*CommDestroy)(ncclComm_t_) = nullptr;
    ncclResult_t_ (*GroupStart)() = nullptr;
    ncclResult_t_ (*GroupEnd)() = nullptr;
    ncclResult_t_ (*Send)(const void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
    ncclResult_t_ (*Recv)(void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
    ncclResult_t_ (*AllGather)(const void*, void*, size_t, int, ncclComm_t_, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t_) = nullptr;
    std::string err;

    bool load() {
        if (lib) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names)
            if ((lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!lib) {
            err = std::string("NCCL not found: ") + dlerror();
            return false;
        }
#define GMD_SYM(f, s) f = reinterpret_cast<decltype(f)>(dlsym(lib, s))
        GMD_SYM(GetUniqueId, "ncclGetUniqueId");
        GMD_SYM(CommInitRank, "ncclCommInitRank");
        GMD_SYM(CommDestroy, "ncclCommDestroy");
        GMD_SYM(GroupStart, "ncclGroupStart");
        GMD_SYM(GroupEnd, "ncclGroupEnd");
        GMD_SYM(Send, "ncclSend");
        GMD_SYM(Recv, "ncclRecv");
        GMD_SYM(AllGather, "ncclAllGather");
        GMD_SYM(GetErrorString, "ncclGetErrorString");
#undef GMD_SYM
        if (!GetUniqueId || !CommInitRank || !Send || !Recv || !AllGather || !GroupStart ||
            !GroupEnd) {
            err = "NCCL library lacks required symbols";
            return false;
        }
        return true;
    }
};

NcclApi& nccl() {
    static NcclApi api;
    return api;
}

constexpr int kNcclInt64 = 4, kNcclFloat32 = 7, kNcclFloat64 = 8;  // ncclDataType_t

void nccl_check(int rc, const char* what) {
    if (rc != 0)
        raise(kCuda, std::string("NCCL error in ") + what + ": " +
                         (nccl().GetErrorString ? nccl().GetErrorString(rc) : "?"));
}

struct NcclTransport final : Transport {
    ncclComm_t_ comm = nullptr;
    void* dtmp = nullptr;
    size_t dcap = 0;
    NcclTransport(int r, int w, const unsigned char id[128], int device) {
        rank = r;
        world = w;
        if (!nccl().load()) raise(kCuda, nccl().err);
        GMD_CUDA(cudaSetDevice(device));
        NcclId idc;
        std::memcpy(idc.internal, id, 128);
        nccl_check(nccl().CommInitRank(&comm, w, idc, r), "ncclCommInitRank");
    }
    ~NcclTransport() override {
        if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
        if (dtmp) cudaFree(dtmp);
    }
    const char* name() const override { return "nccl"; }

    void exchange(cudaStream_t s, const float* send, const int64_t* soff, const int64_t* scnt,
                  float* recv, const int64_t* roff, const int64_t* rcnt, int width) override {
        nccl_check(nccl().GroupStart(), "ncclGroupStart");
        for (int j = 0; j < world; ++j) {
            if (j == rank) continue;
            if (scnt[j])
                nccl_check(nccl().Send(send + soff[j] * width, (size_t)scnt[j] * width, kNcclFloat32,
                                       j, comm, s), "ncclSend");
            if (rcnt[j])
                nccl_check(nccl().Recv(recv + roff[j] * width, (size_t)rcnt[j] * width, kNcclFloat32,
                                       j, comm, s), "ncclRecv");
        }
        nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    }

    void* tmp(size_t bytes) {
        if (bytes > dcap) {
            if (dtmp) cudaFree(dtmp);
            GMD_CUDA(cudaMalloc(&dtmp, bytes));
            dcap = bytes;
        }
        return dtmp;
    }
    void gather(cudaStream_t s, const void* in, size_t n, size_t es, int type, void* out) {
        char* d = static_cast<char*>(tmp(n * es * (world + 1)));
        GMD_CUDA(cudaMemcpyAsync(d, in, n * es, cudaMemcpyHostToDevice, s));
        nccl_check(nccl().AllGather(d, d + n * es, n, type, comm, s), "ncclAllGather");
        GMD_CUDA(cudaMemcpyAsync(out, d + n * es, n * es * world, cudaMemcpyDeviceToHost, s));
        GMD_CUDA(cudaStreamSynchronize(s));
    }
    void allgather_f64(cudaStream_t s, const double* in, int n, double* out) override {
        gather(s, in, n, 8, kNcclFloat64, out);
    }
    void allgather_i64(cudaStream_t s, const int64_t* in, int n, int64_t* out) override {
        gather(s, in, n, 8, kNcclInt64, out);
    }
};

// ---------------------------------------------------------------------------
// CUDA-IPC peer transport: every rank exposes one device "window" (flags,
// all-gather slots, double-buffered halo staging) through cudaIpcMemHandle_t;
// peers map it and write into it directly -- P2P stores over NVLink on a
// multi-GPU node, plain device memory when the ranks share a GPU.  Per
// exchange k (parity k & 1):
//   send kernel   : wait until peer j consumed my exchange k-2 (ack), then the
//                   packed rows for j are stored into j's staging[k&1][me]
//   signal kernel : peer_j.ready[me] = k   (release, system scope)
//   recv kernel   : wait until ready[j] >= k for every peer, then copy
//                   staging[k&1][j] -> recv + roff[j] * width
//   ack kernel    : peer_j.ack[me] = k
// All four are stream-ordered on the handle's stream; no host round trip.
// ---------------------------------------------------------------------------
constexpr int kIpcMaxWorld = 16;
constexpr size_t kIpcFlags = 4 * 64 * sizeof(long long);   // ready, ack, gready, gack
constexpr size_t kIpcGather = 64 * 32 * sizeof(double);    // all-gather slots
constexpr int kIpcGatherMax = 32;

struct IpcWin {  // views of one rank's window
    long long* ready;
    long long* ack;
    long long* gready;
    long long* gack;
    double* gather;  // [src][32]
    float* staging;  // [2][world][slot_rows * 16]
};

__host__ __device__ inline IpcWin ipc_view(void* base) {
    char* b = static_cast<char*>(base);
    IpcWin w;
    w.ready = reinterpret_cast<long long*>(b);
    w.ack = w.ready + 64;
    w.gready = w.ready + 128;
    w.gack = w.ready + 192;
    w.gather = reinterpret_cast<double*>(b + kIpcFlags);
    w.staging = reinterpret_cast<float*>(b + kIpcFlags + kIpcGather);
    return w;
}

__device__ __forceinline__ long long ld_acquire(const long long* p) {
    long long v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(long long* p, long long v) {
    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// block-wide wait until flags[idx[i]] >= v for i < n (thread 0 spins)
__device__ void wait_flags(long long* const* flags, int n, long long v) {
    if (threadIdx.x == 0)
        for (int i = 0; i < n; ++i)
            while (ld_acquire(flags[i]) < v) __nanosleep(256);
    __syncthreads();
}

struct IpcPeers {
    int n;                          // peers (world - 1)
    long long* wflag[kIpcMaxWorld];  // flag to wait on, per peer
    long long* sflag[kIpcMaxWorld];  // flag to set, per peer
    float* dst[kIpcMaxWorld];
    const float* src[kIpcMaxWorld];
    long long cnt[kIpcMaxWorld];     // floats per peer
};

__global__ void k_ipc_copy(IpcPeers P, long long wait_v) {
    if (wait_v > 0) wait_flags(P.wflag, P.n, wait_v);
    for (int j = 0; j < P.n; ++j) {
        const long long c = P.cnt[j];
        const float4* src = reinterpret_cast<const float4*>(P.src[j]);
        float4* dst = reinterpret_cast<float4*>(P.dst[j]);
        const long long c4 = c >> 2;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < c4;
             i += (long long)gridDim.x * blockDim.x)
            dst[i] = __ldcg(src + i);
        for (long long i = (c4 << 2) + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < c;
             i += (long long)gridDim.x * blockDim.x)
            P.dst[j][i] = __ldcg(P.src[j] + i);
    }
    __threadfence_system();
}

__global__ void k_ipc_signal(IpcPeers P, long long v) {
    if (threadIdx.x < P.n) st_release(P.sflag[threadIdx.x], v);
}

// one fused launch per direction: the last block to finish (fenced
// counter) publishes the flags, so pack + send + signal and receive + ack are
// one kernel each instead of five launches per exchange
struct IpcRows {
    int n;
    long long* wflag[kIpcMaxWorld];
    long long* sflag[kIpcMaxWorld];
    uint32_t* dst[kIpcMaxWorld];
    const uint32_t* src[kIpcMaxWorld];   // base of the rows
    const int32_t* idx[kIpcMaxWorld];    // row indices into src (nullptr: contiguous)
    long long rows[kIpcMaxWorld];
};

__global__ void k_ipc_rows(IpcRows P, int wwords, long long wait_v, long long sig_v,
                           unsigned int* done) {
    if (wait_v > 0) wait_flags(P.wflag, P.n, wait_v);
    for (int j = 0; j < P.n; ++j) {
        const long long tot = P.rows[j] * wwords;
        for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
             t += (long long)gridDim.x * blockDim.x) {
            const long long r = t / wwords;
            const int c = (int)(t - r * wwords);
            const long long sr = P.idx[j] ? (long long)P.idx[j][r] : r;
            P.dst[j][t] = __ldcg(P.src[j] + sr * wwords + c);
        }
    }
    __threadfence_system();  // this block's stores before its arrival
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(done, 1u) == gridDim.x - 1) {
        __threadfence_system();
        *done = 0u;  // next launch on this stream starts from zero
        for (int j = 0; j < P.n; ++j) st_release(P.sflag[j], sig_v);
    }
}

struct IpcTransport final : Transport {
    int device = 0;
    int64_t slot_rows = 0;
    void* mine = nullptr;                       // this rank's window (owned)
    std::vector<void*> peer;                    // mapped windows (peer[rank] = mine)
    long long epoch = 0, gepoch = 0;
    explicit IpcTransport(int r, int w, int dev, int64_t rows, void* win) {
        rank = r;
        world = w;
        device = dev;
        slot_rows = rows;
        mine = win;
    }
    unsigned int* done = nullptr;               // arrival counters of k_ipc_rows (2)
    ~IpcTransport() override {
        for (int j = 0; j < world; ++j)
            if (j != rank && peer.size() == (size_t)world && peer[j]) cudaIpcCloseMemHandle(peer[j]);
        if (mine) cudaFree(mine);
        if (done) cudaFree(done);
    }
    bool fused_gather() const override { return true; }

    // send: rows sidx[soff[j] ..] of src -> peer j's staging, then ready;
    // receive: my staging -> recv + roff[j], then ack (2 launches)
    void exchange_gather(cudaStream_t s, const float* src, const int32_t* sidx, const int64_t* soff,
                         const int64_t* scnt, float* recv, const int64_t* roff, const int64_t* rcnt,
                         int width) override {
        exchange_gather_begin(s, src, sidx, soff, scnt, recv, roff, rcnt, width);
        exchange_gather_end(s);
    }
    IpcRows pending{};  // receive half of the exchange begun last
    long long pending_k = 0;
    int pending_w = 0, pending_grid = 0;
    void exchange_gather_begin(cudaStream_t s, const float* src, const int32_t* sidx,
                               const int64_t* soff, const int64_t* scnt, float* recv,
                               const int64_t* roff, const int64_t* rcnt, int width) override {
        if (pending_k) raise(kRuntime, "internal: IPC exchange begun twice");
        if (!done) {
            GMD_CUDA(cudaMalloc(&done, 2 * sizeof(unsigned int)));
            GMD_CUDA(cudaMemsetAsync(done, 0, 2 * sizeof(unsigned int), s));
        }
        const long long k = ++epoch;
        const int par = (int)(k & 1);
        IpcRows snd{}, rcv{};
        long long maxrows = 0;
        for (int j = 0; j < world; ++j) {
            if (j == rank) continue;
            if (scnt[j] * width > slot_rows * 16 || rcnt[j] * width > slot_rows * 16)
                raise(kConfig, "IPC staging too small for the halo (raise staging_rows)");
            const IpcWin pw = ipc_view(peer[j]), mw = ipc_view(mine);
            const int i = snd.n;
            snd.wflag[i] = mw.ack + j;  // j consumed my exchange k-2 (j writes my window)
            snd.sflag[i] = pw.ready + rank;
            snd.dst[i] = reinterpret_cast<uint32_t*>(staging(peer[j], par, rank));
            snd.src[i] = reinterpret_cast<const uint32_t*>(src);
            snd.idx[i] = sidx + soff[j];
            snd.rows[i] = scnt[j];
            rcv.wflag[i] = mw.ready + j;
            rcv.sflag[i] = pw.ack + rank;  // j may reuse staging[k & 1][it] at k + 2
            rcv.dst[i] = reinterpret_cast<uint32_t*>(recv + roff[j] * width);
            rcv.src[i] = reinterpret_cast<const uint32_t*>(staging(mine, par, j));
            rcv.idx[i] = nullptr;
            rcv.rows[i] = rcnt[j];
            maxrows = std::max<long long>(maxrows, std::max<long long>(scnt[j], rcnt[j]));
            snd.n = rcv.n = i + 1;
        }
        const int grid = (int)std::max<long long>(1, std::min<long long>(148, (maxrows * width + 255) / 256));
        k_ipc_rows<<<grid, 256, 0, s>>>(snd, width, k - 2, k, done);
        GMD_LAUNCH_CHECK();
        pending = rcv;
        pending_k = k;
        pending_w = width;
        pending_grid = grid;
    }
    void exchange_gather_end(cudaStream_t s) override {
        if (!pending_k) raise(kRuntime, "internal: IPC exchange not begun");
        k_ipc_rows<<<pending_grid, 256, 0, s>>>(pending, pending_w, pending_k, pending_k, done + 1);
        pending_k = 0;
        GMD_LAUNCH_CHECK();
    }
    const char* name() const override { return "ipc"; }

    float* staging(void* base, int par, int slot) const {
        return ipc_view(base).staging + ((size_t)par * world + slot) * (size_t)slot_rows * 16;
    }

    void exchange(cudaStream_t s, const float* send, const int64_t* soff, const int64_t* scnt,
                  float* recv, const int64_t* roff, const int64_t* rcnt, int width) override {
        const long long k = ++epoch;
        const int par = (int)(k & 1);
        IpcPeers snd{}, sig{}, rcv{}, ack{};
        for (int j = 0; j < world; ++j) {
            if (j == rank) continue;
            if (scnt[j] * width > slot_rows * 16 || rcnt[j] * width > slot_rows * 16)
                raise(kConfig, "IPC staging too small for the halo (raise staging_rows)");
            const IpcWin pw = ipc_view(peer[j]), mw = ipc_view(mine);
            const int i = snd.n;
            snd.wflag[i] = mw.ack + j;  // j consumed my exchange k-2 (j writes my window)
            snd.dst[i] = staging(peer[j], par, rank);
            snd.src[i] = send + soff[j] * width;
            snd.cnt[i] = scnt[j] * width;
            sig.sflag[i] = pw.ready + rank;
            rcv.wflag[i] = mw.ready + j;
            rcv.dst[i] = recv + roff[j] * width;
            rcv.src[i] = staging(mine, par, j);
            rcv.cnt[i] = rcnt[j] * width;
            ack.sflag[i] = pw.ack + rank;
            snd.n = sig.n = rcv.n = ack.n = i + 1;
        }
        k_ipc_copy<<<148, 256, 0, s>>>(snd, k - 2);
        GMD_LAUNCH_CHECK();
        k_ipc_signal<<<1, 32, 0, s>>>(sig, k);
        GMD_LAUNCH_CHECK();
        k_ipc_copy<<<148, 256, 0, s>>>(rcv, k);
        GMD_LAUNCH_CHECK();
        // ack into each sender's window: it may reuse staging[k & 1][it] at k + 2
        k_ipc_signal<<<1, 32, 0, s>>>(ack, k);
        GMD_LAUNCH_CHECK();
    }

    void gather(cudaStream_t s, const void* in, int n, void* out) {
        if (n > kIpcGatherMax) raise(kRuntime, "internal: IPC all-gather too large");
        const long long k = ++gepoch;
        IpcPeers w{}, sig{};
        for (int j = 0; j < world; ++j) {
            if (j == rank) continue;
            w.wflag[w.n++] = ipc_view(mine).gack + j;  // j read my previous payload
        }
        // my payload into every window's slot `rank` (mine included)
        double* stage = ipc_view(mine).gather + (size_t)rank * 32;
        GMD_CUDA(cudaMemcpyAsync(stage, in, 8 * n, cudaMemcpyHostToDevice, s));
        IpcPeers cp{};
        for (int j = 0; j < world; ++j) {
            if (j == rank) continue;
            const int i = cp.n++;
            cp.wflag[i] = w.wflag[i];
            cp.dst[i] = reinterpret_cast<float*>(ipc_view(peer[j]).gather + (size_t)rank * 32);
            cp.src[i] = reinterpret_cast<const float*>(stage);
            cp.cnt[i] = 2 * n;
            sig.sflag[sig.n++] = ipc_view(peer[j]).gready + rank;
        }
        k_ipc_copy<<<1, 64, 0, s>>>(cp, k - 1);
        GMD_LAUNCH_CHECK();
        k_ipc_signal<<<1, 32, 0, s>>>(sig, k);
        GMD_LAUNCH_CHECK();
        IpcPeers rd{};
        for (int j = 0; j < world; ++j)
            if (j != rank) rd.wflag[rd.n++] = ipc_view(mine).gready + j;
        k_ipc_copy<<<1, 32, 0, s>>>(rd, k);  // wait only (no copies)
        GMD_LAUNCH_CHECK();
        std::vector<double> all((size_t)world * 32);
        GMD_CUDA(cudaMemcpyAsync(all.data(), ipc_view(mine).gather, 8 * all.size(),
                                 cudaMemcpyDeviceToHost, s));
        IpcPeers ak{};
        for (int j = 0; j < world; ++j)
            if (j != rank) ak.sflag[ak.n++] = ipc_view(peer[j]).gack + rank;
        k_ipc_signal<<<1, 32, 0, s>>>(ak, k);
        GMD_LAUNCH_CHECK();
        GMD_CUDA(cudaStreamSynchronize(s));
        for (int j = 0; j < world; ++j)
            std::memcpy(static_cast<char*>(out) + (size_t)j * 8 * n, all.data() + (size_t)j * 32, 8 * n);
    }
    void allgather_f64(cudaStream_t s, const double* in, int n, double* out) override {
        gather(s, in, n, out);
    }
    void allgather_i64(cudaStream_t s, const int64_t* in, int n, int64_t* out) override {
        gather(s, in, n, out);
    }
};

}  // namespace

size_t ipc_window_bytes(int world, int64_t slot_rows) {
    return kIpcFlags + kIpcGather + sizeof(float) * 2 * (size_t)world * (size_t)slot_rows * 16;
}

void* ipc_window_create(int world, int64_t slot_rows, unsigned char handle[64]) {
    if (world < 1 || world > kIpcMaxWorld) raise(kConfig, "IPC transport supports 1..16 ranks");
    void* w = nullptr;
    GMD_CUDA(cudaMalloc(&w, ipc_window_bytes(world, slot_rows)));
    GMD_CUDA(cudaMemset(w, 0, kIpcFlags + kIpcGather));
    cudaIpcMemHandle_t hd;
    GMD_CUDA(cudaIpcGetMemHandle(&hd, w));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    std::memcpy(handle, &hd, 64);
    return w;
}

Transport* make_ipc_transport(int rank, int world, int device, int64_t slot_rows, void* window,
                              const unsigned char* handles) {
    auto* t = new IpcTransport(rank, world, device, slot_rows, window);
    t->peer.assign(world, nullptr);
    for (int j = 0; j < world; ++j) {
        if (j == rank) {
            t->peer[j] = window;
            continue;
        }
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, handles + 64 * (size_t)j, 64);
        cudaError_t e = cudaIpcOpenMemHandle(&t->peer[j], hd, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            t->peer[j] = nullptr;
            delete t;
            raise(kCuda, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        }
    }
    return t;
}

Transport* make_local_transport(LocalGroup* g, int rank) { return new LocalTransport(g, rank); }

bool nccl_unique_id(unsigned char id[128], std::string* err) {
    if (!nccl().load()) {
        if (err) *err = nccl().err;
        return false;
    }
    int rc = nccl().GetUniqueId(id);
    if (rc != 0) {
        if (err) *err = "ncclGetUniqueId failed";
        return false;
    }
    return true;
}

Transport* make_nccl_transport(int rank, int world, const unsigned char id[128], int device) {
    return new NcclTransport(rank, world, id, device);
}

}  // namespace gmd
