// Halo-exchange transports (see gmd_comm.cuh).
#include <dlfcn.h>

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

    explicit LocalGroup(int w)
        : world(w), refs(w), send(w), soff(w), scnt(w), dbuf(w), ibuf(w) {}

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
        for (int j = 0; j < world; ++j) {
            if (j == rank || rcnt[j] == 0) continue;
            if (g->scnt[j][rank] != rcnt[j]) raise(kRuntime, "transfer plan misalignment");
            GMD_CUDA(cudaMemcpyAsync(recv + roff[j] * width, g->send[j] + g->soff[j][rank] * width,
                                     sizeof(float) * rcnt[j] * width, cudaMemcpyDefault, s));
        }
        GMD_CUDA(cudaStreamSynchronize(s));
        g->barrier();  // peers are done reading this rank's send buffer
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

}  // namespace

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
