// Shared device/host helpers for the graphmd B200 path (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace gmd {

// Error carrying a C-ABI status code; the ABI layer turns it into a return
// value plus the handle's last-error string (no exceptions cross the ABI).
struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum : int {
    kOk = 0,
    kConfig = 2,   // invalid configuration / input (reference: graphmd::Error)
    kRuntime = 3,  // runtime failure (non-finite features, plan misalignment)
    kCuda = 4,     // CUDA / NCCL failure
    kArg = 5,      // bad handle / pointer / index
};

[[noreturn]] inline void raise(int code, const std::string& m) { throw Status(code, m); }

#define GMD_CUDA(x)                                                                  \
    do {                                                                             \
        cudaError_t _e = (x);                                                        \
        if (_e != cudaSuccess)                                                       \
            ::gmd::raise(::gmd::kCuda, std::string("CUDA error: ") +                 \
                                           cudaGetErrorString(_e) + " at " #x);      \
    } while (0)

// every kernel launch is followed by exactly one GMD_LAUNCH_CHECK(), which
// also counts it (gmd_launch_count) so the bench can report its launches
extern long long g_gmd_launches;
#define GMD_LAUNCH_CHECK()                                   \
    do {                                                     \
        __atomic_add_fetch(&::gmd::g_gmd_launches, 1, __ATOMIC_RELAXED); \
        GMD_CUDA(cudaGetLastError());                        \
    } while (0)

constexpr int kMaxParts = 64;  // requirement masks are u64 (partitioner.cpp:13)

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------------------
// fp64 helpers with explicit round-to-nearest, unfused: the graph decisions
// must reproduce the reference's x86-64 (no FMA) arithmetic bit for bit
// (SURVEY Appendix A).
// ---------------------------------------------------------------------------
struct d3 {
    double x, y, z;
};

__host__ __device__ inline double mul_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
__host__ __device__ inline double add_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
__host__ __device__ inline double sub_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
// ((a.x*b.x + a.y*b.y) + a.z*b.z)
__host__ __device__ inline double dot_rn(d3 a, d3 b) {
    return add_rn(add_rn(mul_rn(a.x, b.x), mul_rn(a.y, b.y)), mul_rn(a.z, b.z));
}
// rows[0]*v.x + rows[1]*v.y + rows[2]*v.z, component-wise left to right
__host__ __device__ inline d3 rowvec_rn(const double* m9, double vx, double vy, double vz) {
    d3 r;
    r.x = add_rn(add_rn(mul_rn(m9[0], vx), mul_rn(m9[3], vy)), mul_rn(m9[6], vz));
    r.y = add_rn(add_rn(mul_rn(m9[1], vx), mul_rn(m9[4], vy)), mul_rn(m9[7], vz));
    r.z = add_rn(add_rn(mul_rn(m9[2], vx), mul_rn(m9[5], vy)), mul_rn(m9[8], vz));
    return r;
}

// Packed periodic-image offset: three signed 10-bit fields.
constexpr int kImgBias = 512;
__host__ __device__ inline uint32_t pack_img(int ox, int oy, int oz) {
    return (uint32_t)(ox + kImgBias) | ((uint32_t)(oy + kImgBias) << 10) |
           ((uint32_t)(oz + kImgBias) << 20);
}
__host__ __device__ inline void unpack_img(uint32_t v, int& ox, int& oy, int& oz) {
    ox = (int)(v & 1023u) - kImgBias;
    oy = (int)((v >> 10) & 1023u) - kImgBias;
    oz = (int)((v >> 20) & 1023u) - kImgBias;
}
__host__ __device__ inline bool img_in_range(int o) { return o >= -kImgBias && o < kImgBias; }

// ---------------------------------------------------------------------------
// Device scan (exclusive) -- decoupled into block reduce / spine / block scan.
// ---------------------------------------------------------------------------
// out[i] = sum(in[0..i)), out[n] = total (out must have n+1 slots).
void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* tmp, size_t tmp_bytes,
                        cudaStream_t s);
void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* tmp, size_t tmp_bytes,
                        cudaStream_t s);
size_t scan_tmp_bytes(int64_t n);

}  // namespace gmd
