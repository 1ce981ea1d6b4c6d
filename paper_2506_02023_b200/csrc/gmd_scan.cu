// Exclusive prefix sums used for every CSR / compaction offset in the build.
// Three passes: per-tile reduce -> single-CTA scan of tile sums -> per-tile
// scan with the tile's base.  Tiles are 4096 items (512 threads x 8).
#include "gmd_common.cuh"

namespace gmd {
long long g_gmd_launches = 0;
namespace {

constexpr int kThreads = 512;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

template <typename T>
__device__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// exclusive scan over the CTA; returns the CTA total through *total
template <typename T>
__device__ T block_excl_scan(T v, T* total) {
    __shared__ T warp_sums[kThreads / 32 + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T inc = warp_incl_scan(v);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T w = lane < kThreads / 32 ? warp_sums[lane] : T(0);
        T wi = warp_incl_scan(w);
        if (lane < kThreads / 32) warp_sums[lane] = wi - w;
        if (lane == kThreads / 32 - 1) warp_sums[kThreads / 32] = wi;  // total slot
    }
    __syncthreads();
    T res = warp_sums[wid] + inc - v;
    if (total) *total = warp_sums[kThreads / 32];
    __syncthreads();
    return res;
}

template <typename T>
__global__ void k_tile_reduce(const T* __restrict__ in, int64_t n, T* __restrict__ sums) {
    int64_t base = (int64_t)blockIdx.x * kTile;
    T acc = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int64_t i = base + (int64_t)k * kThreads + threadIdx.x;
        if (i < n) acc += in[i];
    }
    T tot;
    block_excl_scan<T>(acc, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <typename T>
__global__ void k_spine(T* sums, int64_t nt, T* total_out) {
    T carry = 0;
    for (int64_t b = 0; b < nt; b += kThreads) {
        int64_t i = b + threadIdx.x;
        T v = i < nt ? sums[i] : T(0);
        T tot;
        T ex = block_excl_scan<T>(v, &tot);
        if (i < nt) sums[i] = ex + carry;
        carry += tot;
    }
    if (threadIdx.x == 0) *total_out = carry;
}

template <typename T>
__global__ void k_tile_scan(const T* __restrict__ in, int64_t n, const T* __restrict__ bases,
                            T* __restrict__ out) {
    int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
    T v[kItems];
    T acc = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int64_t i = base + k;
        v[k] = i < n ? in[i] : T(0);
        acc += v[k];
    }
    T ex = block_excl_scan<T>(acc, nullptr) + bases[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int64_t i = base + k;
        if (i < n) out[i] = ex;
        ex += v[k];
    }
}

template <typename T>
void scan_impl(const T* in, T* out, int64_t n, void* tmp, size_t tmp_bytes, cudaStream_t s) {
    int64_t nt = (n + kTile - 1) / kTile;
    if (nt == 0) {
        GMD_CUDA(cudaMemsetAsync(out, 0, sizeof(T), s));
        return;
    }
    if ((size_t)nt * sizeof(T) > tmp_bytes) raise(kRuntime, "scan: temporary buffer too small");
    T* sums = static_cast<T*>(tmp);
    k_tile_reduce<T><<<(unsigned)nt, kThreads, 0, s>>>(in, n, sums);
    GMD_LAUNCH_CHECK();
    k_spine<T><<<1, kThreads, 0, s>>>(sums, nt, out + n);
    GMD_LAUNCH_CHECK();
    k_tile_scan<T><<<(unsigned)nt, kThreads, 0, s>>>(in, n, sums, out);
    GMD_LAUNCH_CHECK();
}

}  // namespace

size_t scan_tmp_bytes(int64_t n) { return (size_t)((n + kTile - 1) / kTile + 1) * 8; }

void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* tmp, size_t tmp_bytes,
                        cudaStream_t s) {
    scan_impl<int32_t>(in, out, n, tmp, tmp_bytes, s);
}
void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* tmp, size_t tmp_bytes,
                        cudaStream_t s) {
    scan_impl<int64_t>(in, out, n, tmp, tmp_bytes, s);
}

}  // namespace gmd
