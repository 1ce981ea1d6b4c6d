// Throughput probe: random 64-byte rows (16 fp32, the model kernels' feature
// rows) from a 64 MB table into shared memory with the Blackwell TMA row
// gather (cp.async.bulk.tensor.2d.tile::gather4: one instruction, four rows by
// index), against per-lane LDG.256 into registers (tools/tma_gather_probe.cu).
// Each CTA double-buffers a tile of rows: the rows of tile s+1 are requested by
// warp 0's lanes (one gather4 per lane) while every thread reads tile s from
// shared memory (LDS.128, 64-byte swizzle so 8-lane phases are conflict-free).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather4_probe tools/gather4_probe.cu
// Prints: validation, then rows/ns for the whole GPU per variant.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                              \
        }                                                                         \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* mb, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mb)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
            su32(mb)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, uint64_t* mb, int col, int r0, int r1,
                                        int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(su32(mb)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

constexpr int kRowsPerTile = 256;  // rows gathered per CTA tile (64 gather4 = 2 per lane of warp 0)
constexpr int kThreads = 256;      // one row per thread per tile

// rows of tile `s` for CTA b: idx[(b * steps + s) * kRowsPerTile + r]
__global__ void __launch_bounds__(kThreads) k_g4(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                 int steps, int nidx, float* out, int swz) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float* buf0 = reinterpret_cast<float*>(sm);
    float* buf1 = buf0 + kRowsPerTile * 16;
    uint64_t* mb = reinterpret_cast<uint64_t*>(buf1 + kRowsPerTile * 16);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {
        mbar_init(mb, 1);
        mbar_init(mb + 1, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](int s) {
        if (warp != 0 || s >= steps) return;
        float* dst = (s & 1) ? buf1 : buf0;
        uint64_t* m = mb + (s & 1);
        if (lane == 0) mbar_expect(m, kRowsPerTile * 64);
        __syncwarp();
        const int64_t base = ((int64_t)blockIdx.x * steps + s) * kRowsPerTile;
#pragma unroll
        for (int q = 0; q < kRowsPerTile / 128; ++q) {
            const int r = (q * 32 + lane) * 4;
            const int* ip = idx + ((base + r) % nidx);
            gather4(dst + r * 16, &tm, m, 0, ip[0], ip[1], ip[2], ip[3]);
        }
    };
    issue(0);
    float acc = 0.f;
    for (int s = 0; s < steps; ++s) {
        issue(s + 1);
        mbar_wait(mb + (s & 1), (s >> 1) & 1);
        const float* src = (s & 1) ? buf1 : buf0;
        // thread t reads row t: 4 x LDS.128 (chunk c at c ^ ((row >> 1) & 3) with 64B swizzle)
        const float4* row = reinterpret_cast<const float4*>(src + t * 16);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int pc = swz ? (c ^ ((t >> 1) & 3)) : c;
            const float4 v = row[pc];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncthreads();  // buffer s&1 is free for tile s+2
    }
    out[blockIdx.x * kThreads + t] = acc;
}

// validation: one tile, copy out what landed
__global__ void k_g4_check(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, float* out, int swz) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float* buf = reinterpret_cast<float*>(sm);
    uint64_t* mb = reinterpret_cast<uint64_t*>(buf + 2 * kRowsPerTile * 16);
    const int t = threadIdx.x, lane = t & 31;
    if (t == 0) mbar_init(mb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (t < 32) {
        if (lane == 0) mbar_expect(mb, kRowsPerTile * 64);
        __syncwarp();
        for (int q = 0; q < kRowsPerTile / 128; ++q) {
            const int r = (q * 32 + lane) * 4;
            gather4(buf + r * 16, &tm, mb, 0, idx[r], idx[r + 1], idx[r + 2], idx[r + 3]);
        }
    }
    mbar_wait(mb, 0);
    for (int i = t; i < kRowsPerTile * 16; i += kThreads) {
        const int r = i / 16, c = (i % 16) / 4, e = i % 4;
        const int pc = swz ? (c ^ ((r >> 1) & 3)) : c;
        out[i] = buf[r * 16 + pc * 4 + e];
    }
}

__global__ void k_ldg(const float* __restrict__ tab, const int* __restrict__ idx, int steps, int nidx, float* out) {
    float acc = 0.f;
    const int t = threadIdx.x;
    for (int s = 0; s < steps; ++s) {
        const int64_t base = ((int64_t)blockIdx.x * steps + s) * kRowsPerTile;
        const int i0 = idx[(base + t) % nidx];
        const float4* a = reinterpret_cast<const float4*>(tab + (size_t)i0 * 16);
        float4 x0, x1, x2, x3;
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(x0.x), "=f"(x0.y), "=f"(x0.z), "=f"(x0.w), "=f"(x1.x), "=f"(x1.y), "=f"(x1.z), "=f"(x1.w)
                     : "l"(a));
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(x2.x), "=f"(x2.y), "=f"(x2.z), "=f"(x2.w), "=f"(x3.x), "=f"(x3.y), "=f"(x3.z), "=f"(x3.w)
                     : "l"(a + 2));
        acc += x0.x + x1.y + x2.z + x3.w + x0.w + x1.z + x2.y + x3.x;
    }
    out[blockIdx.x * kThreads + t] = acc;
}

int main() {
    const int nrows = 1 << 20;  // 64 MB table
    const int nidx = 1 << 22;
    std::vector<float> h(size_t(nrows) * 16);
    for (size_t i = 0; i < h.size(); ++i) h[i] = float(i % 9973) * 0.5f;
    std::vector<int> hi(nidx);
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < nidx; ++i) {
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
        hi[i] = int(x % nrows);
    }
    float *tab, *out;
    int* idx;
    CK(cudaMalloc(&tab, h.size() * 4));
    CK(cudaMalloc(&idx, nidx * 4));
    CK(cudaMalloc(&out, 64 << 20));
    CK(cudaMemcpy(tab, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx, hi.data(), nidx * 4, cudaMemcpyHostToDevice));

    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    int dev = 0, nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));

    for (int swz = 0; swz < 2; ++swz) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {16, (cuuint64_t)nrows};
        cuuint64_t strides[1] = {64};
        cuuint32_t box[2] = {16, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            swz ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode (swizzle %d) failed: %d\n", swz, (int)r);
            continue;
        }
        const size_t smem = 2 * kRowsPerTile * 64 + 64;
        CK(cudaFuncSetAttribute(k_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_g4_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_g4_check<<<1, kThreads, smem>>>(tm, idx, out, swz);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(kRowsPerTile * 16);
        CK(cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int rr = 0; rr < kRowsPerTile; ++rr)
            for (int c = 0; c < 16; ++c)
                if (o[rr * 16 + c] != h[size_t(hi[rr]) * 16 + c]) ++bad;
        printf("gather4 swizzle=%d validation: %d bad of %d\n", swz, bad, kRowsPerTile * 16);

        for (int ctas_per_sm : {1, 2, 4, 8}) {
            const int grid = nsm * ctas_per_sm, steps = 200;
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            k_g4<<<grid, kThreads, smem>>>(tm, idx, steps, nidx, out, swz);
            CK(cudaEventRecord(a));
            k_g4<<<grid, kThreads, smem>>>(tm, idx, steps, nidx, out, swz);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            printf("gather4 swz=%d ctas/SM=%d: %.1f rows/ns (%.3f ms)\n", swz, ctas_per_sm,
                   double(grid) * steps * kRowsPerTile / (ms * 1e6), ms);
        }
    }
    for (int ctas_per_sm : {2, 4, 8}) {
        const int grid = nsm * ctas_per_sm, steps = 200;
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        k_ldg<<<grid, kThreads>>>(tab, idx, steps, nidx, out);
        CK(cudaEventRecord(a));
        k_ldg<<<grid, kThreads>>>(tab, idx, steps, nidx, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("ldg256 ctas/SM=%d: %.1f rows/ns (%.3f ms)\n", ctas_per_sm, double(grid) * steps * kRowsPerTile / (ms * 1e6),
               ms);
    }
    CK(cudaGetLastError());
    return 0;
}
