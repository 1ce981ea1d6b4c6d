// Throughput probe: per-row gathers of random 64-byte rows from a 64 MB
// table into shared memory, three ways, each lane fetching 2 rows per step
// (the backward edge pass's m_bar / h rows):
//   ldg  : 2 x ld.global.nc.v8 (LDG.256) per row into registers
//   tma  : cp.async.bulk 64 B per row with a per-lane mbarrier (expect_tx)
//   lgs  : cp.async.ca 16 B x 4 per row (LDGSTS)
// Prints rows/ns over the whole GPU.   nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_ldg(const float* __restrict__ tab, const int* __restrict__ idx, int steps, float* out) {
    float acc = 0.f;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int s = 0; s < steps; ++s) {
        const int i0 = idx[(t * 2 + s * 977) & 0xfffff], i1 = idx[(t * 2 + 1 + s * 977) & 0xfffff];
        const float4* a = reinterpret_cast<const float4*>(tab + (size_t)i0 * 16);
        const float4* b = reinterpret_cast<const float4*>(tab + (size_t)i1 * 16);
        float4 x0 = __ldg(a), x1 = __ldg(a + 1), x2 = __ldg(a + 2), x3 = __ldg(a + 3);
        float4 y0 = __ldg(b), y1 = __ldg(b + 1), y2 = __ldg(b + 2), y3 = __ldg(b + 3);
        acc += x0.x + x1.y + x2.z + x3.w + y0.x + y1.y + y2.z + y3.w;
    }
    out[t] = acc;
}

// U independent row pairs in flight per thread (memory-level parallelism)
template <int U>
__global__ void k_ldgU(const float* __restrict__ tab, const int* __restrict__ idx, int steps, float* out) {
    float acc[U] = {};
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int s = 0; s < steps; s += U) {
        float4 x[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i0 = idx[(t * 2 + (s + u) * 977) & 0xfffff], i1 = idx[(t * 2 + 1 + (s + u) * 977) & 0xfffff];
            const float4* a = reinterpret_cast<const float4*>(tab + (size_t)i0 * 16);
            const float4* b = reinterpret_cast<const float4*>(tab + (size_t)i1 * 16);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                x[u][c] = __ldg(a + c);
                x[u][4 + c] = __ldg(b + c);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            acc[u] += x[u][0].x + x[u][1].y + x[u][2].z + x[u][3].w + x[u][4].x + x[u][5].y + x[u][6].z + x[u][7].w;
    }
    float r = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) r += acc[u];
    out[t] = r;
}

__global__ void k_tma(const float* __restrict__ tab, const int* __restrict__ idx, int steps, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    float* slot = reinterpret_cast<float*>(sm) + threadIdx.x * 32;
    uint64_t* mb = reinterpret_cast<uint64_t*>(sm + blockDim.x * 128) + threadIdx.x;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mb)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    float acc = 0.f;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t phase = 0;
    for (int s = 0; s < steps; ++s) {
        const int i0 = idx[(t * 2 + s * 977) & 0xfffff], i1 = idx[(t * 2 + 1 + s * 977) & 0xfffff];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 128;" ::"r"(su32(mb)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];"
                     ::"r"(su32(slot)), "l"(tab + (size_t)i0 * 16), "r"(su32(mb)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];"
                     ::"r"(su32(slot + 16)), "l"(tab + (size_t)i1 * 16), "r"(su32(mb)) : "memory");
        asm volatile("{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}"
                     ::"r"(su32(mb)), "r"(phase) : "memory");
        phase ^= 1;
        acc += slot[0] + slot[5] + slot[16] + slot[31];
    }
    out[t] = acc;
}

__global__ void k_lgs(const float* __restrict__ tab, const int* __restrict__ idx, int steps, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    float* slot = reinterpret_cast<float*>(sm) + threadIdx.x * 32;
    float acc = 0.f;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int s = 0; s < steps; ++s) {
        const int i0 = idx[(t * 2 + s * 977) & 0xfffff], i1 = idx[(t * 2 + 1 + s * 977) & 0xfffff];
        for (int c = 0; c < 4; ++c)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(su32(slot + 4 * c)),
                         "l"(tab + (size_t)i0 * 16 + 4 * c));
        for (int c = 0; c < 4; ++c)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(su32(slot + 16 + 4 * c)),
                         "l"(tab + (size_t)i1 * 16 + 4 * c));
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        acc += slot[0] + slot[5] + slot[16] + slot[31];
    }
    out[t] = acc;
}

int main() {
    const int rows = 1 << 20;  // 64 MB table
    float* tab;
    int* idx;
    float* out;
    cudaMalloc(&tab, (size_t)rows * 64);
    cudaMalloc(&idx, sizeof(int) << 20);
    cudaMalloc(&out, sizeof(float) * 148 * 2048);
    cudaMemset(tab, 0, (size_t)rows * 64);
    int* h = new int[1 << 20];
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < (1 << 20); ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[i] = (int)(x % rows);
    }
    cudaMemcpy(idx, h, sizeof(int) << 20, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int steps = 200;
    for (int block : {256, 768}) {
        const int grid = 148 * (block == 256 ? 3 : 1);
        const size_t sm = block * 128 + block * 8;
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(k_lgs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int rep = 0; rep < 2; ++rep) {
            float ms;
            const double nrows = 2.0 * grid * block * steps;
            cudaEventRecord(e0);
            k_ldg<<<grid, block>>>(tab, idx, steps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("block %4d ldg: %.3f ms %.2f rows/ns\n", block, ms, nrows / ms / 1e6);
            cudaEventRecord(e0);
            k_ldgU<4><<<grid, block>>>(tab, idx, steps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("block %4d ldg x4: %.3f ms %.2f rows/ns\n", block, ms, nrows / ms / 1e6);
            cudaEventRecord(e0);
            k_ldgU<2><<<grid, block>>>(tab, idx, steps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("block %4d ldg x2: %.3f ms %.2f rows/ns\n", block, ms, nrows / ms / 1e6);
            cudaEventRecord(e0);
            k_tma<<<grid, block, sm>>>(tab, idx, steps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("block %4d tma: %.3f ms %.2f rows/ns  (%s)\n", block, ms, nrows / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
            cudaEventRecord(e0);
            k_lgs<<<grid, block, sm>>>(tab, idx, steps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("block %4d lgs: %.3f ms %.2f rows/ns\n", block, ms, nrows / ms / 1e6);
        }
    }
    return 0;
}
