// Throughput probe: random 64-byte row gathers from a 64 MB table, by how
// many lanes share one row (the L1TEX data pipe, not DRAM/L2, limits the
// model kernels' gathers: lsu wavefronts at 86 % in k_bwd_edge2).
//   lane1 : each lane reads whole rows        (2 x LDG.256 per row)
//   lane2 : a lane pair reads one row         (1 x LDG.256 per lane)
//   lane4 : a lane quad reads one row         (1 x LDG.128 per lane)
// Each variant reads R rows per lane-step-equivalent; prints rows/ns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_coop_probe tools/gather_coop_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const float* p, float4& a, float4& b) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                   "=f"(b.w)
                 : "l"(p));
}

// G lanes per row; every lane issues 2 row-slices per step (like the
// backward's m_bar/h rows), so rows per warp-step = 2 * 32 / G
template <int G>
__global__ void k_gather(const float* __restrict__ tab, const int* __restrict__ idx, int steps,
                         float* out) {
    float acc = 0.f;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int part = threadIdx.x & (G - 1);
    const int slot = t / G;
    for (int s = 0; s < steps; ++s) {
        const int i0 = __ldg(idx + ((slot * 2 + s * 977) & 0xfffff));
        const int i1 = __ldg(idx + ((slot * 2 + 1 + s * 977) & 0xfffff));
        const float* a = tab + (size_t)i0 * 16;
        const float* b = tab + (size_t)i1 * 16;
        if (G == 1) {
            float4 x0, x1, x2, x3, y0, y1, y2, y3;
            ld256(a, x0, x1);
            ld256(a + 8, x2, x3);
            ld256(b, y0, y1);
            ld256(b + 8, y2, y3);
            acc += x0.x + x1.y + x2.z + x3.w + y0.x + y1.y + y2.z + y3.w;
        } else if (G == 2) {
            float4 x0, x1, y0, y1;
            ld256(a + 8 * part, x0, x1);
            ld256(b + 8 * part, y0, y1);
            acc += x0.x + x1.y + y0.z + y1.w;
        } else {
            const float4 x = __ldg(reinterpret_cast<const float4*>(a) + part);
            const float4 y = __ldg(reinterpret_cast<const float4*>(b) + part);
            acc += x.x + y.w;
        }
    }
    out[t] = acc;
}

// each lane still ends with its own two full rows, but every load
// instruction is shared by a lane pair: in step A the pair reads the two
// halves of the even lane's row, in step B of the odd lane's row; then each
// lane swaps the half it holds of its partner's row (8 SHFL per row)
__global__ void k_pair_swap(const float* __restrict__ tab, const int* __restrict__ idx, int steps,
                            float* out) {
    float acc = 0.f;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, half = lane & 1;
    for (int s = 0; s < steps; ++s) {
        const int i0 = __ldg(idx + ((t * 2 + s * 977) & 0xfffff));
        const int i1 = __ldg(idx + ((t * 2 + 1 + s * 977) & 0xfffff));
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int mine = r ? i1 : i0;
            const int other = __shfl_xor_sync(0xffffffffu, mine, 1);
            const int ra = half ? other : mine;   // row of the even lane
            const int rb = half ? mine : other;   // row of the odd lane
            float4 a0, a1, b0, b1;
            ld256(tab + (size_t)ra * 16 + 8 * half, a0, a1);  // halves of the even lane's row
            ld256(tab + (size_t)rb * 16 + 8 * half, b0, b1);  // halves of the odd lane's row
            // even lane keeps a (its row, half 0) and needs half 0 of... : it
            // holds half 0 of both rows; it needs half 1 of its row (held by
            // the odd lane as a) and gives half 0 of the odd row (b).
            float4 s0 = half ? a0 : b0, s1 = half ? a1 : b1;  // what the partner needs
            float4 g0, g1;
            g0.x = __shfl_xor_sync(0xffffffffu, s0.x, 1); g0.y = __shfl_xor_sync(0xffffffffu, s0.y, 1);
            g0.z = __shfl_xor_sync(0xffffffffu, s0.z, 1); g0.w = __shfl_xor_sync(0xffffffffu, s0.w, 1);
            g1.x = __shfl_xor_sync(0xffffffffu, s1.x, 1); g1.y = __shfl_xor_sync(0xffffffffu, s1.y, 1);
            g1.z = __shfl_xor_sync(0xffffffffu, s1.z, 1); g1.w = __shfl_xor_sync(0xffffffffu, s1.w, 1);
            // own row: even = (a [half 0], g [half 1]); odd = (g [half 0], b [half 1])
            const float4 h0 = half ? g0 : a0, h1 = half ? g1 : a1;
            const float4 h2 = half ? b0 : g0, h3 = half ? b1 : g1;
            acc += h0.x + h1.y + h2.z + h3.w;
        }
    }
    out[t] = acc;
}

int main() {
    const int rows = 1 << 20;
    float *tab, *out;
    int* idx;
    cudaMalloc(&tab, (size_t)rows * 64);
    cudaMalloc(&idx, sizeof(int) << 20);
    cudaMalloc(&out, sizeof(float) * 148 * 2048);
    cudaMemset(tab, 0, (size_t)rows * 64);
    int* h = new int[1 << 20];
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < (1 << 20); ++i) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        h[i] = (int)(x % rows);
    }
    cudaMemcpy(idx, h, sizeof(int) << 20, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int steps = 200;
    for (int block : {256, 768}) {
        const int grid = 148 * (block == 256 ? 3 : 1);
        for (int rep = 0; rep < 2; ++rep) {
            float ms;
            auto run = [&](auto kern, int G, const char* name) {
                cudaEventRecord(e0);
                kern<<<grid, block>>>(tab, idx, steps, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                const double nrows = 2.0 * grid * block / G * steps;
                printf("block %4d %s: %.3f ms %.2f rows/ns\n", block, name, ms, nrows / ms / 1e6);
            };
            run(k_gather<1>, 1, "lane1 (2 x LDG.256 / row)");
            run(k_gather<2>, 2, "lane2 (LDG.256 / lane) ");
            run(k_gather<4>, 4, "lane4 (LDG.128 / lane) ");
            run(k_pair_swap, 1, "pair loads + SHFL swap ");
        }
    }
    return 0;
}
