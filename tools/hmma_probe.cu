// Throughput/latency probe for the legacy warp-level tensor path on sm_100a:
// mma.sync.m16n8k8 tf32 (HMMA.1688.F32.TF32), independent chains vs one
// dependent chain.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 hmma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                    uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                 "{%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CH>
__global__ void k(float* out, int iters) {
    float d[CH][4] = {};
    uint32_t a = threadIdx.x * 0x3f800000u, b = 0x3f000000u;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int c = 0; c < CH; ++c) mma(d[c], a, a + 1, a + 2, a + 3, b, b + c);
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
void run(float* out, int warps_per_sm) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, block = 32 * warps_per_sm, grid = 148;
    k<CH><<<grid, block>>>(out, 16);
    cudaEventRecord(e0);
    k<CH><<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double n = (double)grid * warps_per_sm * iters * CH;  // warp-level mma
    const double cyc = ms * 1e-3 * 1.965e9;
    printf("chains=%d warps/SM=%2d: %.3f ms  %.2f cycles per mma per SMSP  %.1f TFLOP/s (1x tf32)\n", CH,
           warps_per_sm, ms, cyc / (n / 148 / 4), n * 2 * 16 * 8 * 8 / ms / 1e9);
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    run<1>(out, 4);
    run<1>(out, 16);
    run<4>(out, 4);
    run<4>(out, 16);
    run<8>(out, 16);
    run<8>(out, 32);
    return 0;
}
