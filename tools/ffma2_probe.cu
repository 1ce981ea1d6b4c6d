// Throughput probe: scalar FFMA vs packed FFMA2 (sm_100a) vs uniform-operand
// FFMA.  Prints GFMA/s for each; used to pick the FP32 formulation of the
// model kernels.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, int iters, float s) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 0.5f);
    float t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_ffma2(float* out, int iters, float s) {
    float2 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 s2 = make_float2(s, s), h = make_float2(0.5f, 0.5f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], s2, h);
    float t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += a[i].x + a[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 64 * 256 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, grid = 148 * 8, block = 256;
    for (int pass = 0; pass < 2; ++pass) {
        float ms;
        k_ffma<<<grid, block>>>(out, 16, 1.0001f);
        cudaEventRecord(e0);
        k_ffma<<<grid, block>>>(out, iters, 1.0001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fma = (double)grid * block * iters * 16 * 8;
        printf("FFMA : %.3f ms  %.1f TFMA/s  %.1f Tinst(warp)/s\n", ms, fma / ms / 1e9, fma / 32 / ms / 1e9);
        k_ffma2<<<grid, block>>>(out, 16, 1.0001f);
        cudaEventRecord(e0);
        k_ffma2<<<grid, block>>>(out, iters, 1.0001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fma = (double)grid * block * iters * 16 * 8 * 2;
        printf("FFMA2: %.3f ms  %.1f TFMA/s  %.1f Tinst(warp)/s\n", ms, fma / ms / 1e9, fma / 64 / ms / 1e9);
    }
    return 0;
}
