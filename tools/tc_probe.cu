// Standalone probe of the tcgen05 primitives in gmd_tc.cuh:
// D[128 x 32] = A[128 x 8] . B[32 x 8]^T with 3xTF32 split, checked on the host.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2506_02023_b200/csrc/gmd_tc.cuh"
using namespace gmd;

__global__ void k_probe(const float* A, const float* B, float* D) {
    __shared__ __align__(1024) float a_hi[128 * 8], a_lo[128 * 8];
    __shared__ __align__(1024) float b_hi[32 * 8], b_lo[32 * 8];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x;
    for (int k = 0; k < 8; ++k) {
        float h, l;
        tc::split_tf32(A[t * 8 + k], h, l);
        a_hi[tc::kmajor_off(t, k)] = h;
        a_lo[tc::kmajor_off(t, k)] = l;
    }
    if (t < 32)
        for (int k = 0; k < 8; ++k) {
            float h, l;
            tc::split_tf32(B[t * 8 + k], h, l);
            b_hi[tc::kmajor_off(t, k)] = h;
            b_lo[tc::kmajor_off(t, k)] = l;
        }
    if (t == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
    if (t < 32) tc::tmem_alloc(&tbase, 32);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t d = tbase;
    if (t == 0) {
        const uint32_t id = tc::idesc_tf32(128, 32);
        tc::mma_tf32(d, tc::sdesc(a_hi), tc::sdesc(b_hi), id, false);
        tc::mma_tf32(d, tc::sdesc(a_lo), tc::sdesc(b_hi), id, true);
        tc::mma_tf32(d, tc::sdesc(a_hi), tc::sdesc(b_lo), id, true);
        tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    float v[32];
    tc::tmem_ld32(d + ((uint32_t)(32 * (t >> 5)) << 16), v);
    for (int i = 0; i < 32; ++i) D[t * 32 + i] = v[i];
    tc::fence_before();
    __syncthreads();
    if (t < 32) tc::tmem_free(d, 32);
}

int main() {
    std::vector<float> A(128 * 8), B(32 * 8), D(128 * 32);
    srand(1);
    for (auto& x : A) x = (rand() / (float)RAND_MAX);
    for (auto& x : B) x = (rand() / (float)RAND_MAX) * 2 - 1;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    k_probe<<<1, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 32; ++n) {
            double ref = 0;
            for (int k = 0; k < 8; ++k) ref += (double)A[m * 8 + k] * B[n * 8 + k];
            maxerr = fmax(maxerr, fabs(ref - D[m * 32 + n]));
            maxref = fmax(maxref, fabs(ref));
        }
    printf("tc_probe max_abs_err=%.3e max_ref=%.3e D[0][0]=%f D[127][31]=%f\n", maxerr, maxref, D[0], D[127 * 32 + 31]);
    return maxerr < 1e-5 ? 0 : 1;
}
