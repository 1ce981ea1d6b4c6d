// Model kernels for any feature width / basis count (the reference supports
// arbitrary ToyPotentialParams widths, potential.hpp:15-41).  The tuned
// kernels (gmd_model.cu) are compiled for F = 16, K = 8 with the parameters
// in constant memory; these read fp32 parameter tables from global memory,
// one warp per node with lanes over features (F <= 128) and over basis
// functions (K <= 32).  Same row-form, atomics-free formulation, so results
// are partition-invariant; not tuned (the SURVEY configurations use F = 16).
#pragma once
#include "gmd_model.cuh"

namespace gmd {

constexpr int kGenMaxF = 128, kGenMaxK = 32;

struct GenModel {
    int F = 0, K = 0, L = 0;
    const float* emb = nullptr;  // 119 x F
    const float* W = nullptr;    // L x F x F (row f: W[f][g])
    const float* b = nullptr;    // L x F
    const float* P = nullptr;    // F x K
    const float* Pk = nullptr;   // F x K: k P[f][k]
    const float* ro = nullptr;   // F
    const float* P3 = nullptr;   // F x K   (three-body)
    const float* W3 = nullptr;   // F x F
    const float* W4 = nullptr;   // F x F
    // transposed copies, so lanes over f read consecutive addresses
    const float* WT = nullptr;   // L x F x F: WT[l][g][f] = W[l][f][g]
    const float* W3T = nullptr;
    const float* W4T = nullptr;
    const float* P3T = nullptr;  // K x F: P3T[k][f] = P3[f][k]
    float rc = 0, inv_rc = 0, inv_sigma = 0, mu_step = 0;
    float r3 = 1, inv_r3 = 1, inv_sigma3 = 0, mu_step3 = 0;
};

int gen_grid(int64_t n);  // CTAs of the warp-per-node kernels (8 warps each)
void launch_gen_embed(const GenModel& g, int64_t rows, const int32_t* node_array, const int32_t* Z,
                      float* H0, cudaStream_t s, uint8_t* zs = nullptr, unsigned* zmask = nullptr);
// Hout[own] = Hin[own] + tanh(W_l m + b_l); TH_l; per-atom energies on the last layer
void launch_gen_conv(const GenModel& g, const ConvArgs& a, int layer, const float* Hin, float* Hout,
                     float* TH, double* per_atom, cudaStream_t s);
void launch_gen_init_hbar(const GenModel& g, int64_t n, float* HB, cudaStream_t s);
void launch_gen_bwd_node(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                         int layer, const float* HB, const float* TH, float* MB, cudaStream_t s);
// vir_part: gen_grid(n) * 8 records of 6 doubles (one per warp)
void launch_gen_bwd_edge(const GenModel& g, const ConvArgs& a, const float* MB, const float* Hl,
                         float* HB, double4* GRAD, double* vir_part, cudaStream_t s);

// three-body stage (potential.cpp:664-741, 850-961), same slot conventions
// as the tuned kernels (TP/TH3 slot j of a center = the reverse bond of its
// in-bond j); TT / SMR: B x F scratch rows (t of every bond, m_bar_3 per slot)
void launch_gen_tb_t(const GenModel& g, const BondArgs& a, int64_t nbonds, float* TT, cudaStream_t s);
void launch_gen_tb_forward(const GenModel& g, const BondArgs& a, const float* TT, float* TP,
                           float* TH3, int32_t* flags, cudaStream_t s);
void launch_gen_tb_inject(const GenModel& g, const BondArgs& a, const float* TP, float* H, float* TH4,
                          cudaStream_t s);
void launch_gen_tb_bwd_q(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                         const float* HB, const float* TH4, float* QB, cudaStream_t s);
// vir_part: gen_grid(a.n) * 8 records of 9 doubles
void launch_gen_tb_backward(const GenModel& g, const BondArgs& a, const float* QB, const float* TH3,
                            const float* TT, float* SMR, float4* VIN, float4* VOUT, double* vir_part,
                            cudaStream_t s);

}  // namespace gmd
