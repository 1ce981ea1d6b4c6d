// Model kernels for the "CHGNet width" F = 64, K = 8 (SURVEY §8d's C4w):
// feature-major warps (lane = feature pair, so every gathered neighbour row
// is one coalesced 256-byte access), parameters in registers / shared
// memory, packed FP32 (FFMA2), and the per-edge K = 64 contraction of the
// backward (G = X P, X_f = mbar_u,f h_w,f + h_u,f mbar_w,f) on the 5th-gen
// tensor cores: tcgen05.mma kind::tf32 with a 3xTF32 split, X staged in
// shared memory by the feature lanes, G in TMEM read back by edge lanes.
// Same formulas, summation orders per node and atomics-free row form as the
// width-generic kernels (gmd_generic.cu), so results are partition- and
// rank-invariant.
#pragma once
#include "gmd_generic.cuh"

namespace gmd {

constexpr int kWideF = 64, kWideK = 8;

inline bool wide_model(const GenModel& g) { return g.F == kWideF && g.K == kWideK; }

int wide_conv_grid(int64_t n);
int wide_bwd_grid(int64_t n);  // = number of 6-double virial records of launch_wide_bwd_edge

// Hout[own] = Hin[own] + tanh(W_l m + b_l); TH_l; per-atom energies on the last layer
// zs / zmask (layer 0, h0 = the embeddings): the species-sum form
void launch_wide_conv(const GenModel& g, const ConvArgs& a, int layer, const float* Hin, float* Hout,
                      float* TH, double* per_atom, cudaStream_t s, const uint8_t* zs = nullptr,
                      const unsigned* zmask = nullptr);
// MB[row] = W_l^T (HB (.) (1 - TH_l^2)); init: HB := readout first
void launch_wide_bwd_node(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                          int layer, float* HB, const float* TH, float* MB, bool init,
                          cudaStream_t s);
// HB += gathered adjoints, GRAD += positional gradient, virial records
void launch_wide_bwd_edge(const GenModel& g, const ConvArgs& a, const float* MB, const float* Hl,
                          float* HB, double4* GRAD, double* vir_part, cudaStream_t s, bool hbar = true);

// three-body stage (potential.cpp:664-741, 850-961), slot conventions of
// the width-generic kernels; W3 / W3^T per bond on tcgen05
int wide_tb_grid(int64_t n);  // 9-double virial records of launch_wide_tb_backward
void launch_wide_tb_t(const GenModel& g, const BondArgs& a, float* TT, cudaStream_t s);
void launch_wide_tb_forward(const GenModel& g, const BondArgs& a, const float* TT, float* TP, float* TH3,
                            cudaStream_t s);
void launch_wide_tb_inject(const GenModel& g, const BondArgs& a, const float* TP, float* H, float* TH4,
                           cudaStream_t s);
void launch_wide_tb_bwd_q(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                          const float* HB, const float* TH4, float* QB, cudaStream_t s);
void launch_wide_tb_backward(const GenModel& g, const BondArgs& a, const float* QB, const float* TH3,
                             const float* TT, float* SMR, float4* VIN, float4* VOUT, double* vir_part,
                             cudaStream_t s);

}  // namespace gmd
