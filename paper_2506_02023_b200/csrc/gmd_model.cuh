// Message passing, halo exchange and the hand-written backward of the toy
// invariant MLIP (proj/src/potential.cpp:19-78, 563-985) on the GPU.
#pragma once
#include "gmd_common.cuh"

namespace gmd {

constexpr int kMaxLayers = 8;
constexpr int kF = 16;  // feature width of the compiled kernels
constexpr int kK = 8;   // radial basis count of the compiled kernels
constexpr int kMaxBondsPerAtom = 64;

// fp32 copy of ToyPotentialParams (potential.hpp:15-41) in constant memory
struct ModelConst {
    float emb[119 * kF];
    float W[kMaxLayers][kF * kF];
    float b[kMaxLayers][kF];
    alignas(16) float P[kF * kK];   // f-major: (P[f][k], P[f][k+1]) pairs
    alignas(16) float PT[kK * kF];  // k-major: (P[f][k], P[f+1][k]) pairs
    alignas(16) float Pk[kF * kK];  // k * P[f][k] (derivative of the radial channel)
    alignas(16) float P3[kF * kK];
    alignas(16) float P3T[kK * kF];  // k-major: (P3[f][k], P3[f+1][k]) pairs
    alignas(16) float W3[kF * kF];   // rows f: (W3[f][g], W3[f][g+1]) pairs
    alignas(16) float W3T[kF * kF];  // W3T[g][f] = W3[f][g]
    alignas(16) float W4[kF * kF];
    alignas(16) float W4T[kF * kF];
    alignas(16) float B3[kF * kK];   // (W3 P3)[f][k], fp64 product rounded once: E = B3^T y
    float ro[kF];
    float rc, inv_rc, inv_sigma, mu_step;     // atom radial basis
    float a2, pi_rc;                          // sqrt(log2 e)/sigma, pi/rc
    float bx[kK];                             // mu_k sqrt(log2 e)/sigma
    float r3, inv_r3, inv_sigma3, mu_step3;   // three-body radial basis
    int L;
};

void upload_model(const ModelConst& m, cudaStream_t s);

// Row/edge views used by the kernels.  Node loops run over global ids
// [0, n) of owned atoms in ascending order; crow maps an id to its row in the
// (super-)layout of its owner partition (nullptr = identity); lsrc is the
// source row per edge.
struct ConvArgs {
    int64_t n;              // number of owned nodes processed
    const int32_t* nodes;   // their global ids, ascending (nullptr: 0..n-1)
    const int32_t* crow;
    const int32_t* row;
    const int32_t* lsrc;
    const float4* vd;  // (vx, vy, vz, d) per edge (backward)
    const float* d;    // d per edge (forward)
    int64_t k0 = 0;    // first node processed (launch_bwd_edge: nodes [k0, n))
    // conv kernels: first non-finite feature, atomicMin of (layer << 40 | row)
    // with row the node's layout row (crow) -- the reference's check_finite
    // order (potential.cpp:107-115; partitions ascending, layout order)
    unsigned long long* nonfinite = nullptr;
};

__device__ __forceinline__ void note_nonfinite(const ConvArgs& a, int layer, int64_t row, float h) {
    if (a.nonfinite && !isfinite(h))
        atomicMin(a.nonfinite, ((unsigned long long)layer << 40) | (unsigned long long)row);
}

int model_grid(int64_t n);  // fixed grid => deterministic reductions
int bwd_edge_grid(int64_t n);  // grid (= virial partial count) of launch_bwd_edge

// zs / zmask (optional): per-row species byte and the species presence mask
// for the layer-0 species-sum conv
void launch_embed(int64_t rows, const int32_t* node_array, const int32_t* Z, float* H0,
                  cudaStream_t s, uint8_t* zs = nullptr, unsigned* zmask = nullptr);
void launch_exchange(int64_t nx, const int32_t* xdst, const int32_t* xsrc, float* buf, int width,
                     cudaStream_t s);
// forward conv layer l: Hout[own] = Hin[own] + tanh(W_l m + b_l); TH_l = tanh(.)
// last layer additionally writes per-atom energies and per-CTA energy partials
// zs / zmask (layer 0 only, h0 = the embeddings): the species-sum form
void launch_conv(const ConvArgs& a, int layer, const float* Hin, float* Hout, float* TH,
                 double* per_atom, double* e_part, cudaStream_t s, const uint8_t* zs = nullptr,
                 const unsigned* zmask = nullptr);
// backward: MB[row(v)] = W_l^T (HB[v] * (1 - TH_l[v]^2)); init: HB := readout
// first (the first backward layer, replacing launch_init_hbar)
void launch_bwd_node(int64_t n, const int32_t* nodes, const int32_t* crow, int layer,
                     float* HB, const float* TH, float* MB, bool init, cudaStream_t s);
// backward edge pass (row form, no atomics): HB += gathered adjoints,
// GRAD += positional gradient, virial partials per CTA (6 doubles)
// vir_grp / grid: node-chunked launches (default kernel only) pass a fixed
// grid and a carry buffer of grid * bwd_edge_stride(grid) / ... per-group
// virial sums; with chunk starts k0 that are multiples of
// bwd_edge_stride(grid) every node meets the same CTA group in the same order
// as in one launch, so the virial (and everything else) is bitwise the same
// hbar = false: skip h_bar (the last backward layer, layer 0, whose h_bar is
// the embedding gradient -- no position dependence, never read)
// zs / zmask (layer 0, Hl = h0 = emb[Z]): source h rows from the species
// table instead of gathered rows (bitwise equal)
void launch_bwd_edge(const ConvArgs& a, const float* MB, const float* Hl, float* HB, double4* GRAD,
                     double* vir_part, cudaStream_t s, double* vir_grp = nullptr, int grid = 0,
                     bool hbar = true, const uint8_t* zs = nullptr, const unsigned* zmask = nullptr);
// the default kernel takes node ranges (a.k0 > 0); grid = bwd_edge_grid(n - k0)
bool bwd_edge_ranges();
// nodes per sweep of the default kernel's grid (node k -> group k mod stride)
int64_t bwd_edge_stride(int grid);

// the same pass with the radial contractions on tcgen05 (TMEM accumulator);
// tcgen05 backward edge pass over 16-edge chunk records (one per chunk of a
// node's in-edges): count per node -> exclusive scan -> fill + per-CTA ranges.
// grid = bwd_tc_grid(n) CTAs, vir_part holds grid x 6 doubles
int bwd_tc_grid(int64_t n);
void launch_chunk_count(const ConvArgs& a, int32_t* cnt, cudaStream_t s);  // n + 1 entries
void launch_chunk_fill(const ConvArgs& a, const int32_t* cstart, int4* tab, int grid,
                       int32_t* cta, cudaStream_t s);
void launch_bwd_edge_tc(const ConvArgs& a, const int4* ctab, const int32_t* ccta, int grid,
                        const float* MB, const float* Hl, float* HB, double4* GRAD,
                        double* vir_part, cudaStream_t s);

// three-body stage (global bond CSR by dst; slot = in-bond position)
struct BondArgs {
    int64_t n;              // centers this handle updates
    const int32_t* nodes;   // n: their global ids (one rank per GPU), null = 0..n-1
    const int32_t* crow;
    const int32_t* brow;    // n + 1
    const int32_t* bedge;   // B: edge id of bond
    const int32_t* brev;    // B: bond id of the reverse bond
    const int32_t* esrc;    // E: global source id per edge
    const float4* vd;       // E
};
// max_bonds: largest in-bond count of a center (sizes the per-group staging)
void launch_tb_forward(const BondArgs& a, float* TP, float* TH3, int32_t* flags, int max_bonds,
                       cudaStream_t s);
void launch_tb_inject(const BondArgs& a, const float* TP, float* H, float* TH4, cudaStream_t s);
void launch_tb_bwd_q(int64_t n, const int32_t* nodes, const int32_t* crow, const float* HB,
                     const float* TH4, float* QB, cudaStream_t s);  // QB by layout row
// max_bonds: largest in-bond count of a center (sizes the per-group staging)
void launch_tb_backward(const BondArgs& a, const float* QB, const float* TH3, float4* VIN,
                        float4* VOUT, double* vir_part, int max_bonds, cudaStream_t s);
void launch_tb_grad(const BondArgs& a, const float4* VIN, const float4* VOUT, double4* GRAD,
                    cudaStream_t s);

void launch_init_hbar(int64_t n, float* HB, cudaStream_t s);
void launch_forces_out(int64_t n, const int32_t* nodes, const double4* GRAD, double* forces,
                       float* forces32, cudaStream_t s);
// sum nparts consecutive records of width w into out[w] in fixed order
void launch_reduce_partials(const double* parts, int nparts, int w, double* out, cudaStream_t s);
// up to 3 partial sets [nparts[k] x w[k]] into consecutive columns of out
void launch_reduce_sets(int nsets, const double* const* parts, const int* nparts, const int* w,
                        double* out, cudaStream_t s);

}  // namespace gmd
