// Partitioned three-body line graph on the GPU (linegraph.cpp:67-171).
//
// The line graph is never materialized for the model (gmd_model.cu works per
// center atom on its in-bond list); these kernels build the reference's
// per-partition structures -- bond owners, bond requirement masks (and from
// them the bond PURE/TO/FROM layouts via the shared layout compaction), and
// the (e, e') line-edge list in (e', e) order -- for export and parity.
#include "gmd_common.cuh"

namespace gmd {
namespace {

__global__ void k_bond_owner(int64_t n, const int32_t* __restrict__ brow,
                             const int32_t* __restrict__ owner, int32_t* __restrict__ bown) {
    int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (v >= n) return;
    const int o = owner[v];
    for (int b = brow[v] + (threadIdx.x & 31); b < brow[v + 1]; b += 32) bown[b] = o;
}

// bond e (into s) is required by owner(e') for every line edge (e, e') whose
// owner differs (linegraph.cpp:95-105): e' = reverse of another in-bond of s
__global__ void k_bond_req(int64_t n, const int32_t* __restrict__ brow,
                           const int32_t* __restrict__ bedge, const int32_t* __restrict__ esrc,
                           const int32_t* __restrict__ owner,
                           unsigned long long* __restrict__ breq) {
    int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= n) return;
    const int b0 = brow[s], k = brow[s + 1] - b0, os = owner[s];
    for (int j = threadIdx.x & 31; j < k; j += 32) {
        unsigned long long m = 0ull;
        for (int o = 0; o < k; ++o) {
            if (o == j) continue;
            int ow = owner[esrc[bedge[b0 + o]]];
            if (ow != os) m |= 1ull << ow;
        }
        breq[b0 + j] = m;
    }
}

// line edges of e' = (w -> v): one per in-bond of w except rev(e')
__global__ void k_line_count(int64_t nb, const int32_t* __restrict__ bedge,
                             const int32_t* __restrict__ esrc, const int32_t* __restrict__ brow,
                             int32_t* __restrict__ cnt) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int w = esrc[bedge[b]];
    cnt[b] = brow[w + 1] - brow[w] - 1;
}

__global__ void k_line_fill(int64_t nb, const int32_t* __restrict__ bedge,
                            const int32_t* __restrict__ esrc, const int32_t* __restrict__ brow,
                            const int32_t* __restrict__ brev, const int32_t* __restrict__ lpos,
                            int32_t* __restrict__ pairs) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int w = esrc[bedge[b]];
    int pos = lpos[b];
    const int rb = brev[b];
    for (int e = brow[w]; e < brow[w + 1]; ++e) {
        if (e == rb) continue;
        pairs[2 * pos] = e;
        pairs[2 * pos + 1] = (int)b;
        ++pos;
    }
}

}  // namespace

void launch_bond_owner(int64_t n, const int32_t* brow, const int32_t* owner, int32_t* bown,
                       cudaStream_t s) {
    if (n == 0) return;
    k_bond_owner<<<div_up(n, 8), 256, 0, s>>>(n, brow, owner, bown);
    GMD_LAUNCH_CHECK();
}

void launch_bond_req(int64_t n, const int32_t* brow, const int32_t* bedge, const int32_t* esrc,
                     const int32_t* owner, unsigned long long* breq, cudaStream_t s) {
    if (n == 0) return;
    k_bond_req<<<div_up(n, 8), 256, 0, s>>>(n, brow, bedge, esrc, owner, breq);
    GMD_LAUNCH_CHECK();
}

void launch_line_count(int64_t nb, const int32_t* bedge, const int32_t* esrc, const int32_t* brow,
                       int32_t* cnt, cudaStream_t s) {
    if (nb == 0) return;
    k_line_count<<<div_up(nb, 256), 256, 0, s>>>(nb, bedge, esrc, brow, cnt);
    GMD_LAUNCH_CHECK();
}

void launch_line_fill(int64_t nb, const int32_t* bedge, const int32_t* esrc, const int32_t* brow,
                      const int32_t* brev, const int32_t* lpos, int32_t* pairs, cudaStream_t s) {
    if (nb == 0) return;
    k_line_fill<<<div_up(nb, 256), 256, 0, s>>>(nb, bedge, esrc, brow, brev, lpos, pairs);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
