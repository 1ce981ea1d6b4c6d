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


// ---------------------------------------------------------------------------
// One rank per GPU: bond halo plan (SURVEY 8e "bond-feature exchange").
// A bond b = (w -> u) with u owned here and w owned by rank j needs the rows
// (t', v_bar) its reverse bond (u -> w) gets at center w on rank j.  Receive
// rows: per j, the bonds b in (u, row) order.  Send rows for rank j: per
// halo atom x of FROM_r[j] (ascending id), the slots c = (x -> w) at owned
// centers w, sorted by (w, -image) -- the order of x's row on rank j.
// ---------------------------------------------------------------------------
__global__ void k_bond_halo_flag(int64_t nb, const int32_t* __restrict__ bedge,
                                 const int32_t* __restrict__ esrc,
                                 const int32_t* __restrict__ owner, int j,
                                 int32_t* __restrict__ flag) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb) return;
    flag[b] = b < nb && owner[esrc[bedge[b]]] == j;
}

__global__ void k_bond_halo_assign(int64_t nb, const int32_t* __restrict__ bedge,
                                   const int32_t* __restrict__ esrc,
                                   const int32_t* __restrict__ owner, int j,
                                   const int32_t* __restrict__ pos, int32_t base,
                                   int32_t* __restrict__ brev) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    if (owner[esrc[bedge[b]]] == j) brev[b] = base + pos[b];
}

__global__ void k_bond_center(int64_t n, const int32_t* __restrict__ nodes,
                              const int32_t* __restrict__ brow, int32_t* __restrict__ bcen) {
    const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k >= n) return;
    const int w = nodes[k];
    for (int b = brow[w] + (threadIdx.x & 31); b < brow[w + 1]; b += 32) bcen[b] = w;
}

__global__ void k_bond_send_count(int64_t nb, const int32_t* __restrict__ bedge,
                                  const int32_t* __restrict__ esrc,
                                  const int32_t* __restrict__ owner, int r,
                                  const int32_t* __restrict__ crow, int32_t from0,
                                  int32_t* __restrict__ cnt) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int x = esrc[bedge[b]];
    if (owner[x] != r) atomicAdd(&cnt[crow[x] - from0], 1);
}

__global__ void k_bond_send_fill(int64_t nb, const int32_t* __restrict__ bedge,
                                 const int32_t* __restrict__ esrc,
                                 const int32_t* __restrict__ owner, int r,
                                 const int32_t* __restrict__ crow, int32_t from0,
                                 const int32_t* __restrict__ offs, int32_t* __restrict__ fill,
                                 int32_t* __restrict__ xs) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int x = esrc[bedge[b]];
    if (owner[x] != r) {
        const int row = crow[x] - from0;
        xs[offs[row] + atomicAdd(&fill[row], 1)] = (int32_t)b;
    }
}

__device__ __forceinline__ unsigned long long send_key(int b, const int32_t* bcen,
                                                       const int32_t* bedge,
                                                       const uint32_t* img) {
    int o0, o1, o2;
    unpack_img(img[bedge[b]], o0, o1, o2);  // image of (x -> w); rank j sees -o
    return ((unsigned long long)(uint32_t)bcen[b] << 30) |
           ((unsigned long long)(512 - o0) << 20) | ((unsigned long long)(512 - o1) << 10) |
           (unsigned long long)(512 - o2);
}

__global__ void k_bond_send_sort(int32_t nrows, const int32_t* __restrict__ offs,
                                 int32_t* __restrict__ xs, const int32_t* __restrict__ bcen,
                                 const int32_t* __restrict__ bedge,
                                 const uint32_t* __restrict__ img) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    const int a0 = offs[i], a1 = offs[i + 1];
    for (int t = a0 + 1; t < a1; ++t) {  // insertion sort (<= 64 bonds per atom)
        const int b = xs[t];
        const unsigned long long kb = send_key(b, bcen, bedge, img);
        int u = t - 1;
        while (u >= a0 && send_key(xs[u], bcen, bedge, img) > kb) {
            xs[u + 1] = xs[u];
            --u;
        }
        xs[u + 1] = b;
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

void launch_bond_halo_flag(int64_t nb, const int32_t* bedge, const int32_t* esrc,
                           const int32_t* owner, int j, int32_t* flag, cudaStream_t s) {
    k_bond_halo_flag<<<div_up(nb + 1, 256), 256, 0, s>>>(nb, bedge, esrc, owner, j, flag);
    GMD_LAUNCH_CHECK();
}

void launch_bond_halo_assign(int64_t nb, const int32_t* bedge, const int32_t* esrc,
                             const int32_t* owner, int j, const int32_t* pos, int32_t base,
                             int32_t* brev, cudaStream_t s) {
    if (nb == 0) return;
    k_bond_halo_assign<<<div_up(nb, 256), 256, 0, s>>>(nb, bedge, esrc, owner, j, pos, base, brev);
    GMD_LAUNCH_CHECK();
}

void launch_bond_send_plan(int64_t n_own, const int32_t* nodes, const int32_t* brow, int64_t nb,
                           const int32_t* bedge, const int32_t* esrc, const uint32_t* img,
                           const int32_t* owner, int r, const int32_t* crow, int32_t from0,
                           int phase, const int32_t* offs, int32_t* cnt_or_fill, int32_t* bcen,
                           int32_t* xs, int32_t nrows, cudaStream_t s) {
    if (phase == 0) {  // count per FROM row
        if (n_own > 0) {
            k_bond_center<<<div_up(n_own, 8), 256, 0, s>>>(n_own, nodes, brow, bcen);
            GMD_LAUNCH_CHECK();
        }
        if (nb > 0) {
            k_bond_send_count<<<div_up(nb, 256), 256, 0, s>>>(nb, bedge, esrc, owner, r, crow,
                                                              from0, cnt_or_fill);
            GMD_LAUNCH_CHECK();
        }
    } else {  // fill + per-row sort
        if (nb > 0) {
            k_bond_send_fill<<<div_up(nb, 256), 256, 0, s>>>(nb, bedge, esrc, owner, r, crow, from0,
                                                             offs, cnt_or_fill, xs);
            GMD_LAUNCH_CHECK();
        }
        if (nrows > 0) {
            k_bond_send_sort<<<div_up(nrows, 128), 128, 0, s>>>(nrows, offs, xs, bcen, bedge, img);
            GMD_LAUNCH_CHECK();
        }
    }
}

}  // namespace gmd
