// Device side of the reference's free builder API (see gmd_builders.cuh).
#include "gmd_builders.cuh"
#include "gmd_graph.cuh"

namespace gmd {
namespace {

__global__ void k_graph_import(int64_t ne, const int32_t* __restrict__ off3,
                               const double* __restrict__ dist, double bond_bound,
                               uint32_t* __restrict__ img, uint8_t* __restrict__ ebond,
                               int32_t* __restrict__ flags) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int o0 = off3[3 * e], o1 = off3[3 * e + 1], o2 = off3[3 * e + 2];
    // +-511: an offset and its negation both pack (the reverse-pair key)
    if (abs(o0) >= kImgBias || abs(o1) >= kImgBias || abs(o2) >= kImgBias)
        atomicOr(&flags[1], kErrImgRange);
    img[e] = pack_img(o0, o1, o2);
    // collect_bonds (linegraph.cpp:34-35): keep iff !(distance > r + tau)
    if (ebond) ebond[e] = (bond_bound >= 0.0 && !(dist[e] > bond_bound)) ? 1 : 0;
}

__global__ void k_row_bond_count(const int32_t* __restrict__ row, const uint8_t* __restrict__ ebond,
                                 int64_t n, int32_t* __restrict__ bcnt) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int c = 0;
    for (int e = row[v]; e < row[v + 1]; ++e) c += ebond[e];
    bcnt[v] = c;
}

__global__ void k_closure_init(const int32_t* __restrict__ owner, int64_t n,
                               unsigned long long* __restrict__ mask) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) mask[v] = 1ull << owner[v];
}

__global__ void k_closure_hop(const int32_t* __restrict__ row, const int32_t* __restrict__ src,
                              int64_t n, const unsigned long long* __restrict__ in,
                              unsigned long long* __restrict__ out) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    unsigned long long m = in[v];
    for (int e = row[v]; e < row[v + 1]; ++e) m |= in[src[e]];  // in_set[src] -> next[dst]
    out[v] = m;
}

__global__ void k_bond_tables(int64_t nb, const int32_t* __restrict__ bedge,
                              const int32_t* __restrict__ edst, const int32_t* __restrict__ src,
                              const unsigned long long* __restrict__ mask,
                              unsigned long long* __restrict__ bmask) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int e = bedge[b];
    bmask[b] = mask[src[e]] & mask[edst[e]];
}

// the reference's Vec3 arithmetic, unfused, in its operand order
__device__ __forceinline__ void raw_vector(const BruteNL& b, const double* pos, int j, int i, int o0,
                                           int o1, int o2, double vr[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        // lattice[0] * off0 + lattice[1] * off1 + lattice[2] * off2
        const double sh = __dadd_rn(__dadd_rn(__dmul_rn(b.L[c], (double)o0), __dmul_rn(b.L[3 + c], (double)o1)),
                                    __dmul_rn(b.L[6 + c], (double)o2));
        vr[c] = __dadd_rn(__dsub_rn(pos[3 * j + c], pos[3 * i + c]), sh);
    }
}

__device__ __forceinline__ double norm2_rn(const double v[3]) {
    return __dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])), __dmul_rn(v[2], v[2]));
}

__global__ void k_brute_nl(const BruteNL b, int64_t n, const double* __restrict__ pos,
                           const int32_t* __restrict__ cell, int32_t* __restrict__ cnt,
                           const int32_t* __restrict__ rowoff, int32_t* __restrict__ out_src,
                           int32_t* __restrict__ out_off) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    int mine = 0, written = 0;
    for (int64_t jb = 0; jb < n; jb += 32) {
        const int64_t j = jb + lane;
        for (int nx = -b.span[0]; nx <= b.span[0]; ++nx)
            for (int ny = -b.span[1]; ny <= b.span[1]; ++ny)
                for (int nz = -b.span[2]; nz <= b.span[2]; ++nz) {
                    bool hit = false;
                    int o0 = 0, o1 = 0, o2 = 0;
                    if (j < n) {
                        o0 = nx - cell[3 * j] + cell[3 * i];
                        o1 = ny - cell[3 * j + 1] + cell[3 * i + 1];
                        o2 = nz - cell[3 * j + 2] + cell[3 * i + 2];
                        double vr[3];
                        raw_vector(b, pos, (int)j, (int)i, o0, o1, o2, vr);
                        const double d2 = norm2_rn(vr);
                        hit = !(d2 > b.cutoff2) && d2 != 0.0;
                    }
                    if (!out_src) {
                        mine += hit;
                        continue;
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, hit);
                    if (hit) {
                        const int k = rowoff[i] + written + __popc(m & ((1u << lane) - 1u));
                        out_src[k] = (int32_t)j;
                        out_off[3 * k] = o0;
                        out_off[3 * k + 1] = o1;
                        out_off[3 * k + 2] = o2;
                    }
                    written += __popc(m);
                }
    }
    if (!out_src) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        if (lane == 0) cnt[i] = mine;
    }
}

__global__ void k_edge_geometry(const BruteNL b, int64_t ne, const double* __restrict__ pos,
                                const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                const int32_t* __restrict__ off, double* __restrict__ dist,
                                double* __restrict__ vec) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    double vr[3];
    raw_vector(b, pos, src[e], dst[e], off[3 * e], off[3 * e + 1], off[3 * e + 2], vr);
    dist[e] = __dsqrt_rn(norm2_rn(vr));
    vec[3 * e] = vr[0];
    vec[3 * e + 1] = vr[1];
    vec[3 * e + 2] = vr[2];
}

__global__ void k_brute_line(int64_t n, const int32_t* __restrict__ in_row,
                             const int32_t* __restrict__ in_bonds, const int32_t* __restrict__ out_row,
                             const int32_t* __restrict__ out_bonds, const int32_t* __restrict__ bedge,
                             const int32_t* __restrict__ src, const int32_t* __restrict__ edst,
                             const uint32_t* __restrict__ img, int32_t* __restrict__ cnt,
                             const int32_t* __restrict__ off, int32_t* __restrict__ pairs) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    int k = 0;
    for (int a = in_row[u]; a < in_row[u + 1]; ++a) {
        const int e = bedge[in_bonds[a]];  // e: (x -> u)
        int o0, o1, o2;
        unpack_img(img[e], o0, o1, o2);
        const uint32_t rev = pack_img(-o0, -o1, -o2);
        for (int c = out_row[u]; c < out_row[u + 1]; ++c) {
            const int ep = bedge[out_bonds[c]];  // e': (u -> y)
            // is_reverse_pair (linegraph.cpp:16-21)
            if (edst[ep] == src[e] && src[ep] == edst[e] && img[ep] == rev) continue;
            if (pairs) {
                pairs[2 * (off[u] + k)] = e;
                pairs[2 * (off[u] + k) + 1] = ep;
            }
            ++k;
        }
    }
    if (!pairs) cnt[u] = k;
}

}  // namespace

void launch_graph_import(int64_t ne, const int32_t* off3, const double* dist, double bond_bound,
                         uint32_t* img, uint8_t* ebond, int32_t* flags, cudaStream_t s) {
    if (ne <= 0) return;
    k_graph_import<<<div_up(ne, 256), 256, 0, s>>>(ne, off3, dist, bond_bound, img, ebond, flags);
    GMD_LAUNCH_CHECK();
}

void launch_row_bond_count(const int32_t* row, const uint8_t* ebond, int64_t n, int32_t* bcnt,
                           cudaStream_t s) {
    k_row_bond_count<<<div_up(n, 256), 256, 0, s>>>(row, ebond, n, bcnt);
    GMD_LAUNCH_CHECK();
}

void launch_closure_init(const int32_t* owner, int64_t n, unsigned long long* mask, cudaStream_t s) {
    k_closure_init<<<div_up(n, 256), 256, 0, s>>>(owner, n, mask);
    GMD_LAUNCH_CHECK();
}

void launch_closure_hop(const int32_t* row, const int32_t* src, int64_t n,
                        const unsigned long long* in, unsigned long long* out, cudaStream_t s) {
    k_closure_hop<<<div_up(n, 256), 256, 0, s>>>(row, src, n, in, out);
    GMD_LAUNCH_CHECK();
}

void launch_bond_tables(int64_t nb, const int32_t* bedge, const int32_t* edst, const int32_t* src,
                        const unsigned long long* mask, unsigned long long* bmask, cudaStream_t s) {
    if (nb <= 0) return;
    k_bond_tables<<<div_up(nb, 256), 256, 0, s>>>(nb, bedge, edst, src, mask, bmask);
    GMD_LAUNCH_CHECK();
}

void launch_brute_nl(const BruteNL& b, int64_t n, const double* pos, const int32_t* cell,
                     int32_t* cnt, const int32_t* rowoff, int32_t* out_src, int32_t* out_off,
                     cudaStream_t s) {
    k_brute_nl<<<div_up(n * 32, 256), 256, 0, s>>>(b, n, pos, cell, cnt, rowoff, out_src, out_off);
    GMD_LAUNCH_CHECK();
}

void launch_edge_geometry(const BruteNL& b, int64_t ne, const double* pos, const int32_t* src,
                          const int32_t* dst, const int32_t* off, double* dist, double* vec,
                          cudaStream_t s) {
    if (ne <= 0) return;
    k_edge_geometry<<<div_up(ne, 256), 256, 0, s>>>(b, ne, pos, src, dst, off, dist, vec);
    GMD_LAUNCH_CHECK();
}

void launch_brute_line(int64_t n, const int32_t* in_row, const int32_t* in_bonds,
                       const int32_t* out_row, const int32_t* out_bonds, const int32_t* bedge,
                       const int32_t* src, const int32_t* edst, const uint32_t* img, int32_t* cnt,
                       const int32_t* off, int32_t* pairs, cudaStream_t s) {
    k_brute_line<<<div_up(n, 128), 128, 0, s>>>(n, in_row, in_bonds, out_row, out_bonds, bedge, src,
                                                 edst, img, cnt, off, pairs);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
