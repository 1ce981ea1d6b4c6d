// Cell-list periodic radius graph, bit-exact with the reference's
// build_neighbor_list (proj/src/neighborlist.cpp:108-197).
//
// Layout: atoms are counting-sorted into fractional-space bins (SoA copies
// of wrapped/raw positions and cell offsets, so candidate loads coalesce);
// one CTA per destination bin stages the bin's destination atoms in shared
// memory and streams the (2s+1)^3 stencil bins' atoms through registers, 32
// candidates per warp, testing each against every destination (broadcast
// from shared memory).  Every fp64 decision uses unfused __dmul_rn/__dadd_rn
// in the reference's operand order.  Two passes: count
// (-> CSR row offsets) and fill (per-destination warp bitonic sort by
// (src, image) so rows come out in canonical order, neighborlist.cpp:21-24).
#include "gmd_graph.cuh"

namespace gmd {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSCap = 128;  // stencil cells per batch held in shared memory

__device__ __forceinline__ void wrap_one(const Geom& g, const double* __restrict__ pos, int64_t i,
                                         int c[3], double fw[3]) {
    const double px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
    // fractional() = inv.rowvec_mul(r) (system.cpp:79-85)
    d3 f = rowvec_rn(g.inv, px, py, pz);
    double fr[3] = {f.x, f.y, f.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // wrap_for_search (neighborlist.cpp:42-50)
        double fl = floor(fr[k]);
        c[k] = (int)fl;
        double w = sub_rn(fr[k], fl);
        if (w >= 1.0) {
            w = 0.0;
            c[k] += 1;
        }
        fw[k] = w;
    }
}

__device__ __forceinline__ int64_t bin_of(const Geom& g, const double fw[3], int b[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // neighborlist.cpp:128-134
        int v = (int)mul_rn(fw[k], (double)g.bins[k]);
        b[k] = v < g.bins[k] - 1 ? v : g.bins[k] - 1;
    }
    return ((int64_t)b[0] * g.bins[1] + b[1]) * g.bins[2] + b[2];
}

__global__ void k_wrap(const Geom g, int64_t n, const double* __restrict__ pos,
                       int32_t* __restrict__ cell, double* __restrict__ fw_axis,
                       int32_t* __restrict__ bin, int32_t* __restrict__ bin_cnt) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int c[3], b[3];
    double fw[3];
    wrap_one(g, pos, i, c, fw);
    cell[3 * i] = c[0];
    cell[3 * i + 1] = c[1];
    cell[3 * i + 2] = c[2];
    fw_axis[i] = fw[g.axis];
    int64_t bi = bin_of(g, fw, b);
    bin[i] = (int32_t)bi;
    atomicAdd(&bin_cnt[bi], 1);
}

// Scatter atoms into bin order.  Order inside a bin is arbitrary (atomic
// slot); every output is sorted afterwards so it never leaks into results.
__global__ void k_bin_scatter(const Geom g, int64_t n, const double* __restrict__ pos,
                              const int32_t* __restrict__ cell, const int32_t* __restrict__ bin,
                              const int32_t* __restrict__ bin_start, int32_t* __restrict__ fill,
                              int32_t* __restrict__ s_id, double* __restrict__ s_w,
                              double* __restrict__ s_p, int32_t* __restrict__ s_c) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int c[3];
    double fw[3];
    wrap_one(g, pos, i, c, fw);
    d3 w = rowvec_rn(g.L, fw[0], fw[1], fw[2]);  // neighborlist.cpp:55-56
    int b = bin[i];
    int slot = bin_start[b] + atomicAdd(&fill[b], 1);
    s_id[slot] = (int32_t)i;
    s_w[slot] = w.x;
    s_w[n + slot] = w.y;
    s_w[2 * n + slot] = w.z;
    s_p[slot] = pos[3 * i];
    s_p[n + slot] = pos[3 * i + 1];
    s_p[2 * n + slot] = pos[3 * i + 2];
    s_c[slot] = cell[3 * i];
    s_c[n + slot] = cell[3 * i + 1];
    s_c[2 * n + slot] = cell[3 * i + 2];
}

struct NLSmem {
    int sc_bin[kSCap];
    int sc_pre[kSCap + 1];
    int sc_q[kSCap][3];
    double sc_shift[kSCap][3];
};

__device__ __forceinline__ uint32_t qcode(int qx, int qy, int qz) {
    return ((uint32_t)(qx + 128) << 16) | ((uint32_t)(qy + 128) << 8) | (uint32_t)(qz + 128);
}

// One CTA per destination bin.  FILL=false counts edges per destination,
// FILL=true collects (src, image) keys, sorts them and writes the CSR rows.
template <bool FILL>
__global__ void __launch_bounds__(kThreads) k_nl(
    const Geom g, int64_t nbins, int64_t n, int group, int cap,
    const int32_t* __restrict__ bin_start, const int32_t* __restrict__ s_id,
    const double* __restrict__ s_w, const double* __restrict__ s_p,
    const int32_t* __restrict__ s_c, const double* __restrict__ pos,
    const int32_t* __restrict__ cell, int32_t* __restrict__ deg, int32_t* __restrict__ flags,
    const int32_t* __restrict__ row, int32_t* __restrict__ e_src, uint32_t* __restrict__ e_img,
    float4* __restrict__ e_vd, uint8_t* __restrict__ e_bond, int32_t* __restrict__ bcnt) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    NLSmem& S = *reinterpret_cast<NLSmem*>(smem_raw);
    double* d_w = reinterpret_cast<double*>(smem_raw + sizeof(NLSmem));  // group x 3
    double* d_p = d_w + 3 * group;                                         // group x 3
    int* d_c = reinterpret_cast<int*>(d_p + 3 * group);                     // group x 3
    int* d_id = d_c + 3 * group;                                            // group
    int* d_cnt = d_id + group;                                              // group
    unsigned long long* keys =
        reinterpret_cast<unsigned long long*>(smem_raw + sizeof(NLSmem) +
                                              (((size_t)group * (48 + 20) + 15) & ~(size_t)15));

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sx = 2 * g.sten[0] + 1, sy = 2 * g.sten[1] + 1, sz = 2 * g.sten[2] + 1;
    const int ncell = sx * sy * sz;

    for (int64_t bb = blockIdx.x; bb < nbins; bb += gridDim.x) {
        const int b0 = bin_start[bb], b1 = bin_start[bb + 1];
        if (b1 == b0) continue;  // uniform across the CTA
        const int bz = (int)(bb % g.bins[2]);
        const int by = (int)((bb / g.bins[2]) % g.bins[1]);
        const int bx = (int)(bb / ((int64_t)g.bins[2] * g.bins[1]));

        for (int gbase = b0; gbase < b1; gbase += group) {
            const int nd = min(group, b1 - gbase);
            __syncthreads();
            for (int t = threadIdx.x; t < nd; t += kThreads) {
                int slot = gbase + t;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    d_w[3 * t + k] = s_w[k * n + slot];
                    d_p[3 * t + k] = s_p[k * n + slot];
                    d_c[3 * t + k] = s_c[k * n + slot];
                }
                d_id[t] = s_id[slot];
                d_cnt[t] = 0;
            }
            for (int cbase = 0; cbase < ncell; cbase += kSCap) {
                const int nc = min(kSCap, ncell - cbase);
                __syncthreads();
                // stencil batch table: wrapped bin, image q, shift, candidate prefix
                for (int ci = threadIdx.x; ci < nc; ci += kThreads) {
                    int c = cbase + ci;
                    int dz = c % sz - g.sten[2];
                    int dy = (c / sz) % sy - g.sten[1];
                    int dx = c / (sz * sy) - g.sten[0];
                    int cc[3] = {bx + dx, by + dy, bz + dz};
                    int q[3], cw[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {  // neighborlist.cpp:165-170
                        int nb = g.bins[k];
                        q[k] = cc[k] >= 0 ? cc[k] / nb : -((-cc[k] + nb - 1) / nb);
                        cw[k] = cc[k] - q[k] * nb;
                        S.sc_q[ci][k] = q[k];
                    }
                    // shift = L0*q0 + L1*q1 + L2*q2 (neighborlist.cpp:171-173)
                    d3 sh = rowvec_rn(g.L, (double)q[0], (double)q[1], (double)q[2]);
                    S.sc_shift[ci][0] = sh.x;
                    S.sc_shift[ci][1] = sh.y;
                    S.sc_shift[ci][2] = sh.z;
                    int64_t wb = ((int64_t)cw[0] * g.bins[1] + cw[1]) * g.bins[2] + cw[2];
                    S.sc_bin[ci] = (int)wb;
                    S.sc_pre[ci + 1] = bin_start[wb + 1] - bin_start[wb];
                    if (q[0] < -128 || q[0] > 127 || q[1] < -128 || q[1] > 127 || q[2] < -128 ||
                        q[2] > 127)
                        atomicOr(&flags[1], kErrQRange);
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    int acc = 0;
                    S.sc_pre[0] = 0;
                    for (int ci = 0; ci < nc; ++ci) {
                        acc += S.sc_pre[ci + 1];
                        S.sc_pre[ci + 1] = acc;
                    }
                }
                __syncthreads();
                const int total = S.sc_pre[nc];
                for (int kb = warp * 32; kb < total; kb += kThreads) {
                    const int k = kb + lane;
                    const bool valid = k < total;
                    double cx = 0, cy = 0, cz = 0, px = 0, py = 0, pz = 0;
                    int nx = 0, ny = 0, nz = 0, jid = 0;
                    uint32_t qc = 0;
                    if (valid) {
                        int lo = 0, hi = nc - 1;  // last cell with pre <= k
                        while (lo < hi) {
                            int mid = (lo + hi + 1) >> 1;
                            if (S.sc_pre[mid] <= k) lo = mid; else hi = mid - 1;
                        }
                        const int ci = lo;
                        const int slot = bin_start[S.sc_bin[ci]] + (k - S.sc_pre[ci]);
                        // candidate = wrapped_j + shift (neighborlist.cpp:176)
                        cx = add_rn(s_w[slot], S.sc_shift[ci][0]);
                        cy = add_rn(s_w[n + slot], S.sc_shift[ci][1]);
                        cz = add_rn(s_w[2 * n + slot], S.sc_shift[ci][2]);
                        px = s_p[slot];
                        py = s_p[n + slot];
                        pz = s_p[2 * n + slot];
                        nx = S.sc_q[ci][0] - s_c[slot];
                        ny = S.sc_q[ci][1] - s_c[n + slot];
                        nz = S.sc_q[ci][2] - s_c[2 * n + slot];
                        jid = s_id[slot];
                        qc = qcode(S.sc_q[ci][0], S.sc_q[ci][1], S.sc_q[ci][2]);
                    }
                    for (int t = 0; t < nd; ++t) {
                        bool hit = false;
                        if (valid) {
                            // prefilter on wrapped positions (neighborlist.cpp:176-177)
                            d3 v = {sub_rn(cx, d_w[3 * t]), sub_rn(cy, d_w[3 * t + 1]),
                                    sub_rn(cz, d_w[3 * t + 2])};
                            if (!(dot_rn(v, v) > g.pre2)) {
                                // exact test through raw positions (:178-191)
                                int o0 = nx + d_c[3 * t], o1 = ny + d_c[3 * t + 1],
                                    o2 = nz + d_c[3 * t + 2];
                                d3 raw = rowvec_rn(g.L, (double)o0, (double)o1, (double)o2);
                                d3 vr = {add_rn(sub_rn(px, d_p[3 * t]), raw.x),
                                         add_rn(sub_rn(py, d_p[3 * t + 1]), raw.y),
                                         add_rn(sub_rn(pz, d_p[3 * t + 2]), raw.z)};
                                double d2 = dot_rn(vr, vr);
                                hit = !(d2 > g.cutoff2) && d2 != 0.0;
                            }
                        }
                        unsigned m = __ballot_sync(0xffffffffu, hit);
                        if (m == 0) continue;
                        if (!FILL) {
                            if (lane == 0) atomicAdd(&d_cnt[t], __popc(m));
                        } else {
                            int base = 0;
                            if (lane == 0) base = atomicAdd(&d_cnt[t], __popc(m));
                            base = __shfl_sync(0xffffffffu, base, 0);
                            if (hit) {
                                int pos_k = base + __popc(m & ((1u << lane) - 1u));
                                if (pos_k < cap)
                                    keys[(size_t)t * cap + pos_k] =
                                        ((unsigned long long)(uint32_t)jid << 24) | qc;
                                else
                                    atomicOr(&flags[1], kErrCap);
                            }
                        }
                    }
                }
            }
            __syncthreads();
            if (!FILL) {
                for (int t = threadIdx.x; t < nd; t += kThreads) {
                    deg[d_id[t]] = d_cnt[t];
                    atomicMax(&flags[0], d_cnt[t]);
                }
            } else {
                for (int t = warp; t < nd; t += kWarps) {
                    const int cnt = min(d_cnt[t], cap);
                    unsigned long long* kk = keys + (size_t)t * cap;
                    int P = 1;
                    while (P < cnt) P <<= 1;
                    for (int k = cnt + lane; k < P; k += 32) kk[k] = ~0ull;
                    __syncwarp();
                    for (int sz2 = 2; sz2 <= P; sz2 <<= 1)
                        for (int j = sz2 >> 1; j > 0; j >>= 1) {
                            for (int i = lane; i < P; i += 32) {
                                int ixj = i ^ j;
                                if (ixj > i) {
                                    unsigned long long a = kk[i], c2 = kk[ixj];
                                    bool up = (i & sz2) == 0;
                                    if ((a > c2) == up) {
                                        kk[i] = c2;
                                        kk[ixj] = a;
                                    }
                                }
                            }
                            __syncwarp();
                        }
                    const int did = d_id[t];
                    const int e0 = row[did];
                    int nb = 0;
                    for (int k = lane; k < ((cnt + 31) & ~31); k += 32) {
                        bool isb = false;
                        if (k < cnt) {
                            unsigned long long key = kk[k];
                            int j = (int)(key >> 24);
                            int q0 = (int)((key >> 16) & 255) - 128;
                            int q1 = (int)((key >> 8) & 255) - 128;
                            int q2 = (int)(key & 255) - 128;
                            // off = image - cell_of[j] + cell_of[i] (neighborlist.cpp:179-180)
                            int o0 = q0 - cell[3 * j] + d_c[3 * t];
                            int o1 = q1 - cell[3 * j + 1] + d_c[3 * t + 1];
                            int o2 = q2 - cell[3 * j + 2] + d_c[3 * t + 2];
                            if (!img_in_range(o0) || !img_in_range(o1) || !img_in_range(o2))
                                atomicOr(&flags[1], kErrImgRange);
                            d3 raw = rowvec_rn(g.L, (double)o0, (double)o1, (double)o2);
                            d3 vr = {add_rn(sub_rn(pos[3 * j], d_p[3 * t]), raw.x),
                                     add_rn(sub_rn(pos[3 * j + 1], d_p[3 * t + 1]), raw.y),
                                     add_rn(sub_rn(pos[3 * j + 2], d_p[3 * t + 2]), raw.z)};
                            double dd = __dsqrt_rn(dot_rn(vr, vr));
                            const int e = e0 + k;
                            e_src[e] = j;
                            e_img[e] = pack_img(o0, o1, o2);
                            e_vd[e] = make_float4((float)vr.x, (float)vr.y, (float)vr.z, (float)dd);
                            isb = g.bond_bound >= 0.0 && !(dd > g.bond_bound);
                            e_bond[e] = isb ? 1 : 0;
                        }
                        nb += __popc(__ballot_sync(0xffffffffu, isb));
                    }
                    if (lane == 0) bcnt[did] = nb;
                }
            }
        }
    }
}

__global__ void k_minmax_proj(const double* __restrict__ pos, int64_t n, double dx, double dy,
                              double dz, unsigned long long* out) {
    // order-preserving u64 encoding of doubles so atomicMin/Max are exact
    double lo = 1.7976931348623157e308, hi = -1.7976931348623157e308;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        d3 r = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        double t = dot_rn(r, d3{dx, dy, dz});  // r.dot(dir) (system.cpp:258)
        lo = t < lo ? t : lo;
        hi = t > hi ? t : hi;
    }
    auto enc = [](double v) {
        unsigned long long u = (unsigned long long)__double_as_longlong(v);
        return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
    };
    atomicMin(&out[0], enc(lo));
    atomicMax(&out[1], enc(hi));
}

__global__ void k_shift(double* pos, int64_t n, double ax, double ay, double az) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    pos[3 * i] = add_rn(pos[3 * i], ax);
    pos[3 * i + 1] = add_rn(pos[3 * i + 1], ay);
    pos[3 * i + 2] = add_rn(pos[3 * i + 2], az);
}

__global__ void k_edge_dst(const int32_t* __restrict__ row, int64_t n, int32_t* __restrict__ edst) {
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (i >= n) return;
    for (int e = row[i] + (threadIdx.x & 31); e < row[i + 1]; e += 32) edst[e] = (int32_t)i;
}

__global__ void k_export_graph(const Geom g, const double* __restrict__ pos, int64_t ne,
                               const int32_t* __restrict__ edst, const int32_t* __restrict__ src,
                               const uint32_t* __restrict__ img, int64_t* o_src, int64_t* o_dst,
                               int32_t* o_off, double* o_dist, double* o_vec) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    int i = edst[e], j = src[e];
    int o0, o1, o2;
    unpack_img(img[e], o0, o1, o2);
    d3 raw = rowvec_rn(g.L, (double)o0, (double)o1, (double)o2);
    d3 vr = {add_rn(sub_rn(pos[3 * j], pos[3 * i]), raw.x),
             add_rn(sub_rn(pos[3 * j + 1], pos[3 * i + 1]), raw.y),
             add_rn(sub_rn(pos[3 * j + 2], pos[3 * i + 2]), raw.z)};
    if (o_src) o_src[e] = j;
    if (o_dst) o_dst[e] = i;
    if (o_off) {
        o_off[3 * e] = o0;
        o_off[3 * e + 1] = o1;
        o_off[3 * e + 2] = o2;
    }
    if (o_dist) o_dist[e] = __dsqrt_rn(dot_rn(vr, vr));
    if (o_vec) {
        o_vec[3 * e] = vr.x;
        o_vec[3 * e + 1] = vr.y;
        o_vec[3 * e + 2] = vr.z;
    }
}


// bond list in edge order (BondSet::edge_of_bond, linegraph.cpp:25-43),
// grouped by destination: bedge[brow[v] + k] = k-th bond edge into v
__global__ void k_bond_edges(const int32_t* __restrict__ row, const uint8_t* __restrict__ ebond,
                             int64_t n, const int32_t* __restrict__ brow,
                             int32_t* __restrict__ bedge) {
    int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (v >= n) return;
    const int lane = threadIdx.x & 31;
    int base = brow[v];
    for (int eb = row[v]; eb < row[v + 1]; eb += 32) {
        int e = eb + lane;
        bool f = e < row[v + 1] && ebond[e];
        unsigned m = __ballot_sync(0xffffffffu, f);
        if (f) bedge[base + __popc(m & ((1u << lane) - 1u))] = e;
        base += __popc(m);
    }
}

// reverse bond: (w -> v, o) <-> (v -> w, -o), searched in row w which is
// sorted by (src, image) (linegraph.cpp:16-21 is_reverse_pair)
__global__ void k_bond_rev(int64_t n, const int32_t* __restrict__ row,
                           const int32_t* __restrict__ src, const uint32_t* __restrict__ img,
                           const uint8_t* __restrict__ ebond, const int32_t* __restrict__ brow,
                           const int32_t* __restrict__ bedge, int32_t* __restrict__ brev,
                           int32_t* __restrict__ flags) {
    int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (v >= n) return;
    for (int b = brow[v] + (threadIdx.x & 31); b < brow[v + 1]; b += 32) {
        const int e = bedge[b];
        const int w = src[e];
        int o0, o1, o2;
        unpack_img(img[e], o0, o1, o2);
        const uint32_t want = pack_img(-o0, -o1, -o2);
        int lo = row[w], hi = row[w + 1];
        while (lo < hi) {  // first edge of row w with src >= v
            int mid = (lo + hi) >> 1;
            if (src[mid] < v) lo = mid + 1; else hi = mid;
        }
        int er = -1;
        for (int x = lo; x < row[w + 1] && src[x] == v; ++x)
            if (img[x] == want) {
                er = x;
                break;
            }
        int id = -1;
        if (er >= 0 && ebond[er]) {
            id = brow[w];
            for (int x = row[w]; x < er; ++x) id += ebond[x];
        } else {
            atomicOr(&flags[1], 32);
        }
        brev[b] = id;
    }
}

size_t nl_smem(int group, int cap, bool fill) {
    size_t s = sizeof(NLSmem) + (((size_t)group * (48 + 20) + 15) & ~(size_t)15);
    if (fill) s += (size_t)group * cap * 8;
    return s;
}

int nl_grid(int64_t nbins) {
    int64_t g = nbins < 148 * 64 ? nbins : 148 * 64;
    return (int)(g > 0 ? g : 1);
}

}  // namespace

void launch_wrap(const Geom& g, int64_t n, NLBuffers& b, cudaStream_t s) {
    k_wrap<<<div_up(n, 256), 256, 0, s>>>(g, n, b.pos, b.cell, b.fw_axis, b.bin, b.bin_cnt);
    GMD_LAUNCH_CHECK();
}

void launch_bin_scatter(const Geom& g, int64_t n, NLBuffers& b, int32_t* fill, cudaStream_t s) {
    k_bin_scatter<<<div_up(n, 256), 256, 0, s>>>(g, n, b.pos, b.cell, b.bin, b.bin_start, fill,
                                                  b.s_id, b.s_w, b.s_p, b.s_c);
    GMD_LAUNCH_CHECK();
}

void launch_nl_count(const Geom& g, int64_t nbins, int64_t n, NLBuffers& b, cudaStream_t s) {
    const int group = 64;
    size_t sm = nl_smem(group, 0, false);
    k_nl<false><<<nl_grid(nbins), kThreads, sm, s>>>(
        g, nbins, n, group, 0, b.bin_start, b.s_id, b.s_w, b.s_p, b.s_c, b.pos, b.cell, b.deg,
        b.flags, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    GMD_LAUNCH_CHECK();
}

void launch_nl_fill(const Geom& g, int64_t nbins, int cap, NLBuffers& b, GraphDev& gd,
                    cudaStream_t s) {
    int group = 32;
    while (group > 1 && (size_t)group * cap * 8 > 96 * 1024) group >>= 1;
    size_t sm = nl_smem(group, cap, true);
    static bool attr_set = false;
    if (!attr_set) {
        GMD_CUDA(cudaFuncSetAttribute(k_nl<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
        attr_set = true;
    }
    k_nl<true><<<nl_grid(nbins), kThreads, sm, s>>>(
        g, nbins, gd.n, group, cap, b.bin_start, b.s_id, b.s_w, b.s_p, b.s_c, b.pos, b.cell,
        b.deg, b.flags, gd.row, gd.src, gd.img, gd.vd, gd.bond, b.bcnt);
    GMD_LAUNCH_CHECK();
}

void launch_minmax_proj(const double* pos, int64_t n, const double dir[3], double* out2,
                        cudaStream_t s) {
    unsigned long long* o = reinterpret_cast<unsigned long long*>(out2);
    unsigned long long init[2] = {~0ull, 0ull};
    GMD_CUDA(cudaMemcpyAsync(o, init, sizeof init, cudaMemcpyHostToDevice, s));
    k_minmax_proj<<<148, 256, 0, s>>>(pos, n, dir[0], dir[1], dir[2], o);
    GMD_LAUNCH_CHECK();
}

void launch_shift(double* pos, int64_t n, const double add[3], cudaStream_t s) {
    k_shift<<<div_up(n, 256), 256, 0, s>>>(pos, n, add[0], add[1], add[2]);
    GMD_LAUNCH_CHECK();
}

void launch_edge_dst(const int32_t* row, int64_t n, int32_t* edst, cudaStream_t s) {
    k_edge_dst<<<div_up(n, 8), 256, 0, s>>>(row, n, edst);
    GMD_LAUNCH_CHECK();
}

void launch_export_graph(const Geom& g, const double* pos, const GraphDev& gd,
                           const int32_t* edst, int64_t* src, int64_t* dst, int32_t* off,
                           double* dist, double* vec, cudaStream_t s) {
    if (gd.ne == 0) return;
    k_export_graph<<<div_up(gd.ne, 256), 256, 0, s>>>(g, pos, gd.ne, edst, gd.src, gd.img, src,
                                                       dst, off, dist, vec);
    GMD_LAUNCH_CHECK();
}


void launch_bond_edges(const int32_t* row, const uint8_t* ebond, int64_t n, const int32_t* brow,
                       int32_t* bedge, cudaStream_t s) {
    if (n == 0) return;
    k_bond_edges<<<div_up(n, 8), 256, 0, s>>>(row, ebond, n, brow, bedge);
    GMD_LAUNCH_CHECK();
}

void launch_bond_rev(int64_t n, const GraphDev& gd, const int32_t* brow, const int32_t* bedge,
                     int32_t* brev, int32_t* flags, cudaStream_t s) {
    if (n == 0) return;
    k_bond_rev<<<div_up(n, 8), 256, 0, s>>>(n, gd.row, gd.src, gd.img, gd.bond, brow, bedge, brev,
                                            flags);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
