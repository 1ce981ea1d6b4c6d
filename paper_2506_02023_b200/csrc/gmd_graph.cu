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
#include <algorithm>
#include <cstdlib>

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
                       int32_t* __restrict__ bin, int32_t* __restrict__ bin_cnt,
                       int32_t* __restrict__ flags, double4* __restrict__ pos4,
                       int4* __restrict__ cell4) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // max |coordinate| over the input (rounded up to fp32) -> flags[3]: the
    // search's fast-accept band is only sound while the wrapped and raw
    // vectors agree far below its rc * 1e-9 margin (launch_nl_search)
    float m = 0.f;
    if (i < n)
        m = fmaxf(fmaxf(__double2float_ru(fabs(pos[3 * i])), __double2float_ru(fabs(pos[3 * i + 1]))),
                  __double2float_ru(fabs(pos[3 * i + 2])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(&flags[3], __float_as_int(m));
    if (i >= n) return;
    int c[3], b[3];
    double fw[3];
    wrap_one(g, pos, i, c, fw);
    cell[3 * i] = c[0];
    cell[3 * i + 1] = c[1];
    cell[3 * i + 2] = c[2];
    if (pos4) {
        pos4[i] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], 0.0);
        cell4[i] = make_int4(c[0], c[1], c[2], 0);
    }
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

// ---------------------------------------------------------------------------
// Neighbour search, one CTA per destination bin (neighborlist.cpp:154-194).
//
//  1. fp32 prefilter: candidate / destination coordinates relative to the
//     bin origin, rounded to fp32; a pair is dropped only when
//     |v32|^2 > thr32, a threshold proven (host side, see nl_thr32) to keep
//     every pair the reference's fp64 prefilter keeps.
//  2. survivors are compacted into a per-warp queue and tested 32 at a
//     time with the reference's exact fp64 expressions (prefilter, then the
//     raw-position test d2 <= rc^2, d2 != 0) -- no divergence in the fp64 path.
//  3. hits become (src << 24 | image code) keys in a per-destination shared
//     buffer; at the end each destination's keys are bitonic-sorted by one
//     warp (canonical (src, image) order, neighborlist.cpp:21-24) and stored
//     to a fixed-capacity slab; the emit kernel turns slab rows into CSR.
// ---------------------------------------------------------------------------
constexpr int kWSCap = 32;  // stencil cells per batch (per warp)
constexpr int kCodeCap = 128;  // stencil cells whose q code is tabulated
// Row keys in shared memory are 32-bit: src << cbits | stencil-cell index.  For a
// fixed src every stencil cell maps to a distinct image, and the image q is
// monotone in the cell offset per axis, so (src, cell) order is the
// canonical (src, image) order; the 64-bit slab key (src << 24 | q code) is
// rebuilt from the cell index on output.
// The cell field is cbits = ceil(log2(#stencil cells)) wide (launch_nl_search).

struct WarpNL {             // per-warp shared state of the search
    int sc_bin[kWSCap];
    int sc_pre[kWSCap + 1];
    int sc_q[kWSCap][3];
    double sc_shift[kWSCap][3];
    uint32_t code[kCodeCap];      // image q code per stencil cell of the bin
    int cstart[32];               // per candidate chunk: non-empty cell starting at each slot
};

// Bitonic network over 16 R keys held by a 16-lane half-warp, R per lane:
// element i = hl * R + r (r = register), so the strides below R are register
// compare-exchanges and only the strides >= R shuffle (log2(16) * (log2(16) +
// 1) / 2 = 10 shuffle stages whatever R).  The two halves of a warp sort two
// destination rows at once.  Keys are unique; padding slots hold ~0 and sort
// last.  Ascending.
template <int R>
__device__ __forceinline__ void bitonic_half(uint32_t (&k)[R], int hl) {
    constexpr int N = 16 * R;
#pragma unroll
    for (int size = 2; size <= N; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= R) {
                const int ls = stride / R;
                const bool keep_min = (((hl * R) & size) == 0) == ((hl & ls) == 0);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, k[r], ls);
                    k[r] = keep_min ? min(k[r], o) : max(k[r], o);
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r & stride) continue;
                    const bool up = ((hl * R + r) & size) == 0;
                    const uint32_t a = k[r], b = k[r + stride];
                    k[r] = up ? min(a, b) : max(a, b);
                    k[r + stride] = up ? max(a, b) : min(a, b);
                }
            }
        }
}

// Search, one WARP per destination bin (no CTA barriers).  Shared memory per
// warp: WarpNL + the destination group (<= group atoms) + group x cap keys.
template <int CTAS>
__global__ void __launch_bounds__(kThreads, CTAS) k_nl_search(
    const Geom g, float thr32, float acc32, float zero32, int64_t nbins, int64_t n, int group,
    int cap,
    const int32_t* __restrict__ bin_start, const int32_t* __restrict__ s_id,
    const double* __restrict__ s_w, const double* __restrict__ s_p,
    const int32_t* __restrict__ s_c, int32_t* __restrict__ deg, int32_t* __restrict__ flags,
    unsigned long long* __restrict__ slab, const int32_t* __restrict__ owner, int only,
    int cbits, float pos_gate) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per-warp carve-up by byte offsets (keeps the shared address space)
    const size_t head = (sizeof(WarpNL) + 15) & ~(size_t)15;
    const size_t dst_bytes = (size_t)group * (16 + 24 + 24 + 12 + 4 + 4);
    const size_t per_warp = ((head + dst_bytes + 15) & ~(size_t)15) + (size_t)group * cap * 4;
    unsigned char* base = smem_raw + (size_t)warp * per_warp;
    WarpNL& S = *reinterpret_cast<WarpNL*>(base);
    size_t o = head;
    float4* d32 = reinterpret_cast<float4*>(base + o);
    o += sizeof(float4) * group;
    double* d_w = reinterpret_cast<double*>(base + o);
    o += sizeof(double) * 3 * group;
    double* d_p = reinterpret_cast<double*>(base + o);
    o += sizeof(double) * 3 * group;
    int* d_c = reinterpret_cast<int*>(base + o);
    o += sizeof(int) * 3 * group;
    int* d_id = reinterpret_cast<int*>(base + o);
    o += sizeof(int) * group;
    int* d_cnt = reinterpret_cast<int*>(base + o);
    o += sizeof(int) * group;
    o = (o + 15) & ~(size_t)15;
    uint32_t* keys = reinterpret_cast<uint32_t*>(base + o);

    // fast accept only while every |coordinate| <= pos_gate (k_wrap's max in
    // flags[3]; NaN bit patterns compare above the gate)
    if (!(__int_as_float(flags[3]) <= pos_gate)) acc32 = -1.0f;
    const int sx = 2 * g.sten[0] + 1, sy = 2 * g.sten[1] + 1, sz = 2 * g.sten[2] + 1;
    const int ncell = sx * sy * sz;
    const int64_t wg = (int64_t)blockIdx.x * kWarps + warp, nw = (int64_t)gridDim.x * kWarps;

    for (int64_t bb = wg; bb < nbins; bb += nw) {
        const int b0 = bin_start[bb], b1 = bin_start[bb + 1];
        if (b1 == b0) continue;
        const int bz = (int)(bb % g.bins[2]);
        const int by = (int)((bb / g.bins[2]) % g.bins[1]);
        const int bx = (int)(bb / ((int64_t)g.bins[2] * g.bins[1]));
        // bin origin (any common origin works; it only conditions fp32)
        const d3 org = rowvec_rn(g.L, (double)bx / g.bins[0], (double)by / g.bins[1],
                                 (double)bz / g.bins[2]);
        // destination atoms of this bin, in groups of <= `group`; with
        // only >= 0 (one rank per GPU) just the atoms that rank owns
        for (int pos = b0; pos < b1;) {
            int nd = 0;
            __syncwarp();
            while (nd < group && pos < b1) {
                const int slot = pos + lane;
                const bool ok = slot < b1 && (only < 0 || owner[s_id[slot]] == only);
                const unsigned m = __ballot_sync(0xffffffffu, ok);
                const int navail = __popc(m), take = min(navail, group - nd);
                const int rank = __popc(m & ((1u << lane) - 1u));
                if (ok && rank < take) {
                    const int t = nd + rank;
                    double w3[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        w3[k] = s_w[k * n + slot];
                        d_w[3 * t + k] = w3[k];
                        d_p[3 * t + k] = s_p[k * n + slot];
                        d_c[3 * t + k] = s_c[k * n + slot];
                    }
                    d32[t] = make_float4((float)(w3[0] - org.x), (float)(w3[1] - org.y),
                                         (float)(w3[2] - org.z), 0.f);
                    d_id[t] = s_id[slot];
                    d_cnt[t] = 0;
                }
                nd += take;
                pos = take < navail ? pos + (int)__fns(m, 0, take + 1) : pos + 32;
            }
            __syncwarp();
            if (nd == 0) break;
            for (int cbase = 0; cbase < ncell; cbase += kWSCap) {
                const int nc = min(kWSCap, ncell - cbase);
                __syncwarp();
                int cntc = 0;
                if (lane < nc) {
                    const int c = cbase + lane;
                    const int dz = c % sz - g.sten[2];
                    const int dy = (c / sz) % sy - g.sten[1];
                    const int dx = c / (sz * sy) - g.sten[0];
                    const int cc[3] = {bx + dx, by + dy, bz + dz};
                    int qv[3], cwb[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {  // neighborlist.cpp:165-170
                        const int nb = g.bins[k];
                        qv[k] = cc[k] >= 0 ? cc[k] / nb : -((-cc[k] + nb - 1) / nb);
                        cwb[k] = cc[k] - qv[k] * nb;
                        S.sc_q[lane][k] = qv[k];
                    }
                    if (cbase + lane < kCodeCap) S.code[cbase + lane] = qcode(qv[0], qv[1], qv[2]);
                    // shift = L0*q0 + L1*q1 + L2*q2 (neighborlist.cpp:171-173)
                    const d3 sh = rowvec_rn(g.L, (double)qv[0], (double)qv[1], (double)qv[2]);
                    S.sc_shift[lane][0] = sh.x;
                    S.sc_shift[lane][1] = sh.y;
                    S.sc_shift[lane][2] = sh.z;
                    const int64_t wb = ((int64_t)cwb[0] * g.bins[1] + cwb[1]) * g.bins[2] + cwb[2];
                    S.sc_bin[lane] = (int)wb;
                    cntc = bin_start[wb + 1] - bin_start[wb];
                    if (qv[0] < -128 || qv[0] > 127 || qv[1] < -128 || qv[1] > 127 ||
                        qv[2] < -128 || qv[2] > 127)
                        atomicOr(&flags[1], kErrQRange);
                }
                int incl = cntc;  // warp scan of candidate counts
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += u;
                }
                if (lane < nc) S.sc_pre[lane + 1] = incl;
                if (lane == 0) S.sc_pre[0] = 0;
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                const int pre_c = incl - cntc;  // lane c < nc: first candidate of cell c
                int carry = 0;                  // cell holding the chunk's first candidate
                __syncwarp();
                for (int kb = 0; kb < total; kb += 32) {
                    const int k = kb + lane;
                    const bool valid = k < total;
                    // cell of candidate k: the last non-empty cell starting at or
                    // before k (non-empty cells start at distinct slots) -- a
                    // warp max-scan over the chunk's cell starts
                    S.cstart[lane] = -1;
                    __syncwarp();
                    if (cntc > 0 && pre_c >= kb && pre_c < kb + 32) S.cstart[pre_c - kb] = lane;
                    __syncwarp();
                    int cm = S.cstart[lane];
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const int u = __shfl_up_sync(0xffffffffu, cm, off);
                        if (lane >= off) cm = max(cm, u);
                    }
                    cm = max(cm, carry);
                    carry = __shfl_sync(0xffffffffu, cm, 31);
                    float c32x = 0.f, c32y = 0.f, c32z = 0.f;
                    double cv[3] = {0.0, 0.0, 0.0};
                    int ci = 0, slot = 0;
                    uint32_t key = 0u;
                    if (valid) {
                        ci = cm;
                        slot = bin_start[S.sc_bin[ci]] + (k - S.sc_pre[ci]);
#pragma unroll
                        for (int d = 0; d < 3; ++d)  // wrapped_j + shift (neighborlist.cpp:176)
                            cv[d] = add_rn(s_w[d * n + slot], S.sc_shift[ci][d]);
                        key = ((uint32_t)s_id[slot] << cbits) | (uint32_t)(cbase + ci);
                        c32x = (float)(cv[0] - org.x);
                        c32y = (float)(cv[1] - org.y);
                        c32z = (float)(cv[2] - org.z);
                    }
                    // fp32 test of this lane's candidate against every destination
                    // of the group: |v32|^2 in (zero32, acc32] is inside both of the
                    // reference's fp64 tests (and d2 != 0) with a proven margin ->
                    // accepted here; (acc32, thr32] or <= zero32 is borderline ->
                    // exact fp64 below; > thr32 is outside the fp64 prefilter.
                    unsigned mask = 0u;
                    if (valid) {
                        for (int t = 0; t < nd; ++t) {
                            const float4 dd = d32[t];
                            const float vx = c32x - dd.x, vy = c32y - dd.y, vz = c32z - dd.z;
                            const float d2 = fmaf(vz, vz, fmaf(vy, vy, vx * vx));
                            if (d2 <= thr32) {
                                if (d2 <= acc32 && d2 > zero32) {
                                    const int pos = atomicAdd(&d_cnt[t], 1);
                                    if (pos < cap) keys[(size_t)t * cap + pos] = key;
                                } else {
                                    mask |= 1u << t;
                                }
                            }
                        }
                    }
                    // borderline pairs: the reference's exact fp64 expressions
                    // (rare: a band of relative width ~1e-5 around rc, and
                    // coincident atoms)
                    while (mask) {
                        const int t = __ffs(mask) - 1;
                        mask &= mask - 1u;
                        const d3 v = {sub_rn(cv[0], d_w[3 * t]), sub_rn(cv[1], d_w[3 * t + 1]),
                                      sub_rn(cv[2], d_w[3 * t + 2])};
                        if (!(dot_rn(v, v) > g.pre2)) {  // neighborlist.cpp:177
                            const int o0 = S.sc_q[ci][0] - s_c[slot] + d_c[3 * t];
                            const int o1 = S.sc_q[ci][1] - s_c[n + slot] + d_c[3 * t + 1];
                            const int o2 = S.sc_q[ci][2] - s_c[2 * n + slot] + d_c[3 * t + 2];
                            const d3 raw = rowvec_rn(g.L, (double)o0, (double)o1, (double)o2);
                            const d3 vr = {add_rn(sub_rn(s_p[slot], d_p[3 * t]), raw.x),
                                           add_rn(sub_rn(s_p[n + slot], d_p[3 * t + 1]), raw.y),
                                           add_rn(sub_rn(s_p[2 * n + slot], d_p[3 * t + 2]), raw.z)};
                            const double d2 = dot_rn(vr, vr);
                            if (!(d2 > g.cutoff2) && d2 != 0.0) {  // :189-190
                                const int pos = atomicAdd(&d_cnt[t], 1);
                                if (pos < cap) keys[(size_t)t * cap + pos] = key;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            // canonical (src, image) order (neighborlist.cpp:21-24), below.
            // Slab key of a sorted row entry: src << 24 | code of the image of
            // its stencil cell (neighborlist.cpp:165-170)
            auto slab_key = [&](uint32_t k) {
                const int c = (int)(k & ((1u << cbits) - 1u));
                if (c < kCodeCap) return ((unsigned long long)(k >> cbits) << 24) | S.code[c];
                const int cc[3] = {bx + c / (sz * sy) - g.sten[0], by + (c / sz) % sy - g.sten[1],
                                   bz + c % sz - g.sten[2]};
                int qv[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int nb = g.bins[a];
                    qv[a] = cc[a] >= 0 ? cc[a] / nb : -((-cc[a] + nb - 1) / nb);
                }
                return ((unsigned long long)(k >> cbits) << 24) | qcode(qv[0], qv[1], qv[2]);
            };
            // two destination rows per warp, one per half-warp: R keys per
            // lane in a half-warp bitonic network (rows of <= 128 keys), a
            // rank sort above
            const int hl = lane & 15, half = lane >> 4;
            for (int t0 = 0; t0 < nd; t0 += 2) {
                const int t = t0 + half;
                const int full = t < nd ? d_cnt[t] : 0;
                const int cnt = min(full, cap);
                const int cmax = max(cnt, __shfl_xor_sync(0xffffffffu, cnt, 16));
                const uint32_t* kk = keys + (size_t)t * cap;
                unsigned long long* dst = slab + (size_t)(t < nd ? d_id[t] : 0) * cap;
                if (cmax <= 64) {
                    uint32_t k4[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) k4[r] = hl * 4 + r < cnt ? kk[hl * 4 + r] : ~0u;
                    bitonic_half<4>(k4, hl);
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (hl * 4 + r < cnt) dst[hl * 4 + r] = slab_key(k4[r]);
                } else if (cmax <= 128) {
                    uint32_t k8[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) k8[r] = hl * 8 + r < cnt ? kk[hl * 8 + r] : ~0u;
                    bitonic_half<8>(k8, hl);
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (hl * 8 + r < cnt) dst[hl * 8 + r] = slab_key(k8[r]);
                } else {
                    // rare long rows: rank of each key among the row's keys,
                    // 16 keys per half-warp step
                    for (int k0 = 0; k0 < cmax; k0 += 16) {
                        const int ka = k0 + hl;
                        const uint32_t ma = ka < cnt ? kk[ka] : ~0u;
                        int ra = 0;
                        for (int i = 0; i < cnt; ++i) ra += kk[i] < ma;
                        if (ka < cnt) dst[ra] = slab_key(ma);
                    }
                }
                if (hl == 0 && t < nd) {
                    // the row as stored (<= cap: the emit never reads past a
                    // slab row); the true maximum goes to flags[0], and a
                    // build whose maximum exceeds cap is redone
                    deg[d_id[t]] = cnt;
                    atomicMax(&flags[0], full);
                }
            }
        }
    }
}

// slab rows -> canonical CSR (neighborlist.cpp:60-85): recompute the exact
// fp64 vector through the raw positions (:178-191) from (src, image), round
// to fp32 for the model, mark three-body bonds (linegraph.cpp:34-35).
template <int G, int MINB = 1>  // lanes per destination row (16 or 32)
__global__ void __launch_bounds__(128, MINB) k_nl_emit(const Geom g, int64_t n, int cap,
                          const unsigned long long* __restrict__ slab,
                          const int32_t* __restrict__ row, const double* __restrict__ pos,
                          const int32_t* __restrict__ cell, const double4* __restrict__ pos4,
                          const int4* __restrict__ cell4, int32_t* __restrict__ e_src,
                          uint32_t* __restrict__ e_img, float4* __restrict__ e_vd,
                          float* __restrict__ e_d, uint8_t* __restrict__ e_bond,
                          int32_t* __restrict__ bcnt, int32_t* __restrict__ flags,
                          const int32_t* __restrict__ owner, unsigned long long* __restrict__ req) {
    const int64_t i0 = (int64_t)blockIdx.x * (blockDim.x / G) + (threadIdx.x / G);
    const bool live = i0 < n;
    const int64_t i = live ? i0 : 0;
    const int lane = threadIdx.x & (G - 1);
    // lanes of this row (both rows of a warp iterate together for the ballot)
    const unsigned gmask = G == 32 ? 0xffffffffu : (0xffffu << (threadIdx.x & 16));
    const int e0 = row[i], cnt = live ? row[i + 1] - e0 : 0;
    const double4 pi4 = pos4[i];
    const int4 ci4 = cell4[i];
    const double pix = pi4.x, piy = pi4.y, piz = pi4.z;
    const int cix = ci4.x, ciy = ci4.y, ciz = ci4.z;
    int nb = 0;
    // the next slot's key is requested before this slot's gathers complete
    unsigned long long knext = lane < cnt ? __ldg(slab + (size_t)i * cap + lane) : 0ull;
    for (int kb = 0; __any_sync(0xffffffffu, kb < cnt); kb += G) {
        const int k = kb + lane;
        bool isb = false;
        const unsigned long long key = knext;
        if (k + G < cnt) knext = __ldg(slab + (size_t)i * cap + k + G);
        if (k < cnt) {
            const int j = (int)(key >> 24);
            const int q0 = (int)((key >> 16) & 255) - 128;
            const int q1 = (int)((key >> 8) & 255) - 128;
            const int q2 = (int)(key & 255) - 128;
            // the source's raw position and cell_of: one 32-byte and one
            // 16-byte load
            const double4 pj = pos4[j];
            const int4 cj = cell4[j];
            // off = image - cell_of[j] + cell_of[i] (neighborlist.cpp:179-180)
            const int o0 = q0 - cj.x + cix;
            const int o1 = q1 - cj.y + ciy;
            const int o2 = q2 - cj.z + ciz;
            if (!img_in_range(o0) || !img_in_range(o1) || !img_in_range(o2))
                atomicOr(&flags[1], kErrImgRange);
            // off = 0 (most edges): off L is a sum of signed zeros, and
            // x + (+-0) == x for every x the subtraction below can produce
            // (x - x is +0), so skipping it is bitwise the reference
            d3 raw = {0.0, 0.0, 0.0};
            if (o0 | o1 | o2) raw = rowvec_rn(g.L, (double)o0, (double)o1, (double)o2);
            const d3 vr = {add_rn(sub_rn(pj.x, pix), raw.x), add_rn(sub_rn(pj.y, piy), raw.y),
                           add_rn(sub_rn(pj.z, piz), raw.z)};
            const double dd = __dsqrt_rn(dot_rn(vr, vr));
            const int e = e0 + k;
            e_src[e] = j;
            if (e_img) e_img[e] = pack_img(o0, o1, o2);  // null: not needed by this build
            e_vd[e] = make_float4((float)vr.x, (float)vr.y, (float)vr.z, (float)dd);
            e_d[e] = (float)dd;
            isb = g.bond_bound >= 0.0 && !(dd > g.bond_bound);
            if (e_bond) e_bond[e] = isb ? 1 : 0;
            // p > 1 in one process: requirement masks (partitioner.cpp:124-134,
            // the same atomicOr set as k_required) from the edges emitted here
            if (req) {
                const int oi = owner[i], oj = owner[j];
                if (oj != oi) atomicOr(&req[j], 1ull << oi);
            }
        }
        nb += __popc(__ballot_sync(0xffffffffu, isb) & gmask);
    }
    if (live && lane == 0) {
        bcnt[i] = nb;
        if (nb > 0) atomicMax(&flags[2], nb);  // max in-bonds per center
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
                             int32_t* __restrict__ bedge, int32_t* __restrict__ ebid) {
    int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (v >= n) return;
    const int lane = threadIdx.x & 31;
    int base = brow[v];
    for (int eb = row[v]; eb < row[v + 1]; eb += 32) {
        int e = eb + lane;
        bool f = e < row[v + 1] && ebond[e];
        unsigned m = __ballot_sync(0xffffffffu, f);
        const int id = base + __popc(m & ((1u << lane) - 1u));
        if (f) bedge[id] = e;
        if (e < row[v + 1]) ebid[e] = f ? id : -1;  // bond id of an edge (bond_of_edge)
        base += __popc(m);
    }
}

// reverse bond: (w -> v, o) <-> (v -> w, -o), searched in row w which is
// sorted by (src, image) (linegraph.cpp:16-21 is_reverse_pair)
__global__ void k_bond_rev(int64_t n, const int32_t* __restrict__ row,
                           const int32_t* __restrict__ src, const uint32_t* __restrict__ img,
                           const uint8_t* __restrict__ ebond, const int32_t* __restrict__ brow,
                           const int32_t* __restrict__ bedge, const int32_t* __restrict__ ebid,
                           int32_t* __restrict__ brev,
                           int32_t* __restrict__ flags, const int32_t* __restrict__ owner,
                           int only) {
    int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (v >= n) return;
    for (int b = brow[v] + (threadIdx.x & 31); b < brow[v + 1]; b += 32) {
        const int e = bedge[b];
        const int w = src[e];
        if (only >= 0 && owner[w] != only) {  // reverse bond lives on w's rank:
            brev[b] = -1;                     // a halo bond row (rank bond plan)
            continue;
        }
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
        const int id = er >= 0 ? ebid[er] : -1;
        if (id < 0) atomicOr(&flags[1], 32);
        brev[b] = id;
    }
}

size_t nl_smem(int group, int cap) {
    const size_t head = (sizeof(WarpNL) + 15) & ~(size_t)15;
    const size_t dst_bytes = (size_t)group * (16 + 24 + 24 + 12 + 4 + 4);
    const size_t per_warp = ((head + dst_bytes + 15) & ~(size_t)15) + (size_t)group * cap * 4;
    return per_warp * kWarps;
}

int nl_grid(int64_t nbins) {
    int64_t g = (nbins + kWarps - 1) / kWarps;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g > 0 ? g : 1);
}

}  // namespace

void launch_wrap(const Geom& g, int64_t n, NLBuffers& b, cudaStream_t s) {
    k_wrap<<<div_up(n, 256), 256, 0, s>>>(g, n, b.pos, b.cell, b.fw_axis, b.bin, b.bin_cnt,
                                          b.flags, b.pos4, b.cell4);
    GMD_LAUNCH_CHECK();
}

void launch_bin_scatter(const Geom& g, int64_t n, NLBuffers& b, int32_t* fill, cudaStream_t s) {
    k_bin_scatter<<<div_up(n, 256), 256, 0, s>>>(g, n, b.pos, b.cell, b.bin, b.bin_start, fill,
                                                  b.s_id, b.s_w, b.s_p, b.s_c);
    GMD_LAUNCH_CHECK();
}

void launch_nl_search(const Geom& g, float thr32, float acc32, float zero32, float pos_gate,
                      int64_t nbins, int64_t n, int cap,
                      NLBuffers& b, unsigned long long* slab, const int32_t* owner, int only,
                      cudaStream_t s) {
    // destinations staged per warp (the search is latency-bound; occupancy
    // beats fewer candidate rescans)
    static const int gmax = [] {
        const char* v = std::getenv("GMD_NL_GROUP");
        return v ? std::max(1, std::min(32, std::atoi(v))) : 16;
    }();
    // four CTAs per SM (64 registers) when a group of >= 12 destinations still
    // fits their shared memory (C5: 14 destinations, 1.04 -> 0.93 ms);
    // otherwise three (C4's deeper rows leave 9 at four CTAs: more candidate
    // rescans, 0.198 -> 0.214 ms)
    int g4 = gmax;
    while (g4 > 1 && nl_smem(g4, cap) > 55 * 1024) --g4;
    const int ctas = g4 >= 12 ? 4 : 3;
    const size_t fit = ctas == 4 ? 55 * 1024 : 74 * 1024;
    int group = gmax;
    while (group > 4 && nl_smem(group, cap) > fit) --group;
    while (group > 1 && nl_smem(group, cap) > 110 * 1024) group >>= 1;
    const size_t sm = nl_smem(group, cap);
    if (sm > 200 * 1024) raise(kRuntime, "neighbour search: per-atom degree too large");
    static bool attr = false;
    if (!attr) {
        GMD_CUDA(cudaFuncSetAttribute(k_nl_search<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
        GMD_CUDA(cudaFuncSetAttribute(k_nl_search<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
        attr = true;
    }
    const int64_t ncell = (int64_t)(2 * g.sten[0] + 1) * (2 * g.sten[1] + 1) * (2 * g.sten[2] + 1);
    int cbits = 1;
    while (((int64_t)1 << cbits) < ncell) ++cbits;
    if (cbits > 31 || n > ((int64_t)1 << (32 - cbits)))
        raise(kConfig, "neighbour search: atom count too large for the " + std::to_string(ncell) +
                           "-cell stencil (row keys are src << " + std::to_string(cbits) + " | cell)");
    auto kern = ctas == 4 ? k_nl_search<4> : k_nl_search<3>;
    kern<<<nl_grid(nbins), kThreads, sm, s>>>(g, thr32, acc32, zero32, nbins, n, group, cap,
                                                     b.bin_start,
                                                     b.s_id, b.s_w, b.s_p, b.s_c, b.deg, b.flags,
                                                     slab, owner, only, cbits, pos_gate);
    GMD_LAUNCH_CHECK();
}

void launch_nl_emit(const Geom& g, int64_t n, int cap, const unsigned long long* slab,
                    NLBuffers& b, GraphDev& gd, cudaStream_t s, const int32_t* owner,
                    unsigned long long* req) {
    if (n == 0) return;
    if (!b.pos4 || !b.cell4) raise(kRuntime, "internal: emit needs the per-atom records");
    // 16 lanes per row: ~45-edge rows fill 3 x 16 slots (94 %) instead of
    // 2 x 32 (70 %); C5 0.70 -> 0.53 ms
    // 128-thread blocks (C5: 128 0.516 ms, 256 0.527, 512 0.624, 1024 0.656)
    // 12 CTAs per SM (40 registers): 0.480 -> 0.472 ms at C5 (16 CTAs / 32
    // registers spill: 0.595 ms)
    k_nl_emit<16, 12><<<div_up(n, 8), 128, 0, s>>>(g, n, cap, slab, gd.row, b.pos, b.cell, b.pos4, b.cell4, gd.src,
                                               gd.img, gd.vd, gd.d, gd.bond, b.bcnt, b.flags, owner, req);
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
                       int32_t* bedge, int32_t* ebid, cudaStream_t s) {
    if (n == 0) return;
    k_bond_edges<<<div_up(n, 8), 256, 0, s>>>(row, ebond, n, brow, bedge, ebid);
    GMD_LAUNCH_CHECK();
}

void launch_bond_rev(int64_t n, const GraphDev& gd, const int32_t* brow, const int32_t* bedge,
                     const int32_t* ebid, int32_t* brev, int32_t* flags, const int32_t* owner,
                     int only, cudaStream_t s) {
    if (n == 0) return;
    k_bond_rev<<<div_up(n, 8), 256, 0, s>>>(n, gd.row, gd.src, gd.img, gd.bond, brow, bedge, ebid,
                                            brev, flags, owner, only);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
