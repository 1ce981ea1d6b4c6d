// Toy invariant MLIP forward + hand-written backward on the GPU
// (proj/src/potential.cpp:19-78 math, :563-985 distributed pass).
//
// Design (B200-first, no float atomics, partition-invariant):
//  * every per-node reduction is a destination-row (CSR) gather, one warp per
//    node, lanes over in-edges, a fixed-order butterfly reduce -- results do
//    not depend on the partition count;
//  * the backward never scatters to sources: the adjoint of "h[src] feeds
//    m[dst]" is gathered at the source through the reverse edge (s_e is a
//    function of |v_e| only, and the reverse edge has the bitwise-negated
//    vector), so dL/dh, forces and the virial are row-local sums;
//  * the radial channel s = P u(d) / ds = P u'(d) is recomputed in registers
//    per edge and layer (never stored: E x F floats would dominate HBM);
//  * the three-body stage runs per "center" atom s on its in-bond list
//    (bonds e=(w->s) and their reverses e'=(s->w)): every line edge (e, e')
//    with dst(e) = src(e') is a pair of slots of one center.
#include <algorithm>
#include <cstdlib>

#include "gmd_model.cuh"
#include "gmd_tc.cuh"

namespace gmd {

__constant__ ModelConst c_m;

void upload_model(const ModelConst& m, cudaStream_t s) {
    GMD_CUDA(cudaMemcpyToSymbolAsync(c_m, &m, sizeof(ModelConst), 0, cudaMemcpyHostToDevice, s));
}

namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerCta = kThreads / 32;

// u_k(d) = fc(d) exp(-((d - mu_k)/sigma)^2) (potential.cpp:30-50)
__device__ __forceinline__ void basis(float d, float rc, float inv_rc, float inv_sigma,
                                      float mu_step, float u[kK]) {
    const float fc = d < rc ? 0.5f * (cospif(d * inv_rc) + 1.0f) : 0.0f;
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        float x = (d - mu_step * (float)k) * inv_sigma;
        u[k] = fc * __expf(-x * x);
    }
}

__device__ __forceinline__ void basis_d(float d, float rc, float inv_rc, float inv_sigma,
                                        float mu_step, float u[kK], float du[kK]) {
    float sn, cs;
    sincospif(d * inv_rc, &sn, &cs);
    const bool in = d < rc;
    const float fc = in ? 0.5f * (cs + 1.0f) : 0.0f;
    const float dfc = in ? -0.5f * 3.14159265358979f * inv_rc * sn : 0.0f;
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        float x = (d - mu_step * (float)k) * inv_sigma;
        float phi = __expf(-x * x);
        u[k] = fc * phi;
        du[k] = phi * (dfc - 2.0f * fc * x * inv_sigma);
    }
}

__device__ __forceinline__ void fcut3(float d, float& fc, float& dfc) {
    float sn, cs;
    sincospif(d * c_m.inv_r3, &sn, &cs);
    const bool in = d < c_m.r3;
    fc = in ? 0.5f * (cs + 1.0f) : 0.0f;
    dfc = in ? -0.5f * 3.14159265358979f * c_m.inv_r3 * sn : 0.0f;
}

// Fast radial basis for the atom channel on the SFU: fc from __cosf on
// [0, pi], phi_k = ex2(-(d a - b_k)^2) with a = sqrt(log2 e)/sigma and
// b_k = mu_k a (constants in c_m.bx[]); |error| ~1e-7, far inside the fp32
// tolerance of the parity tests.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void phi_fast(float d, float phi[kK]) {
    const float xa = d * c_m.a2;
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        const float x = xa - c_m.bx[k];
        phi[k] = ex2_approx(-x * x);
    }
}
__device__ __forceinline__ float fc_fast(float d) {
    return d < c_m.rc ? 0.5f * __cosf(d * c_m.pi_rc) + 0.5f : 0.0f;
}
__device__ __forceinline__ void fc_dfc_fast(float d, float& fc, float& dfc) {
    float sn, cs;
    __sincosf(d * c_m.pi_rc, &sn, &cs);
    const bool in = d < c_m.rc;
    fc = in ? 0.5f * cs + 0.5f : 0.0f;
    dfc = in ? -0.5f * c_m.pi_rc * sn : 0.0f;
}

// 256-bit read-only load (LDG.E.ENL2.256 on sm_100a): one instruction per
// 32-byte sector, so a 64-byte feature row costs two sector accesses.
__device__ __forceinline__ void ldg256(const float* p, float4& a, float4& b) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                   "=f"(b.w)
                 : "l"(p));
}

__device__ __forceinline__ void load_row16(const float* __restrict__ p, float h[kF]) {
    const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float4 t = __ldg(q + i);
        h[4 * i] = t.x;
        h[4 * i + 1] = t.y;
        h[4 * i + 2] = t.z;
        h[4 * i + 3] = t.w;
    }
}

__device__ __forceinline__ void store_row16(float* p, const float h[kF]) {
    float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = make_float4(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// fixed-order CTA reduction of W doubles per thread-warp; lane 0 of each warp
// deposits, thread 0 sums warps in order
template <int W, int NW = kWarpsPerCta>
__device__ __forceinline__ void cta_partials(const double (&v)[W], double* out) {
    __shared__ double red[NW][W];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double s[W];
#pragma unroll
    for (int c = 0; c < W; ++c) s[c] = warp_sum_d(v[c]);
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < W; ++c) red[warp][c] = s[c];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int c = 0; c < W; ++c) {
            double acc = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += red[w][c];
            out[(size_t)blockIdx.x * W + c] = acc;
        }
    }
}

// --------------------------------------------------------------------------
// h0 rows = emb[Z] for every layout row (potential.cpp:597-602); with zs,
// also the row's species byte and the 119-bit presence mask of the species
// (zmask[4]: an atomic only where the bit is not yet visible) for the
// layer-0 conv's species-sum form
__global__ void k_embed(int64_t rows, const int32_t* __restrict__ node_array,
                        const int32_t* __restrict__ Z, float* __restrict__ H0,
                        uint8_t* __restrict__ zs, unsigned* zmask) {
    __shared__ unsigned smask[4];
    if (threadIdx.x < 4) smask[threadIdx.x] = 0u;
    __syncthreads();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = t < rows * 4;
    const int64_t r = t >> 2;
    const int q = (int)(t & 3);
    int z = 0;
    if (live) {
        const int id = node_array ? node_array[r] : (int)r;
        z = Z[id];
        const float* e = c_m.emb + z * kF + 4 * q;
        reinterpret_cast<float4*>(H0)[t] = make_float4(e[0], e[1], e[2], e[3]);
        if (zs && q == 0) zs[r] = (uint8_t)z;
    }
    if (zs) {  // presence mask: warp OR -> block OR -> one global OR per word
        const bool mine = live && q == 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const unsigned v = __reduce_or_sync(0xffffffffu, mine && (z >> 5) == w ? 1u << (z & 31) : 0u);
            if ((threadIdx.x & 31) == 0 && v) atomicOr(&smask[w], v);
        }
        __syncthreads();
        if (threadIdx.x < 4 && smask[threadIdx.x]) atomicOr(zmask + threadIdx.x, smask[threadIdx.x]);
    }
}

__global__ void k_exchange(int64_t nx, const int32_t* __restrict__ xdst,
                           const int32_t* __restrict__ xsrc, float4* __restrict__ buf, int w4) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nx * w4) return;
    int64_t k = t / w4;
    int q = (int)(t - k * w4);
    buf[(int64_t)xdst[k] * w4 + q] = buf[(int64_t)xsrc[k] * w4 + q];
}

// Sum 16 per-lane values over a 16-lane group; lane l of the group ends with
// feature (l & 15).
__device__ __forceinline__ float transpose_reduce16_g16(float v[kF], int gl) {
    float w8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        bool up = gl & 8;
        float send = up ? v[i] : v[i + 8];
        float keep = up ? v[i + 8] : v[i];
        w8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float w4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        bool up = gl & 4;
        float send = up ? w8[i] : w8[i + 4];
        float keep = up ? w8[i + 4] : w8[i];
        w4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    float w2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        bool up = gl & 2;
        float send = up ? w4[i] : w4[i + 2];
        float keep = up ? w4[i + 2] : w4[i];
        w2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    bool up = gl & 1;
    float send = up ? w2[0] : w2[1];
    float keep = up ? w2[1] : w2[0];
    return keep + __shfl_xor_sync(0xffffffffu, send, 1);
}

// Shared-memory transpose of a 16-lane group's per-lane partial sums: lane gl
// stores its values as one row (STS.128), then sums column gl over the 16 rows
// in the shuffle butterfly's pairwise order (the node's result does not depend on where it
// runs).  ~35 instructions per group for 16 features instead of the 60 of the
// shuffle butterfly (15 SHFL, 15 FADD, 30 FSEL).  Row stride S floats: S a
// multiple of 4 with S/4 odd keeps every 8-lane LDS.128/STS.128 phase on
// distinct bank quads; the 16-float gap between the two groups of a warp puts
// their column reads on opposite bank halves.
template <int S>
struct GroupT {
    static constexpr int kGroup = 16 * S + 16;  // floats per group
};
template <int S>
__device__ __forceinline__ float column_sum16(const float* sT, int col) {
    float r[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = sT[j * S + col];
    // the xor-butterfly's tree (pairs l, l^8 first): bitwise the shuffle
    // reduction, which is invariant under reversing a row of <= 8 edges
    // (the reference's permutation-equivariance test, test_potential.cpp:146)
#pragma unroll
    for (int w = 8; w > 0; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) r[j] += r[j + w];
    return r[0];
}

// Conv node update from the group's per-lane partial sums: m_gl (column sum),
// z_gl = b_gl + sum_g W[gl][g] m_g with m broadcast from shared memory and W
// rows read as float4 (sW row stride 20).  Used by both conv kernel families
// (bitwise-equal energies).
constexpr int kConvTS = 20;
__device__ __forceinline__ float conv_wm(float m, int gl, float* sM, const float* sW, float b);
__device__ __forceinline__ float conv_node_z(const float acc[kF], int gl, float* sT, float* sM,
                                             const float* sW, float b) {
    float4* row = reinterpret_cast<float4*>(sT + gl * kConvTS);
#pragma unroll
    for (int c = 0; c < 4; ++c)
        row[c] = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
    __syncwarp();
    return conv_wm(column_sum16<kConvTS>(sT, gl), gl, sM, sW, b);
}

// z_gl = b + sum_g W[gl][g] m_g from each lane's m_gl (m broadcast through
// shared memory, W rows as float4)
__device__ __forceinline__ float conv_wm(float m, int gl, float* sM, const float* sW, float b) {
    sM[gl] = m;
    __syncwarp();
    const float4* mv = reinterpret_cast<const float4*>(sM);
    const float4* wr = reinterpret_cast<const float4*>(sW + gl * kConvTS);
    float z = b;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float4 m4 = mv[c], w4 = wr[c];
        z = fmaf(w4.x, m4.x, z);
        z = fmaf(w4.y, m4.y, z);
        z = fmaf(w4.z, m4.z, z);
        z = fmaf(w4.w, m4.w, z);
    }
    return z;
}

__device__ __forceinline__ float group_sum16(float v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double group_sum16d(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Newton's third law, exactly: an edge and its reverse produce bitwise
// opposite fp32 gradient terms (symmetric dsum, negated vector), which are
// summed per node in fp64 -- exact for terms within 2^29 of each other -- so
// the forces sum to zero up to the final fp64 rounding (translation invariance,
// momentum conservation; test_potential.cpp:160-172, test_md.cpp:110-122)
__device__ __forceinline__ void grad_add(double4* GRAD, int64_t k, double gx, double gy, double gz) {
    double4 g = GRAD[k];  // one writer per node and kernel: plain read-add-write
    g.x += gx;
    g.y += gy;
    g.z += gz;
    GRAD[k] = g;
}

constexpr int kNodesPerCta = kThreads / 16;  // half-warp (16 lanes) per node

// forward conv layer (potential.cpp:743-774): a 16-lane group per owned node,
// lanes stride over its in-edges two at a time (both edges' loads in flight
// before the math), fixed-order group reduction.  Reads 8 B per edge (d and
// the source row); the radial channel is recomputed in registers.
__device__ __forceinline__ void conv_edge(float d, const float* __restrict__ hrow, float acc[kF]) {
    float4 hv[4];
    ldg256(hrow, hv[0], hv[1]);
    ldg256(hrow + 8, hv[2], hv[3]);
    float phi[kK];
    phi_fast(d, phi);
    const float fc = fc_fast(d);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float4 h4 = hv[c];
        const float hh[4] = {h4.x * fc, h4.y * fc, h4.z * fc, h4.w * fc};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int f = 4 * c + i;
            float sv = 0.0f;
#pragma unroll
            for (int k = 0; k < kK; ++k) sv = fmaf(c_m.P[f * kK + k], phi[k], sv);
            acc[f] = fmaf(hh[i], sv, acc[f]);
        }
    }
}

__global__ void __launch_bounds__(kThreads, 3) k_conv(ConvArgs a, int layer,
                                                      const float* __restrict__ Hin,
                                                      float* __restrict__ Hout,
                                                      float* __restrict__ TH, double* per_atom,
                                                      double* e_part) {
    __shared__ __align__(16) float sW[kF * kConvTS];
    __shared__ __align__(16) float sT[kNodesPerCta * GroupT<kConvTS>::kGroup];
    __shared__ __align__(16) float sM[kNodesPerCta][kF];
    __shared__ float sb[kF], sro[kF];
    for (int i = threadIdx.x; i < kF * kF; i += kThreads) sW[(i / kF) * kConvTS + i % kF] = c_m.W[layer][i];
    if (threadIdx.x < kF) {
        sb[threadIdx.x] = c_m.b[layer][threadIdx.x];
        sro[threadIdx.x] = c_m.ro[threadIdx.x];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int gl = lane & 15;
    const int64_t g0 = (int64_t)blockIdx.x * kNodesPerCta + (threadIdx.x >> 4);
    const int64_t ng = (int64_t)gridDim.x * kNodesPerCta;
    double esum = 0.0;
    // both half-warps iterate the same number of times (shuffles span the warp)
    const int64_t iters = (a.n + ng - 1) / ng;
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t k = g0 + it * ng;  // local node index
        const bool valid = k < a.n;
        const int64_t v = valid ? (a.nodes ? (int64_t)a.nodes[k] : k) : 0;  // global id
        float acc[kF];
#pragma unroll
        for (int f = 0; f < kF; ++f) acc[f] = 0.0f;
        const int e0 = valid ? __ldg(a.row + v) : 0;
        const int e1 = valid ? __ldg(a.row + v + 1) : 0;
        for (int e = e0 + gl; __any_sync(0xffffffffu, e < e1); e += 32) {
            const bool ha = e < e1, hb = e + 16 < e1;
            const float da = ha ? __ldg(a.d + e) : 0.f;
            const float db = hb ? __ldg(a.d + e + 16) : 0.f;
            const int ia = ha ? __ldg(a.lsrc + e) : 0;
            const int ib = hb ? __ldg(a.lsrc + e + 16) : 0;
            if (ha) conv_edge(da, Hin + (size_t)ia * kF, acc);
            if (__any_sync(0xffffffffu, hb) && hb) conv_edge(db, Hin + (size_t)ib * kF, acc);
        }
        const int grp = threadIdx.x >> 4;
        const float z = conv_node_z(acc, gl, sT + grp * GroupT<kConvTS>::kGroup, sM[grp], sW, sb[gl]);
        const float th = tanhf(z);
        float ev = 0.0f;
        if (valid) {
            const int64_t r = a.crow ? a.crow[v] : v;
            const float hn = Hin[r * kF + gl] + th;
            Hout[r * kF + gl] = hn;
            note_nonfinite(a, layer, r, hn);
            TH[k * kF + gl] = th;
            ev = sro[gl] * hn;
        }
        if (per_atom) {
            ev = group_sum16(ev);
            if (valid && gl == 0) {
                per_atom[v] = (double)ev;
                esum += (double)ev;
            }
        }
    }
    if (e_part) {
        double vals[1] = {esum};
        cta_partials<1>(vals, e_part);
    }
}

// m_bar = W^T (h_bar * sech^2) (potential.cpp:816-822), thread per node
// init: the first backward layer, where h_bar is still the readout for every
// node (potential.cpp:808): use it directly and write it as HB's initial value
__global__ void k_bwd_node(int64_t n, const int32_t* __restrict__ nodes,
                           const int32_t* __restrict__ crow, int layer,
                           float* __restrict__ HB, const float* __restrict__ TH,
                           float* __restrict__ MB, bool init) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t v = nodes ? (int64_t)nodes[k] : k;
    float hb[kF], th[kF], y[kF];
    if (init) {
#pragma unroll
        for (int f = 0; f < kF; ++f) hb[f] = c_m.ro[f];
        store_row16(HB + k * kF, hb);
    } else {
        load_row16(HB + k * kF, hb);
    }
    load_row16(TH + k * kF, th);
#pragma unroll
    for (int f = 0; f < kF; ++f) y[f] = hb[f] * (1.0f - th[f] * th[f]);
    float mb[kF];
#pragma unroll
    for (int g = 0; g < kF; ++g) {
        float acc = 0.0f;
#pragma unroll
        for (int f = 0; f < kF; ++f) acc = fmaf(c_m.W[layer][f * kF + g], y[f], acc);
        mb[g] = acc;
    }
    const int64_t r = crow ? crow[v] : v;
    store_row16(MB + r * kF, mb);
}

// backward edge pass in row form (potential.cpp:823-848 restated as
// gathers): a 16-lane group per node u; the node's own m_bar / h_in rows are
// staged in shared memory (broadcast reads); each lane takes two in-edges per
// iteration and issues both edges' neighbour-row loads before any math.
struct BwdEdgeIn {
    float4 q;      // (vx, vy, vz, d)
    float4 m[4];   // m_bar[w]
    float4 h[4];   // h_in[w]
};

__device__ __forceinline__ void bwd_load(const ConvArgs& a, const float* __restrict__ MB,
                                         const float* __restrict__ Hl, int e, BwdEdgeIn& x) {
    x.q = __ldg(a.vd + e);
    const int w = __ldg(a.lsrc + e);
    const float* mw = MB + (size_t)w * kF;
    const float* hw = Hl + (size_t)w * kF;
    ldg256(mw, x.m[0], x.m[1]);
    ldg256(mw + 8, x.m[2], x.m[3]);
    ldg256(hw, x.h[0], x.h[1]);
    ldg256(hw + 8, x.h[2], x.h[3]);
}

__device__ __forceinline__ void bwd_math(const BwdEdgeIn& x, const float4* su_m,
                                         const float4* su_h, float isg, float mus, float acc[kF],
                                         double& gx, double& gy, double& gz, float vr[6]) {
    const float4 q = x.q;
    // s_f = fc A_f, ds_f = dfc A_f - 2 fc/sigma (x0 A_f - a B_f) with
    // A_f = sum_k P_fk phi_k, B_f = sum_k k P_fk phi_k (potential.cpp:30-50)
    float fc, dfc;
    fc_dfc_fast(q.w, fc, dfc);
    float phi[kK];
    phi_fast(q.w, phi);
    const float x0 = q.w * isg, step = mus * isg;
    const float ca = dfc - 2.0f * fc * isg * x0, cb = 2.0f * fc * isg * step;
    float dself = 0.f, drev = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float4 mu4 = su_m[c], hu4 = su_h[c];
        const float mwv[4] = {x.m[c].x, x.m[c].y, x.m[c].z, x.m[c].w};
        const float hwv[4] = {x.h[c].x, x.h[c].y, x.h[c].z, x.h[c].w};
        const float muv[4] = {mu4.x, mu4.y, mu4.z, mu4.w};
        const float huv[4] = {hu4.x, hu4.y, hu4.z, hu4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int f = 4 * c + i;
            float A = 0.f, B = 0.f;
#pragma unroll
            for (int k = 0; k < kK; ++k) {
                A = fmaf(c_m.P[f * kK + k], phi[k], A);
                B = fmaf(c_m.Pk[f * kK + k], phi[k], B);
            }
            const float ds = fmaf(ca, A, cb * B);
            acc[f] = fmaf(mwv[i], fc * A, acc[f]);
            dself = fmaf(muv[i] * hwv[i], ds, dself);
            drev = fmaf(mwv[i] * huv[i], ds, drev);
        }
    }
    const float invd = 1.0f / q.w;
    const float coef = (dself + drev) * invd;  // dself and drev swap on the reverse edge
    gx -= (double)(q.x * coef);
    gy -= (double)(q.y * coef);
    gz -= (double)(q.z * coef);
    const float cself = dself * invd;
    vr[0] = fmaf(cself * q.x, q.x, vr[0]);
    vr[1] = fmaf(cself * q.y, q.y, vr[1]);
    vr[2] = fmaf(cself * q.z, q.z, vr[2]);
    vr[3] = fmaf(cself * q.x, q.y, vr[3]);
    vr[4] = fmaf(cself * q.x, q.z, vr[4]);
    vr[5] = fmaf(cself * q.y, q.z, vr[5]);
}

__global__ void __launch_bounds__(kThreads, 2) k_bwd_edge(ConvArgs a, const float* __restrict__ MB,
                                                          const float* __restrict__ Hl,
                                                          float* __restrict__ HB,
                                                          double4* __restrict__ GRAD,
                                                          double* vir_part) {
    __shared__ __align__(16) float sU[kNodesPerCta][2][kF];  // [group][m_bar_u, h_u][f]
    __shared__ double sVir[kNodesPerCta][6];                // per-group fp64 virial sums
    const int lane = threadIdx.x & 31;
    const int gl = lane & 15, grp = threadIdx.x >> 4;
    const int64_t g0 = (int64_t)blockIdx.x * kNodesPerCta + grp;
    const int64_t ng = (int64_t)gridDim.x * kNodesPerCta;
    const float isg = c_m.inv_sigma, mus = c_m.mu_step;
    if (gl < 6) sVir[grp][gl] = 0.0;
    const int64_t iters = (a.n + ng - 1) / ng;
    // node k + ng's row bounds and own rows are loaded while node k runs
    int e0n = 0, e1n = 0;
    float mun = 0.f, hun = 0.f;
    auto prefetch = [&](int64_t k) {
        if (k < a.n) {
            const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
            const int64_t r = a.crow ? a.crow[v] : v;
            e0n = __ldg(a.row + v);
            e1n = __ldg(a.row + v + 1);
            mun = __ldg(MB + r * kF + gl);
            hun = __ldg(Hl + r * kF + gl);
        } else {
            e0n = e1n = 0;
        }
    };
    prefetch(g0);
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t k = g0 + it * ng;  // local node index
        const bool valid = k < a.n;
        const int e0 = e0n, e1 = e1n;
        __syncwarp();
        if (valid) {
            sU[grp][0][gl] = mun;
            sU[grp][1][gl] = hun;
        }
        __syncwarp();
        prefetch(k + ng);
        float acc[kF];
#pragma unroll
        for (int f = 0; f < kF; ++f) acc[f] = 0.0f;
        double gx = 0.0, gy = 0.0, gz = 0.0;
        float vr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const float4* su_m = reinterpret_cast<const float4*>(sU[grp][0]);
        const float4* su_h = reinterpret_cast<const float4*>(sU[grp][1]);
        for (int e = e0 + gl; __any_sync(0xffffffffu, e < e1); e += 32) {
            const bool ha = e < e1, hb = e + 16 < e1;
            BwdEdgeIn xa, xb;
            if (ha) bwd_load(a, MB, Hl, e, xa);
            if (hb) bwd_load(a, MB, Hl, e + 16, xb);
            if (ha) bwd_math(xa, su_m, su_h, isg, mus, acc, gx, gy, gz, vr);
            if (__any_sync(0xffffffffu, hb) && hb)
                bwd_math(xb, su_m, su_h, isg, mus, acc, gx, gy, gz, vr);
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) vr[c] = group_sum16(vr[c]);
        if (gl == 0)
#pragma unroll
            for (int c = 0; c < 6; ++c) sVir[grp][c] += (double)vr[c];
        const float hb = transpose_reduce16_g16(acc, gl);
        gx = group_sum16d(gx);
        gy = group_sum16d(gy);
        gz = group_sum16d(gz);
        if (valid) {  // one writer per element: plain read-add-write
            HB[k * kF + gl] += hb;
            if (gl == 0) grad_add(GRAD, k, gx, gy, gz);
        }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        double acc6 = 0.0;
        for (int g = 0; g < kNodesPerCta; ++g) acc6 += sVir[g][threadIdx.x];
        vir_part[(size_t)blockIdx.x * 6 + threadIdx.x] = acc6;
    }
}

// ---------------------------------------------------------------------------
// Packed-FP32 (FFMA2) conv and backward edge pass.
//
// sm_100a issues FFMA2 / FMUL2: two IEEE fp32 FMAs per instruction with a
// scalar operand broadcast to both halves and a constant pair from a uniform
// register (LDCU.128 loads two pairs).  The FMA pipe still does 32 lanes per
// cycle, so FFMA2 halves issue slots, not FMA cycles; the model kernels were
// issue-bound (FFMA + LDCU), so packing moves them toward the FMA-pipe bound.
// Feature pairs (f, f+1) are packed: A_(f,f+1) = sum_k (P[f][k], P[f+1][k]) phi_k
// uses the k-major copy PT; G_(k,k+1) = sum_f (P[f][k], P[f][k+1]) g_f uses P.
// Each lane keeps one edge's gathered rows in flight while it computes the
// previous one (software pipeline across the node's in-edges).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 bcast(float x) { return make_float2(x, x); }

// A[i] = (A_2i, A_2i+1), A_f = sum_k P[f][k] ph[k], summed in ascending k
__device__ __forceinline__ void radial_pairs(const float ph[kK], float2 A[kF / 2]) {
    const float2* PT2 = reinterpret_cast<const float2*>(c_m.PT);
#pragma unroll
    for (int i = 0; i < kF / 2; ++i) A[i] = f2fma(PT2[i], bcast(ph[0]), make_float2(0.f, 0.f));
#pragma unroll
    for (int k = 1; k < kK; ++k)
#pragma unroll
        for (int i = 0; i < kF / 2; ++i) A[i] = f2fma(PT2[k * (kF / 2) + i], bcast(ph[k]), A[i]);
}

struct ConvIn {
    float d;
    float4 h[4];
};

// gathered source row w (its index was read one step earlier)
__device__ __forceinline__ void conv_load(const float* __restrict__ Hin, int w, ConvIn& x) {
    const float* hrow = Hin + (size_t)w * kF;
    ldg256(hrow, x.h[0], x.h[1]);
    ldg256(hrow + 8, x.h[2], x.h[3]);
}
// the per-edge streams (source index, d or (v, d)) are read one slot ahead:
// they come from DRAM, the gathered rows mostly from L2
__device__ __forceinline__ int src_of(const ConvArgs& a, int e, int e1) {
    return e < e1 ? __ldg(a.lsrc + e) : 0;
}
__device__ __forceinline__ float d_of(const ConvArgs& a, int e, int e1) {
    return e < e1 ? __ldg(a.d + e) : 0.f;
}
__device__ __forceinline__ float4 vd_of(const ConvArgs& a, int e, int e1) {
    return e < e1 ? __ldg(a.vd + e) : make_float4(0.f, 0.f, 0.f, 1.f);
}

// same arithmetic, per feature and in the same order, as conv_edge
__device__ __forceinline__ void conv_math2(const ConvIn& x, float2 acc[kF / 2]) {
    float phi[kK];
    phi_fast(x.d, phi);
    const float fc = fc_fast(x.d);
    float2 A[kF / 2];
    radial_pairs(phi, A);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float4 h4 = x.h[c];
        const float2 h0 = f2mul(make_float2(h4.x, h4.y), bcast(fc));
        const float2 h1 = f2mul(make_float2(h4.z, h4.w), bcast(fc));
        acc[2 * c] = f2fma(h0, A[2 * c], acc[2 * c]);
        acc[2 * c + 1] = f2fma(h1, A[2 * c + 1], acc[2 * c + 1]);
    }
}

// SPEC (layer 0, h0 = emb[Z], at most two species present): m_f =
// sum_e emb[Z_src][f] s_e,f = sum_s emb[z_s][f] sum_k P[f][k] Phi_s,k with
// Phi_s = sum over in-edges from species s of fc(d) phi(d) -- per edge only
// the radial basis and one species byte (no 64-byte row gather, no 16 x 8
// contraction); per node z = b + sum_s (W diag(emb[z_s]) P) Phi_s, the two
// 16 x 8 matrices staged per CTA.  More than two species: the per-edge form.
template <int CTAS, int NT = kThreads, bool SPEC = false>
__global__ void __launch_bounds__(NT, CTAS) k_conv2(ConvArgs a, int layer,
                                                       const float* __restrict__ Hin,
                                                       float* __restrict__ Hout,
                                                       float* __restrict__ TH, double* per_atom,
                                                       double* e_part, const uint8_t* __restrict__ zs = nullptr,
                                                       const unsigned* __restrict__ zmask = nullptr) {
    __shared__ __align__(16) float sW[kF * kConvTS];
    __shared__ __align__(16) float sT[(NT / 16) * GroupT<kConvTS>::kGroup];
    __shared__ __align__(16) float sM[NT / 16][kF];
    __shared__ float sb[kF], sro[kF];
    // [s][g][k] = (W diag(emb[z_s]) P)[g][k]: z = b + sum_s M_s Phi_s directly
    __shared__ __align__(16) float sPe[SPEC ? 2 * kF * kK : 4];
    for (int i = threadIdx.x; i < kF * kF; i += NT) sW[(i / kF) * kConvTS + i % kF] = c_m.W[layer][i];
    if (threadIdx.x < kF) {
        sb[threadIdx.x] = c_m.b[layer][threadIdx.x];
        sro[threadIdx.x] = c_m.ro[threadIdx.x];
    }
    int nspec = 3, z1 = -1;
    if constexpr (SPEC) {
        int z0 = -1;
        nspec = 0;
        for (int w = 0; w < 4; ++w) {
            unsigned m = zmask[w];
            nspec += __popc(m);
            while (m) {
                const int z = 32 * w + __ffs(m) - 1;
                m &= m - 1u;
                if (z0 < 0) z0 = z; else if (z1 < 0) z1 = z;
            }
        }
        if (z1 < 0) z1 = z0;
        if (nspec <= 2)
            for (int i = threadIdx.x; i < 2 * kF * kK; i += NT) {
                const int sp = i / (kF * kK), gg = (i / kK) % kF, kk = i % kK;
                const float* e = c_m.emb + (sp ? z1 : z0) * kF;
                float acc = 0.f;
                for (int f = 0; f < kF; ++f) acc = fmaf(c_m.W[layer][gg * kF + f], e[f] * c_m.P[f * kK + kk], acc);
                sPe[i] = acc;
            }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int gl = lane & 15;
    const int64_t g0 = (int64_t)blockIdx.x * (NT / 16) + (threadIdx.x >> 4);
    const int64_t ng = (int64_t)gridDim.x * (NT / 16);
    double esum = 0.0;
    const int64_t iters = (a.n + ng - 1) / ng;
    // the next node's bounds and first slot's streams are requested at the
    // start of the current node
    int64_t vn = 0;
    int e0n = 0, e1n = 0, wn = 0;
    float dn = 0.f;
    auto prefetch = [&](int64_t k) {
        if (k < a.n) {
            vn = a.nodes ? (int64_t)a.nodes[k] : k;
            e0n = __ldg(a.row + vn);
            e1n = __ldg(a.row + vn + 1);
            wn = src_of(a, e0n + gl, e1n);
            dn = d_of(a, e0n + gl, e1n);
        } else {
            vn = 0;
            e0n = e1n = 0;
        }
    };
    prefetch(g0);
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t k = g0 + it * ng;
        const bool valid = k < a.n;
        const int64_t v = vn;
        const int e0 = e0n, e1 = e1n;
        int w = wn;
        float dcur = dn;
        prefetch(k + ng);
        float2 acc[kF / 2];
#pragma unroll
        for (int i = 0; i < kF / 2; ++i) acc[i] = make_float2(0.f, 0.f);
        const int grp = threadIdx.x >> 4;
        float z;
        if (SPEC && nspec <= 2) {
            // acc[0..3] = Phi_0 (k pairs), acc[4..7] = Phi_1; the species
            // byte is read one slot ahead, after the slot's radial math
            int zc = e0 + gl < e1 ? zs[w] : 0;
            for (int e = e0 + gl; __any_sync(0xffffffffu, e < e1); e += 16) {
                if (e < e1) {
                    const float d = dcur;
                    const float w1 = zc == z1 ? 1.0f : 0.0f, w0 = 1.0f - w1;
                    w = src_of(a, e + 16, e1);
                    dcur = d_of(a, e + 16, e1);
                    float phi[kK];
                    phi_fast(d, phi);
                    const float fc = fc_fast(d);
                    zc = e + 16 < e1 ? zs[w] : 0;
#pragma unroll
                    for (int j = 0; j < kK / 2; ++j) {
                        const float2 u = f2mul(make_float2(phi[2 * j], phi[2 * j + 1]), bcast(fc));
                        acc[j] = f2fma(bcast(w0), u, acc[j]);
                        acc[kK / 2 + j] = f2fma(bcast(w1), u, acc[kK / 2 + j]);
                    }
                }
            }
            float accf[kF];
#pragma unroll
            for (int i = 0; i < kF / 2; ++i) {
                accf[2 * i] = acc[i].x;
                accf[2 * i + 1] = acc[i].y;
            }
            // lane gl: Phi_{gl / 8, gl % 8} summed over the group; then m_gl
            float* T = sT + grp * GroupT<kConvTS>::kGroup;
            float4* rw = reinterpret_cast<float4*>(T + gl * kConvTS);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                rw[c] = make_float4(accf[4 * c], accf[4 * c + 1], accf[4 * c + 2], accf[4 * c + 3]);
            __syncwarp();
            const float phis = column_sum16<kConvTS>(T, gl);
            __syncwarp();
            T[gl] = phis;  // row 0 is free again: Phi broadcast
            __syncwarp();
            const float4* ph4 = reinterpret_cast<const float4*>(T);
            const float4* pe0 = reinterpret_cast<const float4*>(sPe + gl * kK);
            const float4* pe1 = reinterpret_cast<const float4*>(sPe + kF * kK + gl * kK);
            float zz = sb[gl];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const float4 p = ph4[c], q = pe0[c];
                zz = fmaf(q.x, p.x, zz);
                zz = fmaf(q.y, p.y, zz);
                zz = fmaf(q.z, p.z, zz);
                zz = fmaf(q.w, p.w, zz);
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const float4 p = ph4[2 + c], q = pe1[c];
                zz = fmaf(q.x, p.x, zz);
                zz = fmaf(q.y, p.y, zz);
                zz = fmaf(q.z, p.z, zz);
                zz = fmaf(q.w, p.w, zz);
            }
            __syncwarp();
            z = zz;
        } else {
            // one gathered row per lane in flight; index and d one slot ahead
            ConvIn x;
            for (int e = e0 + gl; __any_sync(0xffffffffu, e < e1); e += 16) {
                if (e < e1) {
                    conv_load(Hin, w, x);
                    x.d = dcur;
                    w = src_of(a, e + 16, e1);
                    dcur = d_of(a, e + 16, e1);
                    conv_math2(x, acc);
                }
            }
            float accf[kF];
#pragma unroll
            for (int i = 0; i < kF / 2; ++i) {
                accf[2 * i] = acc[i].x;
                accf[2 * i + 1] = acc[i].y;
            }
            z = conv_node_z(accf, gl, sT + grp * GroupT<kConvTS>::kGroup, sM[grp], sW, sb[gl]);
        }
        const float th = tanhf(z);
        float ev = 0.0f;
        if (valid) {
            const int64_t r = a.crow ? a.crow[v] : v;
            const float hn = Hin[r * kF + gl] + th;
            Hout[r * kF + gl] = hn;
            note_nonfinite(a, layer, r, hn);
            TH[k * kF + gl] = th;
            ev = sro[gl] * hn;
        }
        if (per_atom) {
            ev = group_sum16(ev);
            if (valid && gl == 0) {
                per_atom[v] = (double)ev;
                esum += (double)ev;
            }
        }
    }
    if (e_part) {
        double vals[1] = {esum};
        cta_partials<1, NT / 32>(vals, e_part);
    }
}

// Backward per edge e = (w -> u) in the "dsum" form (potential.cpp:823-848):
//   ds_f = sum_k P_fk psi_k,  psi_k = phi_k (ca + cb k)     (u'_k restated)
//   dbar_e + dbar_rev(e) = sum_f (mbar_u,f h_w,f + h_u,f mbar_w,f) ds_f
//                        = sum_k psi_k G_k,  G = P^T g  (128 FMA, not 2 x 128)
// grad_u -= v_e (dbar_e + dbar_rev)/d_e as before; the virial takes half of
// the pair sum per edge: the reverse edge has the same v (x) v and d, so
// sum_e dbar_e v v^T / d = 1/2 sum_e (dbar_e + dbar_rev(e)) v v^T / d over any
// edge set closed under reversal (all edges, or all in-edges of the atoms a
// rank owns, summed over ranks).
__device__ __forceinline__ void bwd_load2(const float* __restrict__ MB, const float* __restrict__ Hl,
                                          int w, BwdEdgeIn& x) {
    const float* mw = MB + (size_t)w * kF;
    const float* hw = Hl + (size_t)w * kF;
    ldg256(mw, x.m[0], x.m[1]);
    ldg256(mw + 8, x.m[2], x.m[3]);
    ldg256(hw, x.h[0], x.h[1]);
    ldg256(hw + 8, x.h[2], x.h[3]);
}

template <typename Acc, bool HBAR = true>
__device__ __forceinline__ void bwd_math2(const BwdEdgeIn& x, const float4* su_m,
                                          const float4* su_h, float isg, float mus,
                                          float2 acc[kF / 2], Acc& gx, Acc& gy, Acc& gz,
                                          float vr[6]) {
    const float4 q = x.q;
    float fc, dfc;
    fc_dfc_fast(q.w, fc, dfc);
    float phi[kK];
    phi_fast(q.w, phi);
    const float x0 = q.w * isg, step = mus * isg;
    const float ca = dfc - 2.0f * fc * isg * x0, cb = 2.0f * fc * isg * step;
    // g_f = mbar_u,f h_w,f + h_u,f mbar_w,f
    float g[kF];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float4 mu4 = su_m[c], hu4 = su_h[c];
        float2 ga, gb;
        if (sizeof(Acc) == 8) {
            // exact mode: g = 1/2 (S_u S_w - D_u D_w), S = mbar + h, D = mbar - h,
            // a form symmetric under u <-> w whatever ptxas fuses (it contracts
            // add.rn.f32x2 of two mul.rn.f32x2 into an FFMA2, which makes
            // m_u h_w + h_u m_w round differently at the two ends); the 1/2
            // is applied to dsum
            const float2 su0 = __fadd2_rn(make_float2(mu4.x, mu4.y), make_float2(hu4.x, hu4.y));
            const float2 du0 = __fadd2_rn(make_float2(mu4.x, mu4.y), make_float2(-hu4.x, -hu4.y));
            const float2 sw0 = __fadd2_rn(make_float2(x.m[c].x, x.m[c].y), make_float2(x.h[c].x, x.h[c].y));
            const float2 dw0 = __fadd2_rn(make_float2(x.m[c].x, x.m[c].y), make_float2(-x.h[c].x, -x.h[c].y));
            ga = f2fma(su0, sw0, f2mul(make_float2(-du0.x, -du0.y), dw0));
            const float2 su1 = __fadd2_rn(make_float2(mu4.z, mu4.w), make_float2(hu4.z, hu4.w));
            const float2 du1 = __fadd2_rn(make_float2(mu4.z, mu4.w), make_float2(-hu4.z, -hu4.w));
            const float2 sw1 = __fadd2_rn(make_float2(x.m[c].z, x.m[c].w), make_float2(x.h[c].z, x.h[c].w));
            const float2 dw1 = __fadd2_rn(make_float2(x.m[c].z, x.m[c].w), make_float2(-x.h[c].z, -x.h[c].w));
            gb = f2fma(su1, sw1, f2mul(make_float2(-du1.x, -du1.y), dw1));
        } else {
            ga = f2fma(make_float2(hu4.x, hu4.y), make_float2(x.m[c].x, x.m[c].y),
                       f2mul(make_float2(mu4.x, mu4.y), make_float2(x.h[c].x, x.h[c].y)));
            gb = f2fma(make_float2(hu4.z, hu4.w), make_float2(x.m[c].z, x.m[c].w),
                       f2mul(make_float2(mu4.z, mu4.w), make_float2(x.h[c].z, x.h[c].w)));
        }
        g[4 * c] = ga.x;
        g[4 * c + 1] = ga.y;
        g[4 * c + 2] = gb.x;
        g[4 * c + 3] = gb.y;
    }
    // G_(2j, 2j+1) = sum_f (P[f][2j], P[f][2j+1]) g_f
    const float2* P2 = reinterpret_cast<const float2*>(c_m.P);
    float2 G[kK / 2];
#pragma unroll
    for (int j = 0; j < kK / 2; ++j) G[j] = f2fma(P2[j], bcast(g[0]), make_float2(0.f, 0.f));
#pragma unroll
    for (int f = 1; f < kF; ++f)
#pragma unroll
        for (int j = 0; j < kK / 2; ++j) G[j] = f2fma(P2[f * (kK / 2) + j], bcast(g[f]), G[j]);
    // dsum = sum_k phi_k (ca + cb k) G_k
    float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < kK / 2; ++j) {
        const float2 ck = f2fma(bcast(cb), make_float2((float)(2 * j), (float)(2 * j + 1)), bcast(ca));
        s2 = f2fma(f2mul(make_float2(phi[2 * j], phi[2 * j + 1]), ck), G[j], s2);
    }
    const float dsum = sizeof(Acc) == 8 ? 0.5f * (s2.x + s2.y) : s2.x + s2.y;
    // hbar_u += mbar_w (.) s_e, s = fc P phi (not for layer 0: the gradient
    // with respect to the embeddings carries no position dependence)
    if constexpr (HBAR) {
        float php[kK];
#pragma unroll
        for (int k = 0; k < kK; ++k) php[k] = fc * phi[k];
        float2 A[kF / 2];
        radial_pairs(php, A);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            acc[2 * c] = f2fma(make_float2(x.m[c].x, x.m[c].y), A[2 * c], acc[2 * c]);
            acc[2 * c + 1] = f2fma(make_float2(x.m[c].z, x.m[c].w), A[2 * c + 1], acc[2 * c + 1]);
        }
    }
    const float coef = dsum / q.w;
    gx -= (Acc)(q.x * coef);
    gy -= (Acc)(q.y * coef);
    gz -= (Acc)(q.z * coef);
    const float ch = 0.5f * coef;
    vr[0] = fmaf(ch * q.x, q.x, vr[0]);
    vr[1] = fmaf(ch * q.y, q.y, vr[1]);
    vr[2] = fmaf(ch * q.z, q.z, vr[2]);
    vr[3] = fmaf(ch * q.x, q.y, vr[3]);
    vr[4] = fmaf(ch * q.x, q.z, vr[4]);
    vr[5] = fmaf(ch * q.y, q.z, vr[5]);
}

constexpr int kBwdTS = 28;  // transpose row: h_bar 16 | virial 6 | gradient 3 | pad
// SPEC (layer 0, Hl = h0 = emb[Z], at most two species): the source's h row
// is one of two embedding rows staged in shared memory, picked by its species
// byte -- bitwise the gathered row, one 64-byte gather per edge fewer.
template <int CTAS, int NT, typename Acc, bool HBAR = true, bool SPEC = false>
__global__ void __launch_bounds__(NT, CTAS) k_bwd_edge2(ConvArgs a, const float* __restrict__ MB,
                                                           const float* __restrict__ Hl,
                                                           float* __restrict__ HB,
                                                           double4* __restrict__ GRAD,
                                                           double* vir_part, double* vir_grp,
                                                           const uint8_t* __restrict__ zs = nullptr,
                                                           const unsigned* __restrict__ zmask = nullptr) {
    __shared__ __align__(16) float sU[(NT / 16)][2][kF];  // [group][m_bar_u, h_u][f]
    __shared__ double sVir[(NT / 16)][6];
    __shared__ __align__(16) float sE[SPEC ? 2 * kF : 4];  // emb rows of the two species
    int z1 = -1;
    bool spec = false;
    if constexpr (SPEC) {
        int z0 = -1, ns = 0;
        for (int w = 0; w < 4; ++w) {
            unsigned m = zmask[w];
            ns += __popc(m);
            while (m) {
                const int z = 32 * w + __ffs(m) - 1;
                m &= m - 1u;
                if (z0 < 0) z0 = z; else if (z1 < 0) z1 = z;
            }
        }
        if (z1 < 0) z1 = z0;
        spec = ns <= 2;
        if (threadIdx.x < 2 * kF) sE[threadIdx.x] = c_m.emb[(threadIdx.x < kF ? z0 : z1) * kF + (threadIdx.x % kF)];
        __syncthreads();
    }
    extern __shared__ __align__(16) float sT[];  // fp32 path: (NT / 16) transpose groups
    const int lane = threadIdx.x & 31;
    const int gl = lane & 15, grp = threadIdx.x >> 4;
    const int64_t g0 = (int64_t)blockIdx.x * (NT / 16) + grp;
    const int64_t ng = (int64_t)gridDim.x * (NT / 16);
    const float isg = c_m.inv_sigma, mus = c_m.mu_step;
    // vir_grp (node-chunked launches, k0 a multiple of ng): every group's
    // running virial sum carries over from the previous chunk, so the fp64
    // accumulation order is exactly the unchunked launch's
    if (gl < 6) sVir[grp][gl] = (vir_grp && a.k0 > 0) ? vir_grp[(size_t)g0 * 6 + gl] : 0.0;
    const int64_t iters = (a.n - a.k0 + ng - 1) / ng;  // nodes [k0, n)
    int e0n = 0, e1n = 0;
    float mun = 0.f, hun = 0.f;
    BwdEdgeIn xa;
    int wa = 0;
    float4 qa = make_float4(0.f, 0.f, 0.f, 1.f);
    // node k's row bounds, own rows and first source index are loaded while
    // the previous node finishes
    auto prefetch = [&](int64_t k) {
        if (k < a.n) {
            const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
            const int64_t r = a.crow ? a.crow[v] : v;
            e0n = __ldg(a.row + v);
            e1n = __ldg(a.row + v + 1);
            mun = __ldg(MB + r * kF + gl);
            hun = __ldg(Hl + r * kF + gl);
            wa = src_of(a, e0n + gl, e1n);
            qa = vd_of(a, e0n + gl, e1n);
        } else {
            e0n = e1n = 0;
        }
    };
    prefetch(a.k0 + g0);
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t k = a.k0 + g0 + it * ng;
        const bool valid = k < a.n;
        const int e0 = e0n, e1 = e1n;
        __syncwarp();
        if (valid) {
            sU[grp][0][gl] = mun;
            sU[grp][1][gl] = hun;
        }
        __syncwarp();
        float2 acc[kF / 2];
#pragma unroll
        for (int i = 0; i < kF / 2; ++i) acc[i] = make_float2(0.f, 0.f);
        Acc gx = 0, gy = 0, gz = 0;
        float vr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const float4* su_m = reinterpret_cast<const float4*>(sU[grp][0]);
        const float4* su_h = reinterpret_cast<const float4*>(sU[grp][1]);
        for (int e = e0 + gl; __any_sync(0xffffffffu, e < e1); e += 16) {
            if (e < e1) {
                if (SPEC && spec) {
                    const float* mw = MB + (size_t)wa * kF;
                    ldg256(mw, xa.m[0], xa.m[1]);
                    ldg256(mw + 8, xa.m[2], xa.m[3]);
                    const float4* er = reinterpret_cast<const float4*>(sE + (zs[wa] == z1 ? kF : 0));
#pragma unroll
                    for (int c = 0; c < 4; ++c) xa.h[c] = er[c];
                } else {
                    bwd_load2(MB, Hl, wa, xa);
                }
                xa.q = qa;
                wa = src_of(a, e + 16, e1);
                qa = vd_of(a, e + 16, e1);
                bwd_math2<Acc, HBAR>(xa, su_m, su_h, isg, mus, acc, gx, gy, gz, vr);
            }
        }
        prefetch(k + ng);
        if constexpr (sizeof(Acc) == 4) {
            // one shared-memory transpose for h_bar (16), the virial (6) and
            // the gradient (3): lane gl sums column gl, lanes 0..8 column 16+gl
            // the node's current h_bar / gradient words: read first, written
            // back after the transpose (one writer per element, no atomics)
            float hbo = 0.f;
            double gro = 0.0;
            if (valid) {
                if (HBAR) hbo = HB[k * kF + gl];
                if (gl >= 6 && gl < 9) gro = reinterpret_cast<const double*>(GRAD + k)[gl - 6];
            }
            float* T = sT + grp * GroupT<kBwdTS>::kGroup;
            float4* rw = reinterpret_cast<float4*>(T + gl * kBwdTS);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                rw[c] = make_float4(acc[2 * c].x, acc[2 * c].y, acc[2 * c + 1].x, acc[2 * c + 1].y);
            rw[4] = make_float4(vr[0], vr[1], vr[2], vr[3]);
            rw[5] = make_float4(vr[4], vr[5], (float)gx, (float)gy);
            T[gl * kBwdTS + 24] = (float)gz;
            __syncwarp();
            const float hb = HBAR ? column_sum16<kBwdTS>(T, gl) : 0.f;
            const float xs = column_sum16<kBwdTS>(T, 16 + (gl < 9 ? gl : 0));
            if (gl < 6) sVir[grp][gl] += (double)xs;
            // node k belongs to this group alone and each kernel adds once
            if (valid) {
                if (HBAR) HB[k * kF + gl] = hbo + hb;
                if (gl >= 6 && gl < 9) reinterpret_cast<double*>(GRAD + k)[gl - 6] = gro + (double)xs;
            }
        } else {
#pragma unroll
            for (int c = 0; c < 6; ++c) vr[c] = group_sum16(vr[c]);
            if (gl == 0)
#pragma unroll
                for (int c = 0; c < 6; ++c) sVir[grp][c] += (double)vr[c];
            float accf[kF];
#pragma unroll
            for (int i = 0; i < kF / 2; ++i) {
                accf[2 * i] = acc[i].x;
                accf[2 * i + 1] = acc[i].y;
            }
            const float hb = transpose_reduce16_g16(accf, gl);
            const double sx = group_sum16d(gx), sy = group_sum16d(gy), sz = group_sum16d(gz);
            if (valid) {  // fp64 gradient lanes: one writer per element
                if (HBAR) HB[k * kF + gl] += hb;
                if (gl == 0) grad_add(GRAD, k, sx, sy, sz);
            }
        }
    }
    __syncwarp();
    if (vir_grp && gl < 6) vir_grp[(size_t)g0 * 6 + gl] = sVir[grp][gl];
    __syncthreads();
    if (threadIdx.x < 6) {
        double acc6 = 0.0;
        for (int g = 0; g < (NT / 16); ++g) acc6 += sVir[g][threadIdx.x];
        vir_part[(size_t)blockIdx.x * 6 + threadIdx.x] = acc6;
    }
}

// ---------------------------------------------------------------------------
// Backward edge pass on the 5th-gen tensor cores (tcgen05 + TMEM).
//
// Rows of a 128-row tile are 8 chunks of 16 edge slots; a chunk holds up to 16
// consecutive in-edges of ONE node (a node of degree d uses ceil(d/16)
// chunks), so every chunk reduces with a fixed half-warp tree and a node's
// total is its chunk sums in chunk order -- independent of how nodes are
// spread over CTAs/tiles (partition- and rank-invariant results).
// Per tile: phi[slot][k] (SFU) -> tf32 hi/lo, K-major in shared memory; one
// thread issues D = phi_hi.Pc_hi + phi_lo.Pc_hi + phi_hi.Pc_lo (M=128, N=32,
// K=8, kind::tf32, Pc = [P ; kP]) into TMEM; the epilogue reads its row
// (LDTM): A_f = sum_k P_fk phi_k, B_f = sum_k k P_fk phi_k, and forms
// s_f = fc A_f, ds_f = ca A_f + cb B_f and the products of k_bwd_edge.
// ---------------------------------------------------------------------------
constexpr int kTM = 128;  // rows per tile = threads = MMA M
constexpr int kCH = 16;   // edge slots per chunk
constexpr int kNCH = kTM / kCH;
constexpr int kNV = 19;   // per-node values: 16 h_bar, 3 grad
constexpr int kBwdTcCtas = 4;   // resident CTAs per SM (shared memory bound)
constexpr int kRowStride = 36;  // floats per staged edge row: m_bar 16 | h 16 | pad (bank spread)

// Pipeline per CTA (tile u): indices of tile u+1 and the chunk records of
// tile u+2 are loaded while phi(u) is formed; after MMA(u) is issued the
// gathered rows of tile u+1 are copied into the other shared-memory buffer
// with cp.async, so they are in flight during the epilogue of tile u.
struct BwdTcSmem {
    float a_hi[kTM * kK], a_lo[kTM * kK];   // phi, K-major interleaved (gmd_tc.cuh)
    float b_hi[32 * kK], b_lo[32 * kK];     // [P ; kP]
    alignas(16) float rows[2][kTM * kRowStride];  // gathered m_bar[w], h[w] per slot
    alignas(16) float own[2][kNCH][2 * kF];       // m_bar, h rows of each chunk's node
    float csum[kNCH][kNV + 1];              // chunk sums of the current tile (h_bar)
    double gsum[kNCH][3];                   // chunk sums of the positional gradient
    int cnode[2][kNCH];                     // node (local index) of each chunk, -1: none
    int clast[2][kNCH];                     // chunk is its node's last chunk
    uint64_t mbar;
    uint32_t tbase;
};

__device__ __forceinline__ int64_t node_gid(const ConvArgs& a, int64_t k) {
    return a.nodes ? (int64_t)a.nodes[k] : k;
}

// chunk records: {first edge, node k, node's canonical row, len | last << 8}
__global__ void k_chunk_count(ConvArgs a, int32_t* __restrict__ cnt) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k > a.n) return;
    if (k == a.n) {
        cnt[k] = 0;
        return;
    }
    const int64_t v = node_gid(a, k);
    cnt[k] = (a.row[v + 1] - a.row[v] + kCH - 1) / kCH;
}

__global__ void k_chunk_fill(ConvArgs a, const int32_t* __restrict__ cstart, int4* __restrict__ tab) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= a.n) return;
    const int64_t v = node_gid(a, k);
    const int e0 = a.row[v], deg = a.row[v + 1] - e0;
    const int r = a.crow ? a.crow[v] : (int)v;
    const int nch = (deg + kCH - 1) / kCH;
    int4* t = tab + cstart[k];
    for (int c = 0; c < nch; ++c)
        t[c] = make_int4(e0 + c * kCH, (int)k, r, min(kCH, deg - c * kCH) | ((c == nch - 1) << 8));
}

// CTA b takes chunks [cta[b], cta[b+1]): equal chunk counts, cut at node starts
__global__ void k_chunk_cta(int64_t n, const int32_t* __restrict__ cstart, int grid,
                            int32_t* __restrict__ cta) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > grid) return;
    const int64_t T = cstart[n];
    const int64_t target = T * b / grid;
    int64_t lo = 0, hi = n;  // first k with cstart[k] >= target
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cstart[mid] >= target) hi = mid; else lo = mid + 1;
    }
    cta[b] = cstart[lo];
}

__device__ __forceinline__ void stage_edge_rows(float* dst, const float* __restrict__ MB,
                                                const float* __restrict__ Hl, int w) {
    const float* m = MB + (size_t)w * kF;
    const float* hh = Hl + (size_t)w * kF;
#pragma unroll
    for (int i = 0; i < 4; ++i) tc::cp_async16(dst + 4 * i, m + 4 * i);
#pragma unroll
    for (int i = 0; i < 4; ++i) tc::cp_async16(dst + kF + 4 * i, hh + 4 * i);
}

__global__ void __launch_bounds__(kTM, kBwdTcCtas) k_bwd_edge_tc(
    ConvArgs a, const int4* __restrict__ ctab, const int32_t* __restrict__ ccta,
    const float* __restrict__ MB, const float* __restrict__ Hl, float* __restrict__ HB,
    double4* __restrict__ GRAD, double* vir_part) {
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    BwdTcSmem& S = *reinterpret_cast<BwdTcSmem*>(tc_smem);
    const int tid = threadIdx.x, lane = tid & 31;
    const int ch = tid / kCH, gl = tid % kCH;  // chunk of this thread, lane in chunk
    const int c_lo = ccta[blockIdx.x], c_hi = ccta[blockIdx.x + 1];
    const int ntiles = (c_hi - c_lo + kNCH - 1) / kNCH;
    const float isg = c_m.inv_sigma, mus = c_m.mu_step;

    for (int i = tid; i < 32 * kK; i += kTM) {
        const int nrow = i / kK, k = i % kK;
        const float x = nrow < kF ? c_m.P[nrow * kK + k] : c_m.Pk[(nrow - kF) * kK + k];
        float h, l;
        tc::split_tf32(x, h, l);
        S.b_hi[tc::kmajor_off(nrow, k)] = h;
        S.b_lo[tc::kmajor_off(nrow, k)] = l;
    }
    if (tid == 0) {
        tc::mbar_init(&S.mbar, 1);
        tc::fence_mbar_init();
    }
    if (tid < 32) tc::tmem_alloc(&S.tbase, 32);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = S.tbase;
    const uint32_t idesc = tc::idesc_tf32(kTM, 32);
    const uint32_t trow = tmem + ((uint32_t)(32 * (tid >> 5)) << 16);

    auto chunk_of = [&](int u) -> int4 {
        const int c = c_lo + u * kNCH + ch;
        return (u < ntiles && c < c_hi) ? __ldg(ctab + c) : make_int4(0, -1, 0, 0);
    };
    auto stage_own = [&](int buf, const int4& c) {  // 8 lanes x 16 B per chunk
        if (c.y >= 0 && gl < 8)
            tc::cp_async16(&S.own[buf][ch][(gl >> 2) * kF + (gl & 3) * 4],
                           (gl < 4 ? MB : Hl) + (size_t)c.z * kF + (gl & 3) * 4);
    };

    // prologue: tile 0 staged, tile 1 records loaded
    int4 ci = chunk_of(0);
    int4 cn = chunk_of(1);
    bool valid = ci.y >= 0 && gl < (ci.w & 0xff);
    float4 q = make_float4(0.f, 0.f, 0.f, 1.f);
    if (valid) {
        q = __ldg(a.vd + ci.x + gl);
        stage_edge_rows(S.rows[0] + tid * kRowStride, MB, Hl, __ldg(a.lsrc + ci.x + gl));
    }
    stage_own(0, ci);
    tc::cp_async_commit();

    double vir[6] = {0, 0, 0, 0, 0, 0};
    double carry = 0.0;  // h_bar chunk sums stay fp32 values (exact in fp64)
    int carry_node = -1;
    uint32_t phase = 0;
    for (int u = 0; u < ntiles; ++u) {
        const int buf = u & 1;
        // (1) indices of tile u+1, records of tile u+2
        const bool vn = cn.y >= 0 && gl < (cn.w & 0xff);
        float4 qn = make_float4(0.f, 0.f, 0.f, 1.f);
        int wn = 0;
        if (vn) {
            qn = __ldg(a.vd + cn.x + gl);
            wn = __ldg(a.lsrc + cn.x + gl);
        }
        const int4 cn2 = chunk_of(u + 2);
        if (gl == 0) {
            S.cnode[buf][ch] = ci.y;
            S.clast[buf][ch] = ci.y >= 0 && (ci.w >> 8);
        }
        // (2) phi(u) -> A operand (tf32 hi/lo)
        {
            float phi[kK];
            phi_fast(q.w, phi);
#pragma unroll
            for (int k = 0; k < kK; ++k) {
                float hv = 0.f, lv = 0.f;
                if (valid) tc::split_tf32(phi[k], hv, lv);
                S.a_hi[tc::kmajor_off(tid, k)] = hv;
                S.a_lo[tc::kmajor_off(tid, k)] = lv;
            }
        }
        tc::fence_async_smem();
        tc::cp_async_wait_all();  // rows(u), own(u) of this thread have landed
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (tid == 0) {
            tc::mma_tf32(tmem, tc::sdesc(S.a_hi), tc::sdesc(S.b_hi), idesc, false);
            tc::mma_tf32(tmem, tc::sdesc(S.a_lo), tc::sdesc(S.b_hi), idesc, true);
            tc::mma_tf32(tmem, tc::sdesc(S.a_hi), tc::sdesc(S.b_lo), idesc, true);
            tc::commit(&S.mbar);
        }
        // (3) stage tile u+1 while MMA(u) and the epilogue run
        if (vn) stage_edge_rows(S.rows[buf ^ 1] + tid * kRowStride, MB, Hl, wn);
        stage_own(buf ^ 1, cn);
        tc::cp_async_commit();
        // (4) epilogue(u)
        tc::mbar_wait(&S.mbar, phase);
        phase ^= 1u;
        tc::fence_after();
        float AB[32];
        tc::tmem_ld32(trow, AB);
        double gx = 0.0, gy = 0.0, gz = 0.0;
        if (valid) {
            float fc, dfc;
            fc_dfc_fast(q.w, fc, dfc);
            const float x0 = q.w * isg, step = mus * isg;
            const float ca = dfc - 2.0f * fc * isg * x0, cb = 2.0f * fc * isg * step;
            float dself = 0.f, drev = 0.f;
            const float* rw = S.rows[buf] + tid * kRowStride;
            const float* ow = S.own[buf][ch];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float4 m4 = *reinterpret_cast<const float4*>(rw + 4 * c);
                const float4 h4 = *reinterpret_cast<const float4*>(rw + kF + 4 * c);
                const float4 uu = *reinterpret_cast<const float4*>(ow + 4 * c);
                const float4 hh = *reinterpret_cast<const float4*>(ow + kF + 4 * c);
                const float mw[4] = {m4.x, m4.y, m4.z, m4.w};
                const float hw[4] = {h4.x, h4.y, h4.z, h4.w};
                const float mu[4] = {uu.x, uu.y, uu.z, uu.w};
                const float hu[4] = {hh.x, hh.y, hh.z, hh.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int f = 4 * c + i;
                    const float A = AB[f], B = AB[kF + f];
                    const float ds = fmaf(ca, A, cb * B);
                    AB[f] = mw[i] * (fc * A);
                    dself = fmaf(mu[i] * hw[i], ds, dself);
                    drev = fmaf(mw[i] * hu[i], ds, drev);
                }
            }
            const float invd = 1.0f / q.w;
            const float coef = (dself + drev) * invd;
            gx = -(double)(q.x * coef);
            gy = -(double)(q.y * coef);
            gz = -(double)(q.z * coef);
            const double cself = (double)(dself * invd);
            vir[0] += cself * q.x * q.x;
            vir[1] += cself * q.y * q.y;
            vir[2] += cself * q.z * q.z;
            vir[3] += cself * q.x * q.y;
            vir[4] += cself * q.x * q.z;
            vir[5] += cself * q.y * q.z;
        } else {
#pragma unroll
            for (int f = 0; f < kF; ++f) AB[f] = 0.f;
        }
        // (5) chunk sums: fixed half-warp trees
        const float hsum = transpose_reduce16_g16(AB, gl);  // feature gl
        gx = group_sum16d(gx);
        gy = group_sum16d(gy);
        gz = group_sum16d(gz);
        S.csum[ch][gl] = hsum;
        if (gl == 0) {
            S.gsum[ch][0] = gx;
            S.gsum[ch][1] = gy;
            S.gsum[ch][2] = gz;
        }
        tc::fence_before();
        __syncthreads();
        // (6) node totals in chunk order (carried across tiles); one adder
        // per (node, value), so the reductions below are deterministic
        if (tid < kNV) {
#pragma unroll 1
            for (int k2 = 0; k2 < kNCH; ++k2) {
                const int j = S.cnode[buf][k2];
                if (j < 0) break;
                const double x = tid < kF ? (double)S.csum[k2][tid] : S.gsum[k2][tid - kF];
                carry = j == carry_node ? carry + x : x;
                carry_node = j;
                if (S.clast[buf][k2]) {  // one writer per (node, value)
                    if (tid < kF)
                        HB[(size_t)j * kF + tid] += (float)carry;
                    else
                        reinterpret_cast<double*>(GRAD + j)[tid - kF] += carry;
                    carry_node = -1;
                }
            }
        }
        ci = cn;
        cn = cn2;
        q = qn;
        valid = vn;
    }
    tc::cp_async_wait_all();
    // fp64 virial: thread -> warp -> CTA in fixed order -> vir_part[blockIdx.x]
    __shared__ double wv[kTM / 32][6];
#pragma unroll
    for (int c = 0; c < 6; ++c) {
        double vsum = vir[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
        if (lane == 0) wv[tid >> 5][c] = vsum;
    }
    __syncthreads();
    if (tid < 6) {
        double acc6 = 0.0;
        for (int w = 0; w < kTM / 32; ++w) acc6 += wv[w][tid];
        vir_part[(size_t)blockIdx.x * 6 + tid] = acc6;
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid < 32) tc::tmem_free(tmem, 32);
}

// ---------------------------------------------------------------------------
// three-body stage (potential.cpp:664-741 forward, :850-961 backward)
// ---------------------------------------------------------------------------
constexpr int kTbWarps = 4;
// a 16-lane group per center: centers have ~11 in-bonds (C4: 11.3), so a
// warp per center left two thirds of its lanes idle
constexpr int kTbGroups = kTbWarps * 2;
constexpr size_t kTbSlotBytes = 6 * sizeof(float4) + sizeof(float4);  // backward: u3, u3', E (8 each) + v

// The three-body contractions run on packed FP32 like the atom channel
// (FFMA2 over feature pairs, constant pairs from uniform registers); each
// lane-half performs the scalar kernel's FMAs in the same order, so results
// are bitwise those of the scalar form.
// out_f = sum_k M[f][k] x_k (ascending k) from the k-major copy MT
__device__ __forceinline__ void fk_pairs(const float* MT, const float x[kK], float out[kF]) {
    const float2* M2 = reinterpret_cast<const float2*>(MT);
    float2 o[kF / 2];
#pragma unroll
    for (int i = 0; i < kF / 2; ++i) o[i] = f2mul(M2[i], bcast(x[0]));
#pragma unroll
    for (int k = 1; k < kK; ++k)
#pragma unroll
        for (int i = 0; i < kF / 2; ++i) o[i] = f2fma(M2[k * (kF / 2) + i], bcast(x[k]), o[i]);
#pragma unroll
    for (int i = 0; i < kF / 2; ++i) {
        out[2 * i] = o[i].x;
        out[2 * i + 1] = o[i].y;
    }
}
// out_g = sum_f A[f][g] y_f (ascending f), A row-major F x F: (A[f][g], A[f][g+1]) pairs
__device__ __forceinline__ void ff_pairs(const float* A, const float y[kF], float out[kF]) {
    const float2* A2 = reinterpret_cast<const float2*>(A);
    float2 o[kF / 2];
#pragma unroll
    for (int i = 0; i < kF / 2; ++i) o[i] = f2mul(A2[i], bcast(y[0]));
#pragma unroll
    for (int f = 1; f < kF; ++f)
#pragma unroll
        for (int i = 0; i < kF / 2; ++i) o[i] = f2fma(A2[f * (kF / 2) + i], bcast(y[f]), o[i]);
#pragma unroll
    for (int i = 0; i < kF / 2; ++i) {
        out[2 * i] = o[i].x;
        out[2 * i + 1] = o[i].y;
    }
}

__device__ __forceinline__ void bond_t(float d, float t[kF]) {
    float u[kK];
    basis(d, c_m.r3, c_m.inv_r3, c_m.inv_sigma3, c_m.mu_step3, u);
    fk_pairs(c_m.P3T, u, t);  // t_f = sum_k P3[f][k] u_k
}

// per center s: for each in-bond slot j (bond e1 = (w->s)), compute t' of the
// reverse bond e' = (s->w): m3_{e'} = sum_{e2 != e1} c(e2, e') t_{e2} in
// ascending e2, z3 = W3 m3, t' = t + fc3 tanh(z3).  Stored at slot j.
// per-group staging sized by kc >= the build's max in-bonds (dynamic shared
// memory: C4's 16-slot groups need 10 KB per CTA instead of 40 KB)
__global__ void __launch_bounds__(kTbWarps * 32) k_tb_forward(BondArgs a, float* __restrict__ TP,
                                                              float* __restrict__ TH3,
                                                              int32_t* flags, int kc) {
    extern __shared__ __align__(16) unsigned char tbf_smem[];
    const int gl = threadIdx.x & 15, grp = threadIdx.x >> 4;
    float(*st_g)[kF] = reinterpret_cast<float(*)[kF]>(tbf_smem) + (size_t)grp * kc;
    float4* sv_g = reinterpret_cast<float4*>(tbf_smem + sizeof(float) * kF * kTbGroups * kc) +
                   (size_t)grp * kc;
    const int64_t w0 = (int64_t)blockIdx.x * kTbGroups + grp;
    const int64_t nw = (int64_t)gridDim.x * kTbGroups;
    const int64_t iters = (a.n + nw - 1) / nw;  // same count for both groups of a warp
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t ks = w0 + it * nw;
        int b0 = 0, k = 0;
        if (ks < a.n) {
            const int64_t s = a.nodes ? (int64_t)a.nodes[ks] : ks;
            b0 = a.brow[s];
            k = a.brow[s + 1] - b0;
            if (k > kc) {  // only when k > kMaxBondsPerAtom (kc covers the build's max)
                if (gl == 0) atomicOr(&flags[1], 16);
                k = 0;
            }
        }
        for (int j = gl; j < k; j += 16) {
            float4 q = __ldg(a.vd + a.bedge[b0 + j]);
            sv_g[j] = q;
            float t[kF];
            bond_t(q.w, t);
#pragma unroll
            for (int f = 0; f < kF; ++f) st_g[j][f] = t[f];
        }
        __syncwarp();
        for (int j = gl; j < k; j += 16) {
            const float4 qj = sv_g[j];
            float2 m32[kF / 2];  // feature pairs, packed FP32
#pragma unroll
            for (int i = 0; i < kF / 2; ++i) m32[i] = make_float2(0.f, 0.f);
            for (int e2 = 0; e2 < k; ++e2) {
                if (e2 == j) continue;  // the reverse pair (linegraph.cpp:16-21)
                const float4 q2 = sv_g[e2];
                const float c = (q2.x * qj.x + q2.y * qj.y + q2.z * qj.z) / (q2.w * qj.w);
                const float2* t2 = reinterpret_cast<const float2*>(st_g[e2]);
#pragma unroll
                for (int i = 0; i < kF / 2; ++i) m32[i] = f2fma(bcast(c), t2[i], m32[i]);
            }
            float m3[kF];
#pragma unroll
            for (int i = 0; i < kF / 2; ++i) {
                m3[2 * i] = m32[i].x;
                m3[2 * i + 1] = m32[i].y;
            }
            float fc, dfc;
            fcut3(qj.w, fc, dfc);
            float tp[kF], th[kF], z[kF];
            ff_pairs(c_m.W3T, m3, z);  // z_f = sum_g W3[f][g] m3_g
#pragma unroll
            for (int f = 0; f < kF; ++f) {
                th[f] = tanhf(z[f]);
                tp[f] = st_g[j][f] + fc * th[f];
            }
            store_row16(TP + (size_t)(b0 + j) * kF, tp);
            store_row16(TH3 + (size_t)(b0 + j) * kF, th);
        }
        __syncwarp();
    }
}

// q_u = sum_{b into u} t'_b (ascending b), h_u += tanh(W4 q_u)
__global__ void k_tb_inject(BondArgs a, const float* __restrict__ TP, float* __restrict__ H,
                            float* __restrict__ TH4) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.n) return;
    const int64_t u = a.nodes ? (int64_t)a.nodes[k] : k;
    float q[kF];
#pragma unroll
    for (int f = 0; f < kF; ++f) q[f] = 0.f;
    for (int b = a.brow[u]; b < a.brow[u + 1]; ++b) {
        float t[kF];
        load_row16(TP + (size_t)a.brev[b] * kF, t);
#pragma unroll
        for (int f = 0; f < kF; ++f) q[f] += t[f];
    }
    const int64_t r = a.crow ? a.crow[u] : u;
    float h[kF], th[kF], z[kF];
    load_row16(H + r * kF, h);
    ff_pairs(c_m.W4T, q, z);  // z_f = sum_g W4[f][g] q_g
#pragma unroll
    for (int f = 0; f < kF; ++f) {
        th[f] = tanhf(z[f]);
        h[f] += th[f];
    }
    store_row16(H + r * kF, h);
    store_row16(TH4 + k * kF, th);
}

__global__ void k_tb_bwd_q(int64_t n, const int32_t* __restrict__ nodes,
                           const int32_t* __restrict__ crow, const float* __restrict__ HB,
                           const float* __restrict__ TH4, float* __restrict__ QB) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t v = nodes ? (int64_t)nodes[k] : k;
    float hb[kF], th[kF], y[kF], qb[kF];
    load_row16(HB + k * kF, hb);
    load_row16(TH4 + k * kF, th);
#pragma unroll
    for (int f = 0; f < kF; ++f) y[f] = hb[f] * (1.0f - th[f] * th[f]);
    ff_pairs(c_m.W4, y, qb);  // qb_g = sum_f W4[f][g] y_f
    store_row16(QB + (crow ? (int64_t)crow[v] : v) * kF, qb);
}

// Per center s.  Slot j holds in-bond e_j = (w_j -> s); its reverse e'_j is
// the out-bond (s -> w_j).  VOUT[j] collects the gradient w.r.t. v_{e'_j}
// produced here (fc3 path, identity part of the bond-init adjoint, cos
// gradient of e'_j); VIN[j] the gradient w.r.t. v_{e_j} produced here
// (cos gradient of e_j, line-edge part of its bond-init adjoint).
template <int MINB>
__global__ void __launch_bounds__(kTbWarps * 32, MINB) k_tb_backward(BondArgs a,
                                                               const float* __restrict__ QB,
                                                               const float* __restrict__ TH3,
                                                               float4* __restrict__ VIN,
                                                               float4* __restrict__ VOUT,
                                                               double* vir_part, int kc) {
    // per-group staging of kc >= max in-bonds slots: bond vector, basis u3,
    // its derivative u3' and E = P3^T m_bar_3 (8 floats each)
    extern __shared__ __align__(16) unsigned char tb_smem[];
    const int gl = threadIdx.x & 15, grp = threadIdx.x >> 4;
    float4* sv = reinterpret_cast<float4*>(tb_smem) + (size_t)grp * kc;
    float4* su = reinterpret_cast<float4*>(tb_smem) + (size_t)kTbGroups * kc + (size_t)grp * kc * 2;
    float4* sdu = su + (size_t)kTbGroups * kc * 2;
    float4* sE = sdu + (size_t)kTbGroups * kc * 2;
    const int64_t w0 = (int64_t)blockIdx.x * kTbGroups + grp;
    const int64_t nw = (int64_t)gridDim.x * kTbGroups;
    const int64_t iters = (a.n + nw - 1) / nw;  // same count for both groups of a warp
    double vir[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t ks = w0 + it * nw;
        int b0 = 0, k = 0;
        if (ks < a.n) {
            const int64_t s = a.nodes ? (int64_t)a.nodes[ks] : ks;
            b0 = a.brow[s];
            k = a.brow[s + 1] - b0;
            if (k > kc) k = 0;  // > kMaxBondsPerAtom: flagged in the forward
        }
        for (int j = gl; j < k; j += 16) {
            const int e = a.bedge[b0 + j];
            const float4 q = __ldg(a.vd + e);
            sv[j] = q;
            float u[kK], du[kK];
            basis_d(q.w, c_m.r3, c_m.inv_r3, c_m.inv_sigma3, c_m.mu_step3, u, du);
            su[2 * j] = make_float4(u[0], u[1], u[2], u[3]);
            su[2 * j + 1] = make_float4(u[4], u[5], u[6], u[7]);
            sdu[2 * j] = make_float4(du[0], du[1], du[2], du[3]);
            sdu[2 * j + 1] = make_float4(du[4], du[5], du[6], du[7]);
            // stage 2: adjoints of the reverse bond e'_j
            float tpb[kF], th[kF], ds[kF];
            const int x = __ldg(a.esrc + e);
            load_row16(QB + (size_t)(a.crow ? a.crow[x] : x) * kF, tpb);
            load_row16(TH3 + (size_t)(b0 + j) * kF, th);
            float fc, dfc;
            fcut3(q.w, fc, dfc);
            fk_pairs(c_m.P3T, du, ds);  // ds = P3 u3'
            float dbf = 0.f, da = 0.f, y[kF];
#pragma unroll
            for (int f = 0; f < kF; ++f) {
                dbf = fmaf(tpb[f] * th[f], dfc, dbf);
                da = fmaf(tpb[f], ds[f], da);
                y[f] = tpb[f] * fc * (1.0f - th[f] * th[f]);
            }
            // E = P3^T m_bar_3 = (W3 P3)^T y: phase 2 needs m_bar_3 only
            // through m_bar_3 . t = E . u3 and m_bar_3 . ds = E . u3'
            const float2* B2 = reinterpret_cast<const float2*>(c_m.B3);
            float2 E2[kK / 2];
#pragma unroll
            for (int i = 0; i < kK / 2; ++i) E2[i] = f2mul(B2[i], bcast(y[0]));
#pragma unroll
            for (int f = 1; f < kF; ++f)
#pragma unroll
                for (int i = 0; i < kK / 2; ++i) E2[i] = f2fma(B2[f * (kK / 2) + i], bcast(y[f]), E2[i]);
            sE[2 * j] = make_float4(E2[0].x, E2[0].y, E2[1].x, E2[1].y);
            sE[2 * j + 1] = make_float4(E2[2].x, E2[2].y, E2[3].x, E2[3].y);
            const float c0 = -(dbf + da) / q.w;
            VOUT[b0 + j] = make_float4(q.x * c0, q.y * c0, q.z * c0, 0.f);
        }
        __syncwarp();
        auto dot8 = [](float4 a0, float4 a1, float4 b0_, float4 b1_) {
            float2 r = f2mul(make_float2(a0.x, a0.y), make_float2(b0_.x, b0_.y));
            r = f2fma(make_float2(a0.z, a0.w), make_float2(b0_.z, b0_.w), r);
            r = f2fma(make_float2(a1.x, a1.y), make_float2(b1_.x, b1_.y), r);
            r = f2fma(make_float2(a1.z, a1.w), make_float2(b1_.z, b1_.w), r);
            return r.x + r.y;
        };
        for (int j = gl; j < k; j += 16) {
            const float4 qj = sv[j];
            const float idj = 1.0f / qj.w;
            const float4 uj0 = su[2 * j], uj1 = su[2 * j + 1];
            const float4 dj0 = sdu[2 * j], dj1 = sdu[2 * j + 1];
            const float4 Ej0 = sE[2 * j], Ej1 = sE[2 * j + 1];
            float db = 0.f;
            float vix = 0.f, viy = 0.f, viz = 0.f;  // as incoming bond e = e_j
            float4 vo = VOUT[b0 + j];                // as outgoing bond e' = e'_j
            for (int o = 0; o < k; ++o) {
                if (o == j) continue;
                const float4 qo = sv[o];
                const float ido = 1.0f / qo.w;
                const float dotjo = qj.x * qo.x + qj.y * qo.y + qj.z * qo.z;
                const float c = dotjo * idj * ido;
                const float4 Eo0 = sE[2 * o], Eo1 = sE[2 * o + 1];
                // (a) line edge (e_j, e'_o): c = v_j.v_o/(d_j d_o), a = v_j, b = -v_o;
                //     t_bar_j += c m_bar_3,o (contracted with ds_j below)
                {
                    const float cb = dot8(Eo0, Eo1, uj0, uj1);  // m_bar_3,o . t_j
                    db = fmaf(c, dot8(Eo0, Eo1, dj0, dj1), db);  // c m_bar_3,o . ds_j
                    // dc/da = -(b^ + a^ c)/|a|
                    vix += -(-qo.x * ido + qj.x * idj * c) * idj * cb;
                    viy += -(-qo.y * ido + qj.y * idj * c) * idj * cb;
                    viz += -(-qo.z * ido + qj.z * idj * c) * idj * cb;
                }
                // (b) line edge (e_o, e'_j): a = v_o, b = -v_j
                {
                    const float cb = dot8(Ej0, Ej1, su[2 * o], su[2 * o + 1]);  // m_bar_3,j . t_o
                    // dc/db = -(a^ + b^ c)/|b|
                    vo.x += -(qo.x * ido - qj.x * idj * c) * idj * cb;
                    vo.y += -(qo.y * ido - qj.y * idj * c) * idj * cb;
                    vo.z += -(qo.z * ido - qj.z * idj * c) * idj * cb;
                }
            }
            vix += qj.x * db * idj;
            viy += qj.y * db * idj;
            viz += qj.z * db * idj;
            VIN[b0 + j] = make_float4(vix, viy, viz, 0.f);
            VOUT[b0 + j] = vo;
            const double dx = (double)vix - vo.x, dy = (double)viy - vo.y, dz = (double)viz - vo.z;
            vir[0] += dx * qj.x;
            vir[1] += dx * qj.y;
            vir[2] += dx * qj.z;
            vir[3] += dy * qj.x;
            vir[4] += dy * qj.y;
            vir[5] += dy * qj.z;
            vir[6] += dz * qj.x;
            vir[7] += dz * qj.y;
            vir[8] += dz * qj.z;
        }
        __syncwarp();
    }
    cta_partials<9>(vir, vir_part);
}

// grad[u] += sum_{X into u} (v_bar of rev(X)) - (v_bar of X)
__global__ void k_tb_grad(BondArgs a, const float4* __restrict__ VIN,
                          const float4* __restrict__ VOUT, double4* __restrict__ GRAD) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.n) return;
    const int64_t u = a.nodes ? (int64_t)a.nodes[k] : k;
    // the fp32 term of bond b at u is bitwise the negation of its reverse's
    // term at the bond's source (same operands, exchanged); fp64 sums
    double gx = 0.0, gy = 0.0, gz = 0.0;
    for (int b = a.brow[u]; b < a.brow[u + 1]; ++b) {
        const int rb = a.brev[b];
        const float4 i1 = VIN[rb], o1 = VOUT[b], i2 = VIN[b], o2 = VOUT[rb];
        gx += (double)((i1.x + o1.x) - (i2.x + o2.x));
        gy += (double)((i1.y + o1.y) - (i2.y + o2.y));
        gz += (double)((i1.z + o1.z) - (i2.z + o2.z));
    }
    grad_add(GRAD, k, gx, gy, gz);
}

// h_bar = readout for every node (potential.cpp:808); a row per thread so the
// constant reads are warp-uniform (broadcast) instead of 16-way divergent
__global__ void k_init_hbar(int64_t n, float* HB) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    float4* row = reinterpret_cast<float4*>(HB + k * kF);
#pragma unroll
    for (int q = 0; q < kF / 4; ++q)
        row[q] = make_float4(c_m.ro[4 * q], c_m.ro[4 * q + 1], c_m.ro[4 * q + 2], c_m.ro[4 * q + 3]);
}

__global__ void k_forces_out(int64_t n, const int32_t* __restrict__ nodes,
                             const double4* __restrict__ GRAD, double* forces, float* forces32) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t v = nodes ? (int64_t)nodes[k] : k;
    const double4 g = GRAD[k];
    if (forces) {
        forces[3 * v] = -g.x;
        forces[3 * v + 1] = -g.y;
        forces[3 * v + 2] = -g.z;
    }
    if (forces32) {
        forces32[3 * v] = -(float)g.x;
        forces32[3 * v + 1] = -(float)g.y;
        forces32[3 * v + 2] = -(float)g.z;
    }
}

// fixed-shape reduction of nparts x w partials: block c sums column c with
// strided per-thread sums and a fixed tree over 512 threads (deterministic
// for a given nparts)
__global__ void __launch_bounds__(512) k_reduce_partials(const double* parts, int nparts, int w,
                                                         double* out) {
    __shared__ double sh[512];
    const int t = threadIdx.x, c = blockIdx.x;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int i = t;
    for (; i + 3 * 512 < nparts; i += 4 * 512)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += parts[(size_t)(i + u * 512) * w + c];
    for (; i < nparts; i += 512) acc[0] += parts[(size_t)i * w + c];
    sh[t] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    __syncthreads();
    for (int o = 256; o > 0; o >>= 1) {
        if (t < o) sh[t] += sh[t + o];
        __syncthreads();
    }
    if (t == 0) out[c] = sh[0];
}

}  // namespace

// One wave of the 3-CTA/SM model kernels: all resident CTAs sweep the node
// range together, so the gathered neighbour rows of the active window stay in
// L2 (C5: 1776 CTAs 7.50 ms/step, 888 7.38, 444 7.26, 296 8.35).
int model_grid(int64_t n) {
    static const int cap = [] {
        const char* v = std::getenv("GMD_MODEL_GRID");
        return v ? std::atoi(v) : 148 * 4;
    }();
    int64_t g = (n + kNodesPerCta - 1) / kNodesPerCta;
    if (g > cap) g = cap;
    return (int)(g > 0 ? g : 1);
}

// forward: many small CTAs (C4 tb_forward 0.109 ms at 148 x 32 vs 0.151 at
// 148 x 4); backward: one wave of 4 CTAs per SM, so the final virial barrier
// waits less on uneven centers (0.338 vs 0.353 ms)
static int tb_grid(int64_t n, int cap = 148 * 32) {
    int64_t g = (n + kTbGroups - 1) / kTbGroups;
    if (g > cap) g = cap;
    return (int)(g > 0 ? g : 1);
}
static int tb_bwd_grid(int64_t n) { return tb_grid(n, 148 * 4); }

void launch_embed(int64_t rows, const int32_t* node_array, const int32_t* Z, float* H0,
                  cudaStream_t s, uint8_t* zs, unsigned* zmask) {
    if (rows == 0) return;
    if (zs) GMD_CUDA(cudaMemsetAsync(zmask, 0, 4 * sizeof(unsigned), s));
    k_embed<<<div_up(rows * 4, 256), 256, 0, s>>>(rows, node_array, Z, H0, zs, zmask);
    GMD_LAUNCH_CHECK();
}

void launch_exchange(int64_t nx, const int32_t* xdst, const int32_t* xsrc, float* buf, int width,
                     cudaStream_t s) {
    if (nx == 0) return;
    int w4 = width / 4;
    k_exchange<<<div_up(nx * w4, 256), 256, 0, s>>>(nx, xdst, xsrc, reinterpret_cast<float4*>(buf),
                                                     w4);
    GMD_LAUNCH_CHECK();
}

void launch_conv(const ConvArgs& a, int layer, const float* Hin, float* Hout, float* TH,
                 double* per_atom, double* e_part, cudaStream_t s, const uint8_t* zs,
                 const unsigned* zmask) {
    if (a.n == 0) return;
    if (zs) {  // layer 0 from the embeddings: species-sum form (<= 2 species)
        k_conv2<4, kThreads, true><<<model_grid(a.n), kThreads, 0, s>>>(a, layer, Hin, Hout, TH, per_atom,
                                                                      e_part, zs, zmask);
        GMD_LAUNCH_CHECK();
        return;
    }
    const char* venv = std::getenv("GMD_CONV_VARIANT");  // read per call (tests switch kernels)
    const int variant = venv ? std::atoi(venv) : 0;
    const int g = model_grid(a.n);
    if (variant == 1)  // scalar-FFMA kernel (A/B reference)
        k_conv<<<g, kThreads, 0, s>>>(a, layer, Hin, Hout, TH, per_atom, e_part);
    else  // 4 CTAs x 256 threads per SM (64 registers), one wave of 148 x 4:
          // C5 conv 1.58 -> 1.50 ms per step vs 3 CTAs at 80 registers
        k_conv2<4><<<g, kThreads, 0, s>>>(a, layer, Hin, Hout, TH, per_atom, e_part);
    GMD_LAUNCH_CHECK();
}

void launch_bwd_node(int64_t n, const int32_t* nodes, const int32_t* crow, int layer,
                     float* HB, const float* TH, float* MB, bool init, cudaStream_t s) {
    if (n == 0) return;
    k_bwd_node<<<div_up(n, 128), 128, 0, s>>>(n, nodes, crow, layer, HB, TH, MB, init);
    GMD_LAUNCH_CHECK();
}

static int bwd_variant() {
    const char* venv = std::getenv("GMD_BWD_VARIANT");  // read per call (tests switch kernels)
    return venv ? std::atoi(venv) : 0;
}

// The default backward runs 640-thread CTAs, one per SM: the 40 consecutive
// nodes a CTA works on share most neighbour rows, which then hit in the SM's
// L1 (C5: 3.13 -> 2.98 ms per step vs 3 x 256-thread CTAs per SM; the
// forward conv is faster with 256-thread CTAs).
constexpr int kBwdThreads = 768;       // fp32 gradient lanes (80 registers)
constexpr int kBwdThreads2 = 640;      // the same at 96 registers (A/B: GMD_BWD_THREADS=640)
constexpr int kBwdThreadsExact = 640;  // fp64 gradient lanes (96 registers)

// exact mode (GMD_EXACT_FORCES=1): Newton's third law to the last bit (fp64
// per-lane gradient sums of bitwise-opposite edge terms); the default sums the
// per-lane terms in fp32 (forces sum to zero to ~1e-7 relative)
static bool exact_forces() {
    const char* v = std::getenv("GMD_EXACT_FORCES");  // read per call (tests switch)
    return v && v[0] == '1';
}

static int bwd_threads() {
    if (exact_forces()) return kBwdThreadsExact;
    const char* v = std::getenv("GMD_BWD_THREADS");
    return v && std::atoi(v) == kBwdThreads2 ? kBwdThreads2 : kBwdThreads;
}

int bwd_edge_grid(int64_t n) {
    if (bwd_variant() == 1) return model_grid(n);
    const int64_t per = bwd_threads() / 16;
    int64_t g = (n + per - 1) / per;
    if (g > 148) g = 148;
    return (int)(g > 0 ? g : 1);
}

bool bwd_edge_ranges() { return bwd_variant() != 1; }

int64_t bwd_edge_stride(int grid) { return (int64_t)grid * (bwd_threads() / 16); }

// dynamic shared memory of the fp32 backward (the epilogue's transpose
// groups), opted in once per instantiation
template <int NT, bool HBAR, bool SPEC = false>
static size_t bwd_smem() {
    constexpr size_t bytes = sizeof(float) * (NT / 16) * GroupT<kBwdTS>::kGroup;
    static bool done[64] = {};
    int dev = 0;
    GMD_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !done[dev]) {
        GMD_CUDA(cudaFuncSetAttribute(k_bwd_edge2<1, NT, float, HBAR, SPEC>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        if (dev >= 0 && dev < 64) done[dev] = true;
    }
    return bytes;
}

void launch_bwd_edge(const ConvArgs& a, const float* MB, const float* Hl, float* HB, double4* GRAD,
                     double* vir_part, cudaStream_t s, double* vir_grp, int grid, bool hbar,
                     const uint8_t* zs, const unsigned* zmask) {
    if (a.n - a.k0 <= 0) return;
    const int variant = bwd_variant();
    if (variant == 1 && a.k0 != 0) raise(kRuntime, "internal: node ranges need the default kernel");
    const int g = grid > 0 ? grid : bwd_edge_grid(a.n - a.k0);
    if (variant == 1)  // scalar-FFMA kernel (A/B reference; always forms h_bar)
        k_bwd_edge<<<g, kThreads, 0, s>>>(a, MB, Hl, HB, GRAD, vir_part);
    else if (exact_forces()) {
        if (hbar)
            k_bwd_edge2<1, kBwdThreadsExact, double, true><<<g, kBwdThreadsExact, 0, s>>>(a, MB, Hl, HB, GRAD,
                                                                                      vir_part, vir_grp);
        else if (zs)
            k_bwd_edge2<1, kBwdThreadsExact, double, false, true><<<g, kBwdThreadsExact, 0, s>>>(
                a, MB, Hl, HB, GRAD, vir_part, vir_grp, zs, zmask);
        else
            k_bwd_edge2<1, kBwdThreadsExact, double, false><<<g, kBwdThreadsExact, 0, s>>>(a, MB, Hl, HB, GRAD,
                                                                                       vir_part, vir_grp);
    } else if (bwd_threads() == kBwdThreads2) {
        if (hbar)
            k_bwd_edge2<1, kBwdThreads2, float, true><<<g, kBwdThreads2, bwd_smem<kBwdThreads2, true>(), s>>>(
                a, MB, Hl, HB, GRAD, vir_part, vir_grp);
        else
            k_bwd_edge2<1, kBwdThreads2, float, false><<<g, kBwdThreads2, bwd_smem<kBwdThreads2, false>(), s>>>(
                a, MB, Hl, HB, GRAD, vir_part, vir_grp);
    } else {
        if (hbar)
            k_bwd_edge2<1, kBwdThreads, float, true><<<g, kBwdThreads, bwd_smem<kBwdThreads, true>(), s>>>(
                a, MB, Hl, HB, GRAD, vir_part, vir_grp);
        else if (zs)
            k_bwd_edge2<1, kBwdThreads, float, false, true>
                <<<g, kBwdThreads, bwd_smem<kBwdThreads, false, true>(), s>>>(a, MB, Hl, HB, GRAD, vir_part,
                                                                           vir_grp, zs, zmask);
        else
            k_bwd_edge2<1, kBwdThreads, float, false><<<g, kBwdThreads, bwd_smem<kBwdThreads, false>(), s>>>(
                a, MB, Hl, HB, GRAD, vir_part, vir_grp);
    }
    GMD_LAUNCH_CHECK();
}

int bwd_tc_grid(int64_t n) {
    int64_t g = 148 * kBwdTcCtas;  // one wave
    if (g > (n + 15) / 16) g = (n + 15) / 16;
    return (int)(g > 0 ? g : 1);
}

void launch_chunk_count(const ConvArgs& a, int32_t* cnt, cudaStream_t s) {
    k_chunk_count<<<div_up(a.n + 1, 256), 256, 0, s>>>(a, cnt);
    GMD_LAUNCH_CHECK();
}

void launch_chunk_fill(const ConvArgs& a, const int32_t* cstart, int4* tab, int grid,
                       int32_t* cta, cudaStream_t s) {
    if (a.n > 0) {
        k_chunk_fill<<<div_up(a.n, 256), 256, 0, s>>>(a, cstart, tab);
        GMD_LAUNCH_CHECK();
    }
    k_chunk_cta<<<div_up(grid + 1, 256), 256, 0, s>>>(a.n, cstart, grid, cta);
    GMD_LAUNCH_CHECK();
}

void launch_bwd_edge_tc(const ConvArgs& a, const int4* ctab, const int32_t* ccta, int grid,
                        const float* MB, const float* Hl, float* HB, double4* GRAD,
                        double* vir_part, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        GMD_CUDA(cudaFuncSetAttribute(k_bwd_edge_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(BwdTcSmem)));
        attr = true;
    }
    k_bwd_edge_tc<<<grid, kTM, sizeof(BwdTcSmem), s>>>(a, ctab, ccta, MB, Hl, HB, GRAD, vir_part);
    GMD_LAUNCH_CHECK();
}

static int tb_slots(int max_bonds) {
    return std::min(kMaxBondsPerAtom, std::max(16, (max_bonds + 15) & ~15));
}

void launch_tb_forward(const BondArgs& a, float* TP, float* TH3, int32_t* flags, int max_bonds,
                       cudaStream_t s) {
    if (a.n == 0) return;
    const int kc = tb_slots(max_bonds);
    const size_t smem = (sizeof(float) * kF + sizeof(float4)) * kTbGroups * kc;
    static bool attr = false;
    if (!attr) {
        GMD_CUDA(cudaFuncSetAttribute(k_tb_forward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)((sizeof(float) * kF + sizeof(float4)) * kTbGroups *
                                            kMaxBondsPerAtom)));
        attr = true;
    }
    k_tb_forward<<<tb_grid(a.n), kTbWarps * 32, smem, s>>>(a, TP, TH3, flags, kc);
    GMD_LAUNCH_CHECK();
}

void launch_tb_inject(const BondArgs& a, const float* TP, float* H, float* TH4, cudaStream_t s) {
    if (a.n == 0) return;
    k_tb_inject<<<div_up(a.n, 128), 128, 0, s>>>(a, TP, H, TH4);
    GMD_LAUNCH_CHECK();
}

void launch_tb_bwd_q(int64_t n, const int32_t* nodes, const int32_t* crow, const float* HB,
                     const float* TH4, float* QB, cudaStream_t s) {
    if (n == 0) return;
    k_tb_bwd_q<<<div_up(n, 128), 128, 0, s>>>(n, nodes, crow, HB, TH4, QB);
    GMD_LAUNCH_CHECK();
}

void launch_tb_backward(const BondArgs& a, const float* QB, const float* TH3, float4* VIN,
                        float4* VOUT, double* vir_part, int max_bonds, cudaStream_t s) {
    if (a.n == 0) return;
    const int kc = tb_slots(max_bonds);
    const size_t smem = kTbSlotBytes * kTbGroups * kc;
    static bool attr = false;
    if (!attr) {
        GMD_CUDA(cudaFuncSetAttribute(k_tb_backward<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(kTbSlotBytes * kTbGroups * kMaxBondsPerAtom)));
        attr = true;
    }
    // 4 CTAs x 128 threads per SM (128 registers, no spills): C4 0.353 ms vs
    // 0.380 / 0.409 ms for 5 / 6 CTAs (96 / 80 registers with spills)
    k_tb_backward<4><<<tb_bwd_grid(a.n), kTbWarps * 32, smem, s>>>(a, QB, TH3, VIN, VOUT, vir_part, kc);
    GMD_LAUNCH_CHECK();
}

void launch_tb_grad(const BondArgs& a, const float4* VIN, const float4* VOUT, double4* GRAD,
                    cudaStream_t s) {
    if (a.n == 0) return;
    k_tb_grad<<<div_up(a.n, 128), 128, 0, s>>>(a, VIN, VOUT, GRAD);
    GMD_LAUNCH_CHECK();
}

void launch_init_hbar(int64_t n, float* HB, cudaStream_t s) {
    if (n == 0) return;
    k_init_hbar<<<div_up(n, 256), 256, 0, s>>>(n, HB);
    GMD_LAUNCH_CHECK();
}

void launch_forces_out(int64_t n, const int32_t* nodes, const double4* GRAD, double* forces,
                       float* forces32, cudaStream_t s) {
    if (n == 0) return;
    k_forces_out<<<div_up(n, 256), 256, 0, s>>>(n, nodes, GRAD, forces, forces32);
    GMD_LAUNCH_CHECK();
}

// up to three partial sets in one launch: block c reduces output column c of
// the set it falls in (same per-column arithmetic as k_reduce_partials)
struct ReduceSets {
    const double* parts[3];
    int nparts[3], w[3], col0[3];
    int nsets;
};
__global__ void __launch_bounds__(512) k_reduce_sets(ReduceSets R, double* out) {
    int set = 0;
    while (set + 1 < R.nsets && (int)blockIdx.x >= R.col0[set + 1]) ++set;
    const int c = blockIdx.x - R.col0[set], w = R.w[set], np = R.nparts[set];
    const double* parts = R.parts[set];
    __shared__ double sh[512];
    const int t = threadIdx.x;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int i = t;
    for (; i + 3 * 512 < np; i += 4 * 512)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += parts[(size_t)(i + u * 512) * w + c];
    for (; i < np; i += 512) acc[0] += parts[(size_t)i * w + c];
    sh[t] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    __syncthreads();
    for (int o = 256; o > 0; o >>= 1) {
        if (t < o) sh[t] += sh[t + o];
        __syncthreads();
    }
    if (t == 0) out[blockIdx.x] = sh[0];
}

void launch_reduce_sets(int nsets, const double* const* parts, const int* nparts, const int* w,
                        double* out, cudaStream_t s) {
    ReduceSets R{};
    int cols = 0;
    R.nsets = nsets;
    for (int k = 0; k < nsets; ++k) {
        R.parts[k] = parts[k];
        R.nparts[k] = nparts[k];
        R.w[k] = w[k];
        R.col0[k] = cols;
        cols += w[k];
    }
    k_reduce_sets<<<cols, 512, 0, s>>>(R, out);
    GMD_LAUNCH_CHECK();
}

void launch_reduce_partials(const double* parts, int nparts, int w, double* out, cudaStream_t s) {
    k_reduce_partials<<<w, 512, 0, s>>>(parts, nparts, w, out);
    GMD_LAUNCH_CHECK();
}

int tb_grid_size(int64_t n) { return tb_bwd_grid(n); }

}  // namespace gmd
