// F = 64, K = 8 model kernels (see gmd_wide.cuh).  Formulas as
// gmd_generic.cu / proj/src/potential.cpp:19-78 (radial basis), 743-774
// (conv), 816-848 (backward):
//   u_k(d) = fc(d) exp(-((d - mu_k)/sigma)^2),  s_f = sum_k P_fk u_k
//   m_u    = sum_{e=(w->u)} s_e (.) h_w,  h_u' = h_u + tanh(W m_u + b)
//   backward ("dsum" form, gmd_model.cu): per in-edge e = (w -> u)
//     hbar_u += mbar_w (.) s_e
//     dsum_e  = sum_k psi_k G_k,  G = X P,  X_f = mbar_u,f h_w,f + h_u,f mbar_w,f,
//               psi_k = phi_k (ca + cb k)
//     grad_u -= v_e dsum_e / d_e,  virial += 1/2 dsum_e / d_e v_e (x) v_e
#include <cstdlib>
#include <string>

#include "gmd_tc.cuh"
#include "gmd_wide.cuh"

namespace gmd {
namespace {

constexpr int F = kWideF, K = kWideK;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 bc2(float x) { return make_float2(x, x); }

__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct Basis {  // per-call scalars of the atom-channel radial basis
    float a2;   // sqrt(log2 e) / sigma
    float mu2;  // mu_step * a2
    float rc, pi_rc, isg, mus;
};

__host__ Basis make_basis(const GenModel& g) {
    Basis b;
    b.a2 = 1.2011224087864498f * g.inv_sigma;  // sqrt(log2(e)) / sigma
    b.mu2 = g.mu_step * b.a2;
    b.rc = g.rc;
    b.pi_rc = 3.14159265358979f * g.inv_rc;
    b.isg = g.inv_sigma;
    b.mus = g.mu_step;
    return b;
}

// phi_k = exp(-((d - mu_k)/sigma)^2) = 2^(-(d a2 - k mu2)^2)
__device__ __forceinline__ void phi8(const Basis& b, float d, float phi[K]) {
    const float xa = d * b.a2;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const float x = xa - (float)k * b.mu2;
        phi[k] = ex2a(-x * x);
    }
}

__device__ __forceinline__ float gwarp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}
__device__ __forceinline__ double gwarp_sumd(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// ---------------------------------------------------------------------------
// forward conv: one warp per node, lane l holds features 2l, 2l+1
// ---------------------------------------------------------------------------
constexpr int kConvWarps = 8;

struct ConvSmem {
    float2 WT[F][F / 2];           // WT[q][l] = (W[2l][q], W[2l+1][q])
    float4 u[kConvWarps][32][2];   // fc * phi_0..7 of the chunk's edges
    int src[kConvWarps][32];
    float4 m[kConvWarps][F / 4];   // the node's m row (broadcast reads)
};

// SPEC (layer 0, h0 = emb[Z], at most two species): m = sum_s emb[z_s] (.)
// (P Phi_s), Phi_s = the per-species sum of the in-edges' fc phi -- the
// feature lanes do no per-edge work (F = 16's species-sum form, gmd_model.cu)
template <bool SPEC = false>
__global__ void __launch_bounds__(kConvWarps * 32) k_wide_conv(GenModel g, Basis bs, ConvArgs a,
                                                               int layer, const float* __restrict__ Hin,
                                                               float* __restrict__ Hout,
                                                               float* __restrict__ TH,
                                                               double* __restrict__ per_atom,
                                                               const uint8_t* __restrict__ zs = nullptr,
                                                               const unsigned* __restrict__ zmask = nullptr) {
    __shared__ __align__(16) ConvSmem S;
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    int z1 = -1;
    bool spec = false;
    float2 e0s = make_float2(0.f, 0.f), e1s = make_float2(0.f, 0.f);  // emb[z_s] feature pair
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
        if (spec) {
            e0s = make_float2(g.emb[z0 * F + 2 * lane], g.emb[z0 * F + 2 * lane + 1]);
            e1s = make_float2(g.emb[z1 * F + 2 * lane], g.emb[z1 * F + 2 * lane + 1]);
        }
    }
    const float* W = g.W + (size_t)layer * F * F;  // W[f][q]
    for (int t = threadIdx.x; t < F * F / 2; t += blockDim.x) {
        const int q = t / (F / 2), l = t % (F / 2);
        S.WT[q][l] = make_float2(W[(2 * l) * F + q], W[(2 * l + 1) * F + q]);
    }
    float2 P2[K];  // (P[2l][k], P[2l+1][k])
#pragma unroll
    for (int k = 0; k < K; ++k) P2[k] = make_float2(g.P[(2 * lane) * K + k], g.P[(2 * lane + 1) * K + k]);
    const float2 b2 = make_float2(g.b[layer * F + 2 * lane], g.b[layer * F + 2 * lane + 1]);
    const float2 ro2 = make_float2(g.ro[2 * lane], g.ro[2 * lane + 1]);
    __syncthreads();
    for (int64_t k = (int64_t)blockIdx.x * kConvWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kConvWarps) {
        const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t r = a.crow ? (int64_t)a.crow[v] : v;
        const int e0 = a.row[v], e1 = a.row[v + 1];
        float2 m = make_float2(0.f, 0.f);
        if (SPEC && spec) {
            // lane j: Phi column (s, k) = (j >> 3 & 1, j & 7) over the chunk's
            // even (j < 16) or odd (j >= 16) edges, halves combined at the end
            const int col = lane & 15, half = lane >> 4;
            const int want = col >> 3, kk = col & 7;
            float ph = 0.f;
            for (int eb = e0; eb < e1; eb += 32) {
                const int ne = min(32, e1 - eb);
                if (lane < ne) {
                    const float d = a.d[eb + lane];
                    float phi[K];
                    phi8(bs, d, phi);
                    const float fc = d < bs.rc ? 0.5f * __cosf(d * bs.pi_rc) + 0.5f : 0.0f;
                    S.u[wq][lane][0] = make_float4(fc * phi[0], fc * phi[1], fc * phi[2], fc * phi[3]);
                    S.u[wq][lane][1] = make_float4(fc * phi[4], fc * phi[5], fc * phi[6], fc * phi[7]);
                    S.src[wq][lane] = zs[a.lsrc[eb + lane]] == z1 ? 1 : 0;
                }
                __syncwarp();
                for (int i = half; i < ne; i += 2) {
                    const float u = reinterpret_cast<const float*>(S.u[wq][i])[kk];
                    ph += S.src[wq][i] == want ? u : 0.f;
                }
                __syncwarp();
            }
            ph += __shfl_xor_sync(0xffffffffu, ph, 16);
            float* phs = reinterpret_cast<float*>(S.m[wq]);
            if (lane < 16) phs[lane] = ph;
            __syncwarp();
            float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
            for (int k2 = 0; k2 < K; ++k2) {
                s0 = f2fma(P2[k2], bc2(phs[k2]), s0);
                s1 = f2fma(P2[k2], bc2(phs[K + k2]), s1);
            }
            m = f2fma(e0s, s0, f2mul(e1s, s1));
            __syncwarp();
        }
        for (int eb = e0; !(SPEC && spec) && eb < e1; eb += 32) {
            const int ne = min(32, e1 - eb);
            if (lane < ne) {
                const float d = a.d[eb + lane];
                float phi[K];
                phi8(bs, d, phi);
                const float fc = d < bs.rc ? 0.5f * __cosf(d * bs.pi_rc) + 0.5f : 0.0f;
                S.u[wq][lane][0] = make_float4(fc * phi[0], fc * phi[1], fc * phi[2], fc * phi[3]);
                S.u[wq][lane][1] = make_float4(fc * phi[4], fc * phi[5], fc * phi[6], fc * phi[7]);
                S.src[wq][lane] = a.lsrc[eb + lane];
            }
            __syncwarp();
            int i = 0;
            for (; i + 4 <= ne; i += 4) {  // four gathered rows in flight
                float2 h[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    h[j] = __ldg(reinterpret_cast<const float2*>(Hin + (size_t)S.src[wq][i + j] * F) + lane);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 ua = S.u[wq][i + j][0], ub = S.u[wq][i + j][1];
                    float2 sv = f2mul(P2[0], bc2(ua.x));
                    sv = f2fma(P2[1], bc2(ua.y), sv);
                    sv = f2fma(P2[2], bc2(ua.z), sv);
                    sv = f2fma(P2[3], bc2(ua.w), sv);
                    sv = f2fma(P2[4], bc2(ub.x), sv);
                    sv = f2fma(P2[5], bc2(ub.y), sv);
                    sv = f2fma(P2[6], bc2(ub.z), sv);
                    sv = f2fma(P2[7], bc2(ub.w), sv);
                    m = f2fma(h[j], sv, m);
                }
            }
            for (; i < ne; ++i) {
                const float2 h = __ldg(reinterpret_cast<const float2*>(Hin + (size_t)S.src[wq][i] * F) + lane);
                const float4 ua = S.u[wq][i][0], ub = S.u[wq][i][1];
                float2 sv = f2mul(P2[0], bc2(ua.x));
                sv = f2fma(P2[1], bc2(ua.y), sv);
                sv = f2fma(P2[2], bc2(ua.z), sv);
                sv = f2fma(P2[3], bc2(ua.w), sv);
                sv = f2fma(P2[4], bc2(ub.x), sv);
                sv = f2fma(P2[5], bc2(ub.y), sv);
                sv = f2fma(P2[6], bc2(ub.z), sv);
                sv = f2fma(P2[7], bc2(ub.w), sv);
                m = f2fma(h, sv, m);
            }
            __syncwarp();
        }
        // z = W m + b: m broadcast from shared memory, W column pair per lane
        reinterpret_cast<float2*>(S.m[wq])[lane] = m;
        __syncwarp();
        float2 z = b2;
#pragma unroll 4
        for (int q4 = 0; q4 < F / 4; ++q4) {
            const float4 mm = S.m[wq][q4];
            z = f2fma(S.WT[4 * q4][lane], bc2(mm.x), z);
            z = f2fma(S.WT[4 * q4 + 1][lane], bc2(mm.y), z);
            z = f2fma(S.WT[4 * q4 + 2][lane], bc2(mm.z), z);
            z = f2fma(S.WT[4 * q4 + 3][lane], bc2(mm.w), z);
        }
        __syncwarp();
        const float2 th = make_float2(tanhf(z.x), tanhf(z.y));
        const float2 hin = reinterpret_cast<const float2*>(Hin + (size_t)r * F)[lane];
        const float2 hn = make_float2(hin.x + th.x, hin.y + th.y);
        reinterpret_cast<float2*>(Hout + (size_t)r * F)[lane] = hn;
        note_nonfinite(a, layer, r, hn.x);
        note_nonfinite(a, layer, r, hn.y);
        reinterpret_cast<float2*>(TH + (size_t)k * F)[lane] = th;
        if (per_atom) {
            const float ev = gwarp_sum(fmaf(ro2.x, hn.x, ro2.y * hn.y));
            if (lane == 0) per_atom[v] = (double)ev;
        }
    }
}

// ---------------------------------------------------------------------------
// backward node pass: MB[row] = W^T (HB (.) (1 - th^2)), lane = feature pair
// ---------------------------------------------------------------------------
// (also the three-body q_bar = W4^T (HB (.) (1 - TH4^2)) with W = W4)
__global__ void __launch_bounds__(kConvWarps * 32) k_wide_bwd_node(GenModel g, int64_t n,
                                                                   const int32_t* __restrict__ nodes,
                                                                   const int32_t* __restrict__ crow,
                                                                   const float* __restrict__ W,
                                                                   float* __restrict__ HB,
                                                                   const float* __restrict__ TH,
                                                                   float* __restrict__ MB, int init) {
    __shared__ __align__(16) float2 sW[F][F / 2];  // sW[f][l] = (W[f][2l], W[f][2l+1])
    __shared__ __align__(16) float4 sy[kConvWarps][F / 4];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < F * F / 2; t += blockDim.x)
        sW[t / (F / 2)][t % (F / 2)] = reinterpret_cast<const float2*>(W)[t];
    const float2 ro2 = make_float2(g.ro[2 * lane], g.ro[2 * lane + 1]);
    __syncthreads();
    for (int64_t k = (int64_t)blockIdx.x * kConvWarps + wq; k < n; k += (int64_t)gridDim.x * kConvWarps) {
        const int64_t v = nodes ? (int64_t)nodes[k] : k;
        const int64_t r = crow ? (int64_t)crow[v] : v;
        float2 hb;
        if (init) {  // h_bar starts as the readout (potential.cpp:800-806)
            hb = ro2;
            reinterpret_cast<float2*>(HB + (size_t)k * F)[lane] = hb;
        } else {
            hb = reinterpret_cast<const float2*>(HB + (size_t)k * F)[lane];
        }
        const float2 th = reinterpret_cast<const float2*>(TH + (size_t)k * F)[lane];
        const float2 y = make_float2(hb.x * (1.0f - th.x * th.x), hb.y * (1.0f - th.y * th.y));
        reinterpret_cast<float2*>(sy[wq])[lane] = y;
        __syncwarp();
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int f4 = 0; f4 < F / 4; ++f4) {
            const float4 yy = sy[wq][f4];
            acc = f2fma(sW[4 * f4][lane], bc2(yy.x), acc);
            acc = f2fma(sW[4 * f4 + 1][lane], bc2(yy.y), acc);
            acc = f2fma(sW[4 * f4 + 2][lane], bc2(yy.z), acc);
            acc = f2fma(sW[4 * f4 + 3][lane], bc2(yy.w), acc);
        }
        __syncwarp();
        reinterpret_cast<float2*>(MB + (size_t)r * F)[lane] = acc;
    }
}

// ---------------------------------------------------------------------------
// backward edge pass with the K = 64 contraction on tcgen05
// ---------------------------------------------------------------------------
constexpr int kBW = 8;            // warps per CTA: 8 x 16 edge slots = MMA M = 128
constexpr int kSlots = 16;        // edge slots per warp and step (warps w and w + 4 share a TMEM lane quarter)

constexpr int kXLbo = 144;        // bytes between K-adjacent core matrices (16 B pad: conflict-free stores)
constexpr int kXSbo = 16 * kXLbo; // bytes between 8-row groups (64 K = 16 core matrices)
constexpr int kXBytes = 16 * kXSbo;  // 128 rows
constexpr int kPLbo = 128, kPSbo = 16 * kPLbo;
constexpr int kPBytes = 2 * kPSbo;   // N = 16 rows (P^T in rows 0..7, zeros in 8..15)
constexpr int kNcols = 16;           // MMA N (TMEM columns used)

struct BwdSmem {
    unsigned char x_hi[kXBytes];
    unsigned char x_lo[kXBytes];
    unsigned char p_hi[kPBytes];
    unsigned char p_lo[kPBytes];
    // per-step edge records, double-buffered: step u + 1's are loaded while
    // the tensor cores run step u
    float4 u[2][kBW][kSlots][2];    // fc * phi of the chunk's edges
    float4 psi[2][kBW][kSlots][2];  // psi_k of the chunk's edges (epilogue)
    float4 q[2][kBW][kSlots];       // (v, d) of the chunk's edges (epilogue)
    int src[2][kBW][kSlots];
    uint64_t mbar;
    uint32_t tbase;
};

__device__ __forceinline__ int xoff(int r, int k) {  // byte offset of (row r, K index k)
    return (r >> 3) * kXSbo + (k >> 2) * kXLbo + (r & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ int poff(int r, int k) {
    return (r >> 3) * kPSbo + (k >> 2) * kPLbo + (r & 7) * 16 + (k & 3) * 4;
}

// shared-memory descriptor, K-major, no swizzle, explicit offsets
__device__ __forceinline__ uint64_t sdesc2(const void* base, uint32_t lbo, uint32_t sbo) {
    const uint64_t addr = tc::smem_u32(base);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float v[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void split2(float2 x, float2& hi, float2& lo) {
    tc::split_tf32(x.x, hi.x, lo.x);
    tc::split_tf32(x.y, hi.y, lo.y);
}

template <int kBatch>  // gathered edges in flight per warp
__global__ void __launch_bounds__(kBW * 32, 2) k_wide_bwd_edge(GenModel g, Basis bs, ConvArgs a,
                                                              const float* __restrict__ MB,
                                                              const float* __restrict__ Hl,
                                                              float* __restrict__ HB,
                                                              double4* __restrict__ GRAD,
                                                              double* __restrict__ vir_part) {
    extern __shared__ __align__(1024) unsigned char wsm[];
    BwdSmem& S = *reinterpret_cast<BwdSmem*>(wsm);
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    // B operand: B[n][f] = P[f][n] (n < 8), 0 (n >= 8); tf32 hi / lo
    for (int t = tid; t < kNcols * F; t += blockDim.x) {
        const int nn = t / F, f = t % F;
        const float x = nn < K ? g.P[f * K + nn] : 0.0f;
        float hv, lv;
        tc::split_tf32(x, hv, lv);
        *reinterpret_cast<float*>(S.p_hi + poff(nn, f)) = hv;
        *reinterpret_cast<float*>(S.p_lo + poff(nn, f)) = lv;
    }
    if (tid == 0) {
        tc::mbar_init(&S.mbar, 1);
        tc::fence_mbar_init();
    }
    if (wq == 0) tc::tmem_alloc(&S.tbase, 32);
    float2 P2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) P2[k] = make_float2(g.P[(2 * lane) * K + k], g.P[(2 * lane + 1) * K + k]);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = S.tbase;
    const uint32_t idesc = tc::idesc_tf32(128, kNcols);
    // rows of warp w: lane quarter w % 4, slots 16 (w / 4) .. 16 (w / 4) + 15
    const int row0 = 32 * (wq & 3) + kSlots * (wq >> 2);
    const uint32_t trow = tmem + ((uint32_t)(32 * (wq & 3)) << 16);

    // this warp's node sequence; all warps step together (one MMA per step)
    const int64_t gw = (int64_t)blockIdx.x * kBW + wq, nw = (int64_t)gridDim.x * kBW;
    const int64_t my_nodes = gw < a.n ? (a.n - 1 - gw) / nw + 1 : 0;
    // steps of this CTA = max over its warps of sum of ceil(deg / 32): the
    // first warp of the CTA has the most nodes; count chunks per warp and
    // agree on the maximum through shared memory
    __shared__ int steps_w[kBW];
    int my_steps = 0;
    for (int64_t j = lane; j < my_nodes; j += 32) {
        const int64_t kk = gw + j * nw;
        const int64_t vv = a.nodes ? (int64_t)a.nodes[kk] : kk;
        const int deg = a.row[vv + 1] - a.row[vv];
        my_steps += deg > 0 ? (deg + kSlots - 1) / kSlots : 1;  // empty rows still finalize
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_steps += __shfl_xor_sync(kFull, my_steps, o);
    if (lane == 0) steps_w[wq] = my_steps;
    __syncthreads();
    int steps = 0;
    for (int w = 0; w < kBW; ++w) steps = max(steps, steps_w[w]);

    double vir[6] = {0, 0, 0, 0, 0, 0};
    // schedule: steps of <= 16 edges of one node, in this warp's node order
    struct Step {
        int64_t k, r;
        int pos, ne;
        bool first, last;
    };
    int64_t jn = 0, sk = -1, sr = 0;
    int spos = 0, se1 = 0;
    auto schedule = [&]() {
        Step st{-1, 0, 0, 0, false, false};
        if (spos >= se1) {
            if (jn >= my_nodes) return st;
            sk = gw + jn * nw;
            ++jn;
            const int64_t sv = a.nodes ? (int64_t)a.nodes[sk] : sk;
            sr = a.crow ? (int64_t)a.crow[sv] : sv;
            spos = a.row[sv];
            se1 = a.row[sv + 1];
            st.first = true;
        }
        st.k = sk;
        st.r = sr;
        st.pos = spos;
        st.ne = min(kSlots, se1 - spos);
        spos += st.ne;
        st.last = spos >= se1;
        return st;
    };
    // per-edge scalars of a step into buffer b, lane = edge slot
    auto load_step = [&](int b, const Step& st) {
        if (lane < st.ne) {
            const float4 q = __ldg(a.vd + st.pos + lane);
            const float d = q.w;
            float phi[K];
            phi8(bs, d, phi);
            float sn, cs;
            __sincosf(d * bs.pi_rc, &sn, &cs);
            const bool in = d < bs.rc;
            const float fc = in ? 0.5f * cs + 0.5f : 0.0f;
            const float dfc = in ? -0.5f * bs.pi_rc * sn : 0.0f;
            const float x0 = d * bs.isg, stp = bs.mus * bs.isg;
            const float ca = dfc - 2.0f * fc * bs.isg * x0, cb = 2.0f * fc * bs.isg * stp;
            float psi[K];
#pragma unroll
            for (int kk = 0; kk < K; ++kk) psi[kk] = phi[kk] * fmaf(cb, (float)kk, ca);
            S.psi[b][wq][lane][0] = make_float4(psi[0], psi[1], psi[2], psi[3]);
            S.psi[b][wq][lane][1] = make_float4(psi[4], psi[5], psi[6], psi[7]);
            S.q[b][wq][lane] = q;
            S.u[b][wq][lane][0] = make_float4(fc * phi[0], fc * phi[1], fc * phi[2], fc * phi[3]);
            S.u[b][wq][lane][1] = make_float4(fc * phi[4], fc * phi[5], fc * phi[6], fc * phi[7]);
            S.src[b][wq][lane] = a.lsrc[st.pos + lane];
        }
    };
    float2 mu = make_float2(0.f, 0.f), hu = mu, hb = mu, mun = mu, hun = mu;
    double gx = 0.0, gy = 0.0, gz = 0.0;  // fp64: exact sums of antisymmetric terms
    float vr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint32_t phase = 0;
    Step cur = schedule();
    load_step(0, cur);
    if (cur.first) {
        mu = reinterpret_cast<const float2*>(MB + (size_t)cur.r * F)[lane];
        hu = reinterpret_cast<const float2*>(Hl + (size_t)cur.r * F)[lane];
    }
    for (int step = 0; step < steps; ++step) {
        const int bsel = step & 1;
        const int ne = cur.ne;
        const float2 su = __fadd2_rn(mu, hu), ndu = __fadd2_rn(make_float2(-mu.x, -mu.y), hu);  // S_u, -D_u
        __syncwarp();
        // (1) feature lanes: hbar, and X rows (tf32 hi / lo) of the A operand
        for (int i0 = 0; i0 < ne; i0 += kBatch) {
            float2 mw[kBatch], hw[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                if (i0 + j < ne) {
                    const int w = S.src[bsel][wq][i0 + j];
                    mw[j] = __ldg(reinterpret_cast<const float2*>(MB + (size_t)w * F) + lane);
                    hw[j] = __ldg(reinterpret_cast<const float2*>(Hl + (size_t)w * F) + lane);
                }
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const int i = i0 + j;
                if (i < ne) {
                    const float4 ua = S.u[bsel][wq][i][0], ub = S.u[bsel][wq][i][1];
                    float2 sv = f2mul(P2[0], bc2(ua.x));
                    sv = f2fma(P2[1], bc2(ua.y), sv);
                    sv = f2fma(P2[2], bc2(ua.z), sv);
                    sv = f2fma(P2[3], bc2(ua.w), sv);
                    sv = f2fma(P2[4], bc2(ub.x), sv);
                    sv = f2fma(P2[5], bc2(ub.y), sv);
                    sv = f2fma(P2[6], bc2(ub.z), sv);
                    sv = f2fma(P2[7], bc2(ub.w), sv);
                    hb = f2fma(mw[j], sv, hb);
                    // 2 X = S_u S_w - D_u D_w (S = mbar + h, D = mbar - h):
                    // symmetric under u <-> w whatever ptxas fuses, so the
                    // reverse edge gets bitwise the same X row, G and dsum
                    // (exact Newton's third law; the 1/2 is applied to dsum)
                    const float2 sw = __fadd2_rn(mw[j], hw[j]);
                    const float2 dw = __fadd2_rn(mw[j], make_float2(-hw[j].x, -hw[j].y));
                    const float2 x = f2fma(su, sw, f2mul(ndu, dw));
                    float2 xh, xl;
                    split2(x, xh, xl);
                    const int off = xoff(row0 + i, 2 * lane);
                    *reinterpret_cast<float2*>(S.x_hi + off) = xh;
                    *reinterpret_cast<float2*>(S.x_lo + off) = xl;
                }
            }
        }
        // (2) G = X P on the tensor cores (3xTF32), one thread issues
        tc::fence_async_smem();
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (tid == 0) {
#pragma unroll
            for (int ks = 0; ks < F / 8; ++ks) {
                const uint64_t ah = sdesc2(S.x_hi + ks * 2 * kXLbo, kXLbo, kXSbo);
                const uint64_t al = sdesc2(S.x_lo + ks * 2 * kXLbo, kXLbo, kXSbo);
                const uint64_t bh = sdesc2(S.p_hi + ks * 2 * kPLbo, kPLbo, kPSbo);
                const uint64_t bl = sdesc2(S.p_lo + ks * 2 * kPLbo, kPLbo, kPSbo);
                tc::mma_tf32(tmem, ah, bh, idesc, ks > 0);
                tc::mma_tf32(tmem, al, bh, idesc, true);
                tc::mma_tf32(tmem, ah, bl, idesc, true);
            }
            tc::commit(&S.mbar);
        }
        // (3) the next step's records and own rows load under the MMA
        const Step nxt = schedule();
        load_step(bsel ^ 1, nxt);
        if (nxt.first) {
            mun = reinterpret_cast<const float2*>(MB + (size_t)nxt.r * F)[lane];
            hun = reinterpret_cast<const float2*>(Hl + (size_t)nxt.r * F)[lane];
        }
        tc::mbar_wait(&S.mbar, phase);
        phase ^= 1u;
        tc::fence_after();
        // (4) edge lanes: dsum, gradient, virial (the lane that computed the
        // slot's scalars reads the slot's TMEM row)
        float G[8];
        tmem_ld8(trow, G);
        {
            float Gs[8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) Gs[kk] = __shfl_sync(kFull, G[kk], (lane + kSlots * (wq >> 2)) & 31);
            if (lane < ne) {
                const float4 q = S.q[bsel][wq][lane];
                const float4 p0 = S.psi[bsel][wq][lane][0], p1 = S.psi[bsel][wq][lane][1];
                const float psi[K] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
                float dsum = 0.f;
#pragma unroll
                for (int kk = 0; kk < K; ++kk) dsum = fmaf(psi[kk], Gs[kk], dsum);
                const float coef = (0.5f * dsum) / q.w;
                gx -= (double)(q.x * coef);
                gy -= (double)(q.y * coef);
                gz -= (double)(q.z * coef);
                const float ch = 0.5f * coef;
                vr[0] = fmaf(ch * q.x, q.x, vr[0]);
                vr[1] = fmaf(ch * q.y, q.y, vr[1]);
                vr[2] = fmaf(ch * q.z, q.z, vr[2]);
                vr[3] = fmaf(ch * q.x, q.y, vr[3]);
                vr[4] = fmaf(ch * q.x, q.z, vr[4]);
                vr[5] = fmaf(ch * q.y, q.z, vr[5]);
            }
        }
        // (5) node complete: one writer per element
        if (cur.last) {
            float2* hbp = reinterpret_cast<float2*>(HB + (size_t)cur.k * F) + lane;
            const float2 old = *hbp;
            *hbp = make_float2(old.x + hb.x, old.y + hb.y);
            const double sx = gwarp_sumd(gx), sy = gwarp_sumd(gy), sz = gwarp_sumd(gz);
#pragma unroll
            for (int c = 0; c < 6; ++c) vr[c] = gwarp_sum(vr[c]);
            if (lane == 0) {
                double4 gr = GRAD[cur.k];
                gr.x += sx;
                gr.y += sy;
                gr.z += sz;
                GRAD[cur.k] = gr;
#pragma unroll
                for (int c = 0; c < 6; ++c) vir[c] += (double)vr[c];
            }
            hb = make_float2(0.f, 0.f);
            gx = gy = gz = 0.0;
#pragma unroll
            for (int c = 0; c < 6; ++c) vr[c] = 0.f;
        }
        if (nxt.first) {
            mu = mun;
            hu = hun;
        }
        cur = nxt;
        // no barrier here: the next MMA is issued after the next step's
        // barrier, which every warp reaches only after this epilogue's TMEM
        // reads (fenced before that barrier); X is free once the MMA committed
    }
    // fp64 virial: warp records in fixed order -> CTA record
    __shared__ double wv[kBW][6];
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < 6; ++c) wv[wq][c] = vir[c];
    tc::fence_before();
    __syncthreads();
    if (tid < 6) {
        double acc = 0.0;
        for (int w = 0; w < kBW; ++w) acc += wv[w][tid];
        vir_part[(size_t)blockIdx.x * 6 + tid] = acc;
    }
    if (wq == 0) tc::tmem_free(tmem, 32);
}


// ---------------------------------------------------------------------------
// backward edge pass, packed FP32 with a transposed warp reduction (default)
// ---------------------------------------------------------------------------
// dsum_e = sum_k psi_k (X P)_k = sum_f X_f s'_f with s' = P psi: every lane
// forms its two features' share of s' and of X . s' (8 + 1 FFMA2, the same
// work as the forward's s = P u), keeps one partial per edge of a 32-edge
// chunk, and one transposed butterfly (31 SHFL for 32 edges) leaves lane j
// with dsum of edge j.  The butterfly pairs lanes by their bits -- the same
// tree for every edge slot -- and fp32 addition commutes, so an edge and its
// reverse (bitwise-equal X rows and s') get bitwise-equal dsum: exact
// Newton's third law as in the tcgen05 form, with no CTA-wide MMA steps.
constexpr int kFW = 8;  // warps per CTA

struct BwdFfSmem {
    float4 u[kFW][32][2];    // fc * phi_k of the chunk's edges
    float4 psi[kFW][32][2];  // psi_k of the chunk's edges
    int src[kFW][32];
};

// lane l ends with the sum over lanes of v[l % C] (fixed pairing tree)
template <int C>
__device__ __forceinline__ float transpose_reduce(float (&v)[C], int lane) {
#pragma unroll
    for (int o = 16; o >= C; o >>= 1)
#pragma unroll
        for (int i = 0; i < C; ++i) v[i] += __shfl_xor_sync(kFull, v[i], o);
#pragma unroll
    for (int o = C / 2; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = up ? v[i] : v[i + o];
            const float keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(kFull, send, o);
        }
    }
    return v[0];
}

template <int C, int MINB>  // edges per chunk, CTAs per SM
__global__ void __launch_bounds__(kFW * 32, MINB) k_wide_bwd_edge_ff(GenModel g, Basis bs, ConvArgs a,
                                                                  const float* __restrict__ MB,
                                                                  const float* __restrict__ Hl,
                                                                  float* __restrict__ HB,
                                                                  double4* __restrict__ GRAD,
                                                                  double* __restrict__ vir_part) {
    __shared__ __align__(16) BwdFfSmem S;
    __shared__ double wv[kFW][6];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    float2 P2[K];  // (P[2l][k], P[2l+1][k])
#pragma unroll
    for (int k = 0; k < K; ++k) P2[k] = make_float2(g.P[(2 * lane) * K + k], g.P[(2 * lane + 1) * K + k]);
    if (lane < 6) wv[wq][lane] = 0.0;  // per-warp fp64 virial (lane 0 accumulates)
    __syncwarp();
    for (int64_t k = (int64_t)blockIdx.x * kFW + wq; k < a.n; k += (int64_t)gridDim.x * kFW) {
        const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t r = a.crow ? (int64_t)a.crow[v] : v;
        const int e0 = a.row[v], e1 = a.row[v + 1];
        const float2 mu = reinterpret_cast<const float2*>(MB + (size_t)r * F)[lane];
        const float2 hu = reinterpret_cast<const float2*>(Hl + (size_t)r * F)[lane];
        const float2 su = __fadd2_rn(mu, hu), ndu = __fadd2_rn(make_float2(-mu.x, -mu.y), hu);  // S_u, -D_u
        float2 hb = make_float2(0.f, 0.f);
        double gx = 0.0, gy = 0.0, gz = 0.0;  // fp64: exact sums of antisymmetric terms
        float vr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int eb = e0; eb < e1; eb += C) {
            const int ne = min(C, e1 - eb);
            // (1) edge lanes: radial scalars of the chunk
            float4 q = make_float4(0.f, 0.f, 0.f, 1.f);
            if (lane < ne) {
                q = __ldg(a.vd + eb + lane);
                const float d = q.w;
                float phi[K];
                phi8(bs, d, phi);
                float sn, cs;
                __sincosf(d * bs.pi_rc, &sn, &cs);
                const bool in = d < bs.rc;
                const float fc = in ? 0.5f * cs + 0.5f : 0.0f;
                const float dfc = in ? -0.5f * bs.pi_rc * sn : 0.0f;
                const float x0 = d * bs.isg, stp = bs.mus * bs.isg;
                const float ca = dfc - 2.0f * fc * bs.isg * x0, cb = 2.0f * fc * bs.isg * stp;
                float psi[K];
#pragma unroll
                for (int kk = 0; kk < K; ++kk) psi[kk] = phi[kk] * fmaf(cb, (float)kk, ca);
                S.psi[wq][lane][0] = make_float4(psi[0], psi[1], psi[2], psi[3]);
                S.psi[wq][lane][1] = make_float4(psi[4], psi[5], psi[6], psi[7]);
                S.u[wq][lane][0] = make_float4(fc * phi[0], fc * phi[1], fc * phi[2], fc * phi[3]);
                S.u[wq][lane][1] = make_float4(fc * phi[4], fc * phi[5], fc * phi[6], fc * phi[7]);
                S.src[wq][lane] = a.lsrc[eb + lane];
            }
            __syncwarp();
            // (2) feature lanes: h_bar and this lane's share of X . s' per edge
            float part[C];
#pragma unroll
            for (int i0 = 0; i0 < C; i0 += 4) {
                if (i0 < ne) {
                    float2 mw[4], hw[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int w = S.src[wq][min(i0 + j, ne - 1)];
                        mw[j] = __ldg(reinterpret_cast<const float2*>(MB + (size_t)w * F) + lane);
                        hw[j] = __ldg(reinterpret_cast<const float2*>(Hl + (size_t)w * F) + lane);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int i = i0 + j;
                        part[i] = 0.f;
                        if (i < ne) {
                            const float4 ua = S.u[wq][i][0], ub = S.u[wq][i][1];
                            float2 sv = f2mul(P2[0], bc2(ua.x));
                            sv = f2fma(P2[1], bc2(ua.y), sv);
                            sv = f2fma(P2[2], bc2(ua.z), sv);
                            sv = f2fma(P2[3], bc2(ua.w), sv);
                            sv = f2fma(P2[4], bc2(ub.x), sv);
                            sv = f2fma(P2[5], bc2(ub.y), sv);
                            sv = f2fma(P2[6], bc2(ub.z), sv);
                            sv = f2fma(P2[7], bc2(ub.w), sv);
                            hb = f2fma(mw[j], sv, hb);
                            const float4 pa = S.psi[wq][i][0], pb = S.psi[wq][i][1];
                            float2 sp = f2mul(P2[0], bc2(pa.x));
                            sp = f2fma(P2[1], bc2(pa.y), sp);
                            sp = f2fma(P2[2], bc2(pa.z), sp);
                            sp = f2fma(P2[3], bc2(pa.w), sp);
                            sp = f2fma(P2[4], bc2(pb.x), sp);
                            sp = f2fma(P2[5], bc2(pb.y), sp);
                            sp = f2fma(P2[6], bc2(pb.z), sp);
                            sp = f2fma(P2[7], bc2(pb.w), sp);
                            // 2 X = S_u S_w - D_u D_w: symmetric under u <-> w
                            const float2 sw = __fadd2_rn(mw[j], hw[j]);
                            const float2 dw = __fadd2_rn(mw[j], make_float2(-hw[j].x, -hw[j].y));
                            const float2 x = f2fma(su, sw, f2mul(ndu, dw));
                            const float2 xs = f2mul(x, sp);
                            part[i] = __fadd_rn(xs.x, xs.y);
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) part[i0 + j] = 0.f;
                }
            }
            // (3) lane j: dsum of edge j, gradient and virial
            const float dsum = transpose_reduce<C>(part, lane);
            if (lane < ne) {
                const float coef = (0.5f * dsum) / q.w;
                gx -= (double)(q.x * coef);
                gy -= (double)(q.y * coef);
                gz -= (double)(q.z * coef);
                const float ch = 0.5f * coef;
                vr[0] = fmaf(ch * q.x, q.x, vr[0]);
                vr[1] = fmaf(ch * q.y, q.y, vr[1]);
                vr[2] = fmaf(ch * q.z, q.z, vr[2]);
                vr[3] = fmaf(ch * q.x, q.y, vr[3]);
                vr[4] = fmaf(ch * q.x, q.z, vr[4]);
                vr[5] = fmaf(ch * q.y, q.z, vr[5]);
            }
            __syncwarp();
        }
        // node complete: one writer per element
        float2* hbp = reinterpret_cast<float2*>(HB + (size_t)k * F) + lane;
        const float2 old = *hbp;
        *hbp = make_float2(old.x + hb.x, old.y + hb.y);
        const double sx = gwarp_sumd(gx), sy = gwarp_sumd(gy), sz = gwarp_sumd(gz);
#pragma unroll
        for (int c = 0; c < 6; ++c) vr[c] = gwarp_sum(vr[c]);
        if (lane == 0) {
            double4 gr = GRAD[k];
            gr.x += sx;
            gr.y += sy;
            gr.z += sz;
            GRAD[k] = gr;
#pragma unroll
            for (int c = 0; c < 6; ++c) wv[wq][c] += (double)vr[c];
        }
    }
    // fp64 virial: warp records in fixed order -> CTA record
    __syncthreads();
    if (threadIdx.x < 6) {
        double acc = 0.0;
        for (int w = 0; w < kFW; ++w) acc += wv[w][threadIdx.x];
        vir_part[(size_t)blockIdx.x * 6 + threadIdx.x] = acc;
    }
}

// Same pass with the per-edge partials in shared memory instead of
// registers: lane l stores its share of X . s' for slot i at part[i][l]
// (one conflict-free row per edge), and lane j then sums row j over
// l = 0..31 in order (8 LDS.128) -- the same order for every edge, so the
// exactness argument above holds; 32 registers fewer (three CTAs per SM).
// Slots are padded to a multiple of BATCH with u = psi = 0 and a valid row,
// whose terms are exact zeros: no per-slot branches in the feature loop.
constexpr int kPartLd = 36;  // row stride (floats): 16-byte reads conflict-free

struct BwdSmSmem {
    float4 u[kFW][32][2];
    float4 psi[kFW][32][2];
    int src[kFW][32];
    float part[kFW][32][kPartLd];
};

template <int BATCH, int MINB, bool HBAR = true>
__global__ void __launch_bounds__(kFW * 32, MINB) k_wide_bwd_edge_sm(GenModel g, Basis bs, ConvArgs a,
                                                                     const float* __restrict__ MB,
                                                                     const float* __restrict__ Hl,
                                                                     float* __restrict__ HB,
                                                                     double4* __restrict__ GRAD,
                                                                     double* __restrict__ vir_part) {
    extern __shared__ __align__(16) unsigned char smraw[];
    BwdSmSmem& S = *reinterpret_cast<BwdSmSmem*>(smraw);
    __shared__ double wv[kFW][6];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    float2 P2[K];  // (P[2l][k], P[2l+1][k])
#pragma unroll
    for (int k = 0; k < K; ++k) P2[k] = make_float2(g.P[(2 * lane) * K + k], g.P[(2 * lane + 1) * K + k]);
    if (lane < 6) wv[wq][lane] = 0.0;  // per-warp fp64 virial (lane 0 accumulates)
    __syncwarp();
    float* prow = &S.part[wq][0][lane];
    for (int64_t k = (int64_t)blockIdx.x * kFW + wq; k < a.n; k += (int64_t)gridDim.x * kFW) {
        const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t r = a.crow ? (int64_t)a.crow[v] : v;
        const int e0 = a.row[v], e1 = a.row[v + 1];
        const float2 mu = reinterpret_cast<const float2*>(MB + (size_t)r * F)[lane];
        const float2 hu = reinterpret_cast<const float2*>(Hl + (size_t)r * F)[lane];
        const float2 su = __fadd2_rn(mu, hu), ndu = __fadd2_rn(make_float2(-mu.x, -mu.y), hu);  // S_u, -D_u
        float2 hb = make_float2(0.f, 0.f);
        double gx = 0.0, gy = 0.0, gz = 0.0;  // fp64: exact sums of antisymmetric terms
        float vr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int eb = e0; eb < e1; eb += 32) {
            const int ne = min(32, e1 - eb);
            const int nep = (ne + BATCH - 1) / BATCH * BATCH;
            // (1) edge lanes: radial scalars of the chunk (padding: zeros)
            float4 q = make_float4(0.f, 0.f, 0.f, 1.f);
            if (lane < ne) {
                q = __ldg(a.vd + eb + lane);
                const float d = q.w;
                float phi[K];
                phi8(bs, d, phi);
                float sn, cs;
                __sincosf(d * bs.pi_rc, &sn, &cs);
                const bool in = d < bs.rc;
                const float fc = in ? 0.5f * cs + 0.5f : 0.0f;
                const float dfc = in ? -0.5f * bs.pi_rc * sn : 0.0f;
                const float x0 = d * bs.isg, stp = bs.mus * bs.isg;
                const float ca = dfc - 2.0f * fc * bs.isg * x0, cb = 2.0f * fc * bs.isg * stp;
                float psi[K];
#pragma unroll
                for (int kk = 0; kk < K; ++kk) psi[kk] = phi[kk] * fmaf(cb, (float)kk, ca);
                S.psi[wq][lane][0] = make_float4(psi[0], psi[1], psi[2], psi[3]);
                S.psi[wq][lane][1] = make_float4(psi[4], psi[5], psi[6], psi[7]);
                if (HBAR) {
                    S.u[wq][lane][0] = make_float4(fc * phi[0], fc * phi[1], fc * phi[2], fc * phi[3]);
                    S.u[wq][lane][1] = make_float4(fc * phi[4], fc * phi[5], fc * phi[6], fc * phi[7]);
                }
                S.src[wq][lane] = a.lsrc[eb + lane];
            } else if (lane < nep) {
                const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
                S.psi[wq][lane][0] = S.psi[wq][lane][1] = S.u[wq][lane][0] = S.u[wq][lane][1] = z4;
                S.src[wq][lane] = (int)r;
            }
            __syncwarp();
            // (2) feature lanes: h_bar and this lane's share of X . s' per edge
            for (int i0 = 0; i0 < nep; i0 += BATCH) {
                float2 mw[BATCH], hw[BATCH];
#pragma unroll
                for (int j = 0; j < BATCH; ++j) {
                    const int w = S.src[wq][i0 + j];
                    mw[j] = __ldg(reinterpret_cast<const float2*>(MB + (size_t)w * F) + lane);
                    hw[j] = __ldg(reinterpret_cast<const float2*>(Hl + (size_t)w * F) + lane);
                }
#pragma unroll
                for (int j = 0; j < BATCH; ++j) {
                    const int i = i0 + j;
                    if constexpr (HBAR) {  // layer 0: the embedding gradient is never read
                        const float4 ua = S.u[wq][i][0], ub = S.u[wq][i][1];
                        float2 sv = f2mul(P2[0], bc2(ua.x));
                        sv = f2fma(P2[1], bc2(ua.y), sv);
                        sv = f2fma(P2[2], bc2(ua.z), sv);
                        sv = f2fma(P2[3], bc2(ua.w), sv);
                        sv = f2fma(P2[4], bc2(ub.x), sv);
                        sv = f2fma(P2[5], bc2(ub.y), sv);
                        sv = f2fma(P2[6], bc2(ub.z), sv);
                        sv = f2fma(P2[7], bc2(ub.w), sv);
                        hb = f2fma(mw[j], sv, hb);
                    }
                    const float4 pa = S.psi[wq][i][0], pb = S.psi[wq][i][1];
                    float2 sp = f2mul(P2[0], bc2(pa.x));
                    sp = f2fma(P2[1], bc2(pa.y), sp);
                    sp = f2fma(P2[2], bc2(pa.z), sp);
                    sp = f2fma(P2[3], bc2(pa.w), sp);
                    sp = f2fma(P2[4], bc2(pb.x), sp);
                    sp = f2fma(P2[5], bc2(pb.y), sp);
                    sp = f2fma(P2[6], bc2(pb.z), sp);
                    sp = f2fma(P2[7], bc2(pb.w), sp);
                    // 2 X = S_u S_w - D_u D_w: symmetric under u <-> w
                    const float2 sw = __fadd2_rn(mw[j], hw[j]);
                    const float2 dw = __fadd2_rn(mw[j], make_float2(-hw[j].x, -hw[j].y));
                    const float2 x = f2fma(su, sw, f2mul(ndu, dw));
                    const float2 xs = f2mul(x, sp);
                    prow[i * kPartLd] = __fadd_rn(xs.x, xs.y);
                }
            }
            __syncwarp();
            // (3) lane j: dsum of edge j (row j summed over lanes in order),
            // gradient and virial
            if (lane < ne) {
                const float4* pr = reinterpret_cast<const float4*>(&S.part[wq][lane][0]);
                float dsum = 0.f;
#pragma unroll
                for (int c4 = 0; c4 < 8; ++c4) {
                    const float4 p4 = pr[c4];
                    dsum = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(dsum, p4.x), p4.y), p4.z), p4.w);
                }
                const float coef = (0.5f * dsum) / q.w;
                gx -= (double)(q.x * coef);
                gy -= (double)(q.y * coef);
                gz -= (double)(q.z * coef);
                const float ch = 0.5f * coef;
                vr[0] = fmaf(ch * q.x, q.x, vr[0]);
                vr[1] = fmaf(ch * q.y, q.y, vr[1]);
                vr[2] = fmaf(ch * q.z, q.z, vr[2]);
                vr[3] = fmaf(ch * q.x, q.y, vr[3]);
                vr[4] = fmaf(ch * q.x, q.z, vr[4]);
                vr[5] = fmaf(ch * q.y, q.z, vr[5]);
            }
            __syncwarp();
        }
        // node complete: one writer per element
        if (HBAR) {
            float2* hbp = reinterpret_cast<float2*>(HB + (size_t)k * F) + lane;
            const float2 old = *hbp;
            *hbp = make_float2(old.x + hb.x, old.y + hb.y);
        }
        const double sx = gwarp_sumd(gx), sy = gwarp_sumd(gy), sz = gwarp_sumd(gz);
#pragma unroll
        for (int c = 0; c < 6; ++c) vr[c] = gwarp_sum(vr[c]);
        if (lane == 0) {
            double4 gr = GRAD[k];
            gr.x += sx;
            gr.y += sy;
            gr.z += sz;
            GRAD[k] = gr;
#pragma unroll
            for (int c = 0; c < 6; ++c) wv[wq][c] += (double)vr[c];
        }
    }
    // fp64 virial: warp records in fixed order -> CTA record
    __syncthreads();
    if (threadIdx.x < 6) {
        double acc = 0.0;
        for (int w = 0; w < kFW; ++w) acc += wv[w][threadIdx.x];
        vir_part[(size_t)blockIdx.x * 6 + threadIdx.x] = acc;
    }
}

// ---------------------------------------------------------------------------
// three-body stage (potential.cpp:664-741, 850-961), the generic kernels'
// slot conventions: slot j of center s = in-bond b0 + j (x_j -> s); TP / TH3 /
// SMR slot j belong to its reverse, the out-bond (s -> x_j)
// ---------------------------------------------------------------------------
struct Basis3 {
    float r3, pi_r3, isg3, mus3;
};
__host__ Basis3 make_basis3(const GenModel& g) {
    return Basis3{g.r3, 3.14159265358979f * g.inv_r3, g.inv_sigma3, g.mu_step3};
}
__device__ __forceinline__ void fcut3w(const Basis3& b, float d, float& fc, float& dfc) {
    float sn, cs;
    sincospif(d / b.r3, &sn, &cs);
    const bool in = d < b.r3;
    fc = in ? 0.5f * (cs + 1.0f) : 0.0f;
    dfc = in ? -0.5f * b.pi_r3 * sn : 0.0f;
}
// u3_k (with fc3) or its derivative du3_k, k = 0..7 (uniform across the warp)
__device__ __forceinline__ void u3w(const Basis3& b, float d, float u[K], bool deriv) {
    float fc, dfc;
    fcut3w(b, d, fc, dfc);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const float x = (d - b.mus3 * (float)k) * b.isg3;
        const float e = expf(-x * x);
        u[k] = deriv ? e * (dfc - 2.0f * fc * x * b.isg3) : fc * e;
    }
}
// the same, lane k < 8 evaluating u3_k and broadcasting it (warp-uniform d)
__device__ __forceinline__ void u3l(const Basis3& b, float d, int lane, float u[K], bool deriv) {
    float fc, dfc;
    fcut3w(b, d, fc, dfc);
    float mine = 0.f;
    if (lane < K) {
        const float x = (d - b.mus3 * (float)lane) * b.isg3;
        const float e = expf(-x * x);
        mine = deriv ? e * (dfc - 2.0f * fc * x * b.isg3) : fc * e;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) u[k] = __shfl_sync(kFull, mine, k);
}
__device__ __forceinline__ float2 p3dot(const float2 P32[K], const float u[K]) {
    float2 t = f2mul(P32[0], bc2(u[0]));
#pragma unroll
    for (int k = 1; k < K; ++k) t = f2fma(P32[k], bc2(u[k]), t);
    return t;
}

// TT[b] = P3 u3(d_b) for the in-bonds of every center
__global__ void __launch_bounds__(kConvWarps * 32) k_wide_tb_t(GenModel g, Basis3 b3, BondArgs a,
                                                               float* __restrict__ TT) {
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    float2 P32[K];
#pragma unroll
    for (int k = 0; k < K; ++k) P32[k] = make_float2(g.P3[(2 * lane) * K + k], g.P3[(2 * lane + 1) * K + k]);
    for (int64_t k = (int64_t)blockIdx.x * kConvWarps + wq; k < a.n; k += (int64_t)gridDim.x * kConvWarps) {
        const int64_t s = a.nodes ? (int64_t)a.nodes[k] : k;
        const int b0 = a.brow[s], b1 = a.brow[s + 1];
        for (int bb = b0; bb < b1; bb += 32) {  // lane i loads bond bb + i's distance
            const float dl = bb + lane < b1 ? a.vd[a.bedge[bb + lane]].w : 1.0f;
            const int nbb = min(32, b1 - bb);
            for (int i = 0; i < nbb; ++i) {
                float u[K];
                u3l(b3, __shfl_sync(kFull, dl, i), lane, u, false);
                reinterpret_cast<float2*>(TT + (size_t)(bb + i) * F)[lane] = p3dot(P32, u);
            }
        }
    }
}

// q_u = sum_{b into u} t'_rev(b) (ascending b), h_u += tanh(W4 q_u), TH4
__global__ void __launch_bounds__(kConvWarps * 32) k_wide_tb_inject(GenModel g, BondArgs a,
                                                                    const float* __restrict__ TP,
                                                                    float* __restrict__ H,
                                                                    float* __restrict__ TH4) {
    __shared__ __align__(16) float2 sWT[F][F / 2];  // (W4[2l][q], W4[2l+1][q])
    __shared__ __align__(16) float4 sq[kConvWarps][F / 4];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < F * F / 2; t += blockDim.x) {
        const int q = t / (F / 2), l = t % (F / 2);
        sWT[q][l] = make_float2(g.W4[(2 * l) * F + q], g.W4[(2 * l + 1) * F + q]);
    }
    __syncthreads();
    for (int64_t k = (int64_t)blockIdx.x * kConvWarps + wq; k < a.n; k += (int64_t)gridDim.x * kConvWarps) {
        const int64_t u = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t r = a.crow ? (int64_t)a.crow[u] : u;
        float2 q = make_float2(0.f, 0.f);
        for (int b = a.brow[u]; b < a.brow[u + 1]; ++b) {
            const float2 t = reinterpret_cast<const float2*>(TP + (size_t)a.brev[b] * F)[lane];
            q.x += t.x;
            q.y += t.y;
        }
        reinterpret_cast<float2*>(sq[wq])[lane] = q;
        __syncwarp();
        float2 z = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int q4 = 0; q4 < F / 4; ++q4) {
            const float4 mm = sq[wq][q4];
            z = f2fma(sWT[4 * q4][lane], bc2(mm.x), z);
            z = f2fma(sWT[4 * q4 + 1][lane], bc2(mm.y), z);
            z = f2fma(sWT[4 * q4 + 2][lane], bc2(mm.z), z);
            z = f2fma(sWT[4 * q4 + 3][lane], bc2(mm.w), z);
        }
        __syncwarp();
        const float2 th = make_float2(tanhf(z.x), tanhf(z.y));
        float2* hp = reinterpret_cast<float2*>(H + (size_t)r * F) + lane;
        const float2 h0 = *hp;
        *hp = make_float2(h0.x + th.x, h0.y + th.y);
        reinterpret_cast<float2*>(TH4 + (size_t)k * F)[lane] = th;
    }
}

// per-bond dense contraction Y = X W^T (N = K = 64) on tcgen05: each warp
// stages <= 16 slot rows per step (X in tf32 hi / lo); one thread issues
// the CTA's 24 MMAs; the row's owner lane then reads its 64 outputs
constexpr int kTW = 8;           // warps per CTA
constexpr int kZLd = 68;         // z row stride (floats) in the epilogue: conflict-free 16-byte stores
static_assert(kSlots * kZLd * 4 <= 2 * kXSbo && 32 * kSlots * 4 <= 2 * kXSbo, "per-warp scratch");
constexpr int kWBytes = 8 * kPSbo;  // 64 rows (N) x 64 K, dense (LBO 128, SBO 2048)

struct TbSmem {  // two CTAs per SM: keep 2 x (sizeof + 1 KB) <= 228 KB
    unsigned char x_hi[kXBytes];
    unsigned char x_lo[kXBytes];
    unsigned char w_hi[kWBytes];
    unsigned char w_lo[kWBytes];
    int slot_b[kTW][kSlots];    // bond row of each slot
    union {
        float4 sq[kTW][32];         // forward: bond vectors of the current center (first 32)
        float4 du[kTW][kSlots][2];  // back1: du3_k of the step's slots
    };
    float2 fcd[kTW][kSlots];        // back1: (fc3, fc3') of the step's slots
    int steps_w[kTW];
    uint64_t mbar;
    uint32_t tbase;
};

static_assert(2 * (sizeof(TbSmem) + 1024) <= 228 * 1024, "three-body kernels: two CTAs per SM");

// B operand: B[n][k] = Wsrc[n * ldn + k * ldk] (tf32 hi / lo)
__device__ __forceinline__ void stage_w(TbSmem& S, const float* Wsrc, int ldn, int ldk) {
    for (int t = threadIdx.x; t < F * F; t += blockDim.x) {
        const int nn = t / F, kk = t % F;
        float hv, lv;
        tc::split_tf32(Wsrc[nn * ldn + kk * ldk], hv, lv);
        *reinterpret_cast<float*>(S.w_hi + poff(nn, kk)) = hv;
        *reinterpret_cast<float*>(S.w_lo + poff(nn, kk)) = lv;
    }
}

__device__ __forceinline__ void tb_mma(TbSmem& S, uint32_t tmem, uint32_t& phase, int N = F) {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = tc::idesc_tf32(128, N);
#pragma unroll
        for (int ks = 0; ks < F / 8; ++ks) {
            const uint64_t ah = sdesc2(S.x_hi + ks * 2 * kXLbo, kXLbo, kXSbo);
            const uint64_t al = sdesc2(S.x_lo + ks * 2 * kXLbo, kXLbo, kXSbo);
            const uint64_t bh = sdesc2(S.w_hi + ks * 2 * kPLbo, kPLbo, kPSbo);
            const uint64_t bl = sdesc2(S.w_lo + ks * 2 * kPLbo, kPLbo, kPSbo);
            tc::mma_tf32(tmem, ah, bh, idesc, ks > 0);
            tc::mma_tf32(tmem, al, bh, idesc, true);
            tc::mma_tf32(tmem, ah, bl, idesc, true);
        }
        tc::commit(&S.mbar);
    }
    tc::mbar_wait(&S.mbar, phase);
    phase ^= 1u;
    tc::fence_after();
}

__device__ __forceinline__ void stage_row_x(unsigned char* x_hi, unsigned char* x_lo, int row, int lane,
                                            float2 x) {
    float2 xh, xl;
    split2(x, xh, xl);
    const int off = xoff(row, 2 * lane);
    *reinterpret_cast<float2*>(x_hi + off) = xh;
    *reinterpret_cast<float2*>(x_lo + off) = xl;
}

__device__ __forceinline__ void stage_row(TbSmem& S, int row, int lane, float2 x) {
    float2 xh, xl;
    split2(x, xh, xl);
    const int off = xoff(row, 2 * lane);
    *reinterpret_cast<float2*>(S.x_hi + off) = xh;
    *reinterpret_cast<float2*>(S.x_lo + off) = xl;
}

// the 64 outputs of this lane's TMEM row
__device__ __forceinline__ void tmem_row64(uint32_t trow, float z[F]) {
    tc::tmem_ld32(trow, z);
    tc::tmem_ld32(trow + 32, z + 32);
}

// The warp's centers k = gw + j nw (j < my) and their bond ranges, fetched
// by the lanes 32 centers at a time: one dependent load chain (nodes ->
// brow) per 32 centers instead of one per center.  j is warp-uniform.
struct CenterMeta {
    int b0 = 0, nb = 0;  // lane l: center jbase + l
    int64_t jbase = -64;
};
__device__ __forceinline__ void center_bonds(const BondArgs& a, int64_t gw, int64_t nw, int64_t my, int lane,
                                             CenterMeta& m, int64_t j, int& b0, int& nb) {
    if (j < m.jbase || j >= m.jbase + 32) {
        m.jbase = j;
        const int64_t jj = j + lane;
        m.b0 = 0;
        m.nb = 0;
        if (jj < my) {
            const int64_t kk = gw + jj * nw;
            const int64_t c = a.nodes ? (int64_t)a.nodes[kk] : kk;
            m.b0 = a.brow[c];
            m.nb = a.brow[c + 1] - m.b0;
        }
    }
    b0 = __shfl_sync(kFull, m.b0, (int)(j - m.jbase));
    nb = __shfl_sync(kFull, m.nb, (int)(j - m.jbase));
}
// first center at or after j with bonds (my if none)
__device__ __forceinline__ int64_t next_center(const BondArgs& a, int64_t gw, int64_t nw, int64_t my, int lane,
                                               CenterMeta& m, int64_t j, int& b0, int& nb) {
    for (; j < my; ++j) {
        center_bonds(a, gw, nw, my, lane, m, j, b0, nb);
        if (nb > 0) return j;
    }
    b0 = nb = 0;
    return my;
}

// CTA-wide step count: every step packs 16 slots of a warp's consecutive
// centers, so a warp needs ceil(sum_centers n / 16) steps; max over warps
// (packed = false: every step holds slots of one center, sum of ceil(n / 16))
__device__ __forceinline__ int tb_steps(const BondArgs& a, int64_t gw, int64_t nw, int64_t my, int lane,
                                        int wq, int* steps_w, bool packed = true) {
    int st = 0;
    for (int64_t j = lane; j < my; j += 32) {
        const int64_t kk = gw + j * nw;
        const int64_t s = a.nodes ? (int64_t)a.nodes[kk] : kk;
        const int nbj = a.brow[s + 1] - a.brow[s];
        st += packed ? nbj : (nbj + kSlots - 1) / kSlots;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) st += __shfl_xor_sync(kFull, st, o);
    if (lane == 0) steps_w[wq] = packed ? (st + kSlots - 1) / kSlots : st;
    __syncthreads();
    int steps = 0;
    for (int w = 0; w < kTW; ++w) steps = max(steps, steps_w[w]);
    return steps;
}

// forward: per out-slot j of center s, m3 = sum_{o != j} c(o, j) t_o
// (ascending o, c = v_o . v_j / (d_o d_j)); z3 = W3 m3 on tcgen05;
// TP = t_j + fc3(d_j) tanh(z3), TH3 = tanh(z3)
__global__ void __launch_bounds__(kTW * 32, 2) k_wide_tb_forward(GenModel g, Basis3 b3, BondArgs a,
                                                                 const float* __restrict__ TT,
                                                                 float* __restrict__ TP,
                                                                 float* __restrict__ TH3) {
    extern __shared__ __align__(1024) unsigned char wsm[];
    TbSmem& S = *reinterpret_cast<TbSmem*>(wsm);
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    stage_w(S, g.W3, F, 1);  // B[n][k] = W3[n][k]: z_n = sum_k W3[n][k] m_k
    if (tid == 0) {
        tc::mbar_init(&S.mbar, 1);
        tc::fence_mbar_init();
    }
    if (wq == 0) tc::tmem_alloc(&S.tbase, F);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = S.tbase;
    const int row0 = 32 * (wq & 3) + kSlots * (wq >> 2);
    const uint32_t trow = tmem + ((uint32_t)(32 * (wq & 3)) << 16);
    const bool owner = (lane >> 4) == (wq >> 2);
    const int oslot = lane & 15;
    const int64_t gw = (int64_t)blockIdx.x * kTW + wq, nw = (int64_t)gridDim.x * kTW;
    const int64_t my = gw < a.n ? (a.n - 1 - gw) / nw + 1 : 0;
    const int steps = tb_steps(a, gw, nw, my, lane, wq, S.steps_w, false);

    uint32_t phase = 0;
    // current center: bonds [b0, b0 + nb), next slot jpos; the next center's
    // bond edges (en) and vectors (qn) are fetched one step ahead
    CenterMeta cmeta;
    int b0 = 0, nb = 0, jpos = 0, b0n = 0, nbn = 0;
    int64_t jcur = next_center(a, gw, nw, my, lane, cmeta, 0, b0, nb);
    if (lane < min(nb, 32)) S.sq[wq][lane] = a.vd[a.bedge[b0 + lane]];
    __syncwarp();
    int64_t jnext = next_center(a, gw, nw, my, lane, cmeta, jcur + 1, b0n, nbn);
    int en = lane < min(nbn, 32) ? __ldg(a.bedge + b0n + lane) : 0;
    float4 qn = make_float4(0.f, 0.f, 0.f, 1.f);
    for (int step = 0; step < steps; ++step) {
        if (jpos >= nb && jcur < my) {  // advance to the prefetched center
            __syncwarp();
            if (lane < min(nbn, 32)) S.sq[wq][lane] = qn;
            __syncwarp();
            jcur = jnext;
            b0 = b0n;
            nb = nbn;
            jpos = 0;
            jnext = next_center(a, gw, nw, my, lane, cmeta, jcur + 1, b0n, nbn);
            en = lane < min(nbn, 32) ? __ldg(a.bedge + b0n + lane) : 0;
        }
        // slots jpos .. jpos + ns - 1 of this center; o outer so each t_o row
        // is read once per step, m3 of the step's slots in registers.  The
        // warp's own A-operand rows are free here (the previous MMA has
        // completed): they hold the step's cosine table C[o][i] (x_hi) and
        // the epilogue's z rows (x_lo)
        const int ns = jpos < nb ? min(kSlots, nb - jpos) : 0;
        auto qof = [&](int o) { return o < 32 ? S.sq[wq][o] : a.vd[a.bedge[b0 + o]]; };
        float* Cm = reinterpret_cast<float*>(S.x_hi + (row0 >> 3) * kXSbo);  // [32][16]
        float* Zs = reinterpret_cast<float*>(S.x_lo + (row0 >> 3) * kXSbo);  // [16][kZLd]
        float2 m3[kSlots];
#pragma unroll
        for (int i = 0; i < kSlots; ++i) m3[i] = make_float2(0.f, 0.f);
        for (int oc = 0; oc < nb && ns > 0; oc += 32) {
            const int no = min(32, nb - oc);
            __syncwarp();
            // c(o, j) = v_o . v_j / (d_o d_j); 0 for o == j and unused slots
            for (int t = lane; t < no * kSlots; t += 32) {
                const int o = oc + (t >> 4), i = t & (kSlots - 1);
                float c = 0.f;
                if (i < ns && jpos + i != o) {
                    const float4 qo = qof(o), qj = qof(jpos + i);
                    c = (qo.x * qj.x + qo.y * qj.y + qo.z * qj.z) / (qo.w * qj.w);
                }
                Cm[t] = c;
            }
            __syncwarp();
            for (int o0 = 0; o0 < no; o0 += 4) {
                float2 tv[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)  // four t rows in flight
                    if (o0 + jj < no)
                        tv[jj] = __ldg(reinterpret_cast<const float2*>(TT + (size_t)(b0 + oc + o0 + jj) * F) + lane);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    if (o0 + jj >= no) break;
                    const float4* cr = reinterpret_cast<const float4*>(Cm + (o0 + jj) * kSlots);
#pragma unroll
                    for (int i4 = 0; i4 < kSlots / 4; ++i4) {  // ascending o; + 0 t_j on the diagonal
                        const float4 c4 = cr[i4];
                        m3[4 * i4] = f2fma(bc2(c4.x), tv[jj], m3[4 * i4]);
                        m3[4 * i4 + 1] = f2fma(bc2(c4.y), tv[jj], m3[4 * i4 + 1]);
                        m3[4 * i4 + 2] = f2fma(bc2(c4.z), tv[jj], m3[4 * i4 + 2]);
                        m3[4 * i4 + 3] = f2fma(bc2(c4.w), tv[jj], m3[4 * i4 + 3]);
                    }
                }
            }
        }
        if (lane < min(nbn, 32)) qn = __ldg(a.vd + en);  // next center's vectors (en has landed)
        __syncwarp();
#pragma unroll
        for (int i = 0; i < kSlots; ++i)
            if (i < ns) stage_row(S, row0 + i, lane, m3[i]);
        if (lane < ns) S.slot_b[wq][lane] = b0 + jpos + lane;
        jpos += ns;
        __syncwarp();
        tb_mma(S, tmem, phase);
        {   // z rows (TMEM lane = slot) -> shared memory -> feature lanes
            float z[F];
            tmem_row64(trow, z);
            if (owner && oslot < ns) {
                float4* zr = reinterpret_cast<float4*>(Zs + oslot * kZLd);
#pragma unroll
                for (int c4 = 0; c4 < F / 4; ++c4)
                    zr[c4] = make_float4(z[4 * c4], z[4 * c4 + 1], z[4 * c4 + 2], z[4 * c4 + 3]);
            }
        }
        float fcm = 0.f;
        if (lane < ns) {
            float dfc;
            fcut3w(b3, a.vd[a.bedge[S.slot_b[wq][lane]]].w, fcm, dfc);
        }
        __syncwarp();
        for (int i = 0; i < ns; ++i) {
            const int b = S.slot_b[wq][i];
            const float fc = __shfl_sync(kFull, fcm, i);
            const float2 zz = *reinterpret_cast<const float2*>(Zs + i * kZLd + 2 * lane);
            const float2 th = make_float2(tanhf(zz.x), tanhf(zz.y));
            const float2 t = __ldg(reinterpret_cast<const float2*>(TT + (size_t)b * F) + lane);
            reinterpret_cast<float2*>(TH3 + (size_t)b * F)[lane] = th;
            reinterpret_cast<float2*>(TP + (size_t)b * F)[lane] = make_float2(t.x + fc * th.x, t.y + fc * th.y);
        }
        __syncwarp();
    }
    tc::fence_before();
    __syncthreads();
    if (wq == 0) tc::tmem_free(tmem, F);
}

// backward phase 1 per slot j (out-bond e'_j = (s -> x_j)): tbar' = q_bar[x_j];
// VOUT = v_j (-(dbf + da) / d_j) with dbf = tbar' . th3 fc3', da = tbar' . (P3 u3');
// y = tbar' (.) fc3 (1 - th3^2), m_bar_3 = W3^T y.  Phase 2 only needs
// m_bar_3 through its products with t_o = P3 u3(d_o) and ds_o = P3 u3'(d_o),
// i.e. through E = P3^T m_bar_3 = (W3 P3)^T y (8 values per bond): one
// tcgen05 contraction Y (W3 P3) (M = 128 slots, N = 16 with 8 zero columns,
// K = 64) writes E instead of the 64-wide m_bar_3 rows
__global__ void __launch_bounds__(kTW * 32, 2) k_wide_tb_back1(GenModel g, Basis3 b3, BondArgs a,
                                                               const float* __restrict__ QB,
                                                               const float* __restrict__ TH3,
                                                               float* __restrict__ EB,
                                                               float4* __restrict__ VOUT) {
    extern __shared__ __align__(1024) unsigned char wsm[];
    TbSmem& S = *reinterpret_cast<TbSmem*>(wsm);
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    // B[n][f] = sum_q W3[f][q] P3[q][n] (n < 8), 0 (n = 8..15)
    for (int t = tid; t < 16 * F; t += blockDim.x) {
        const int nn = t / F, f = t % F;
        float x = 0.f;
        if (nn < K)
            for (int q = 0; q < F; ++q) x = fmaf(g.W3[f * F + q], g.P3[q * K + nn], x);
        float hv, lv;
        tc::split_tf32(x, hv, lv);
        *reinterpret_cast<float*>(S.w_hi + poff(nn, f)) = hv;
        *reinterpret_cast<float*>(S.w_lo + poff(nn, f)) = lv;
    }
    if (tid == 0) {
        tc::mbar_init(&S.mbar, 1);
        tc::fence_mbar_init();
    }
    if (wq == 0) tc::tmem_alloc(&S.tbase, 32);
    float2 P32[K];
#pragma unroll
    for (int k = 0; k < K; ++k) P32[k] = make_float2(g.P3[(2 * lane) * K + k], g.P3[(2 * lane + 1) * K + k]);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = S.tbase;
    const int row0 = 32 * (wq & 3) + kSlots * (wq >> 2);
    const uint32_t trow = tmem + ((uint32_t)(32 * (wq & 3)) << 16);
    const bool owner = (lane >> 4) == (wq >> 2);
    const int oslot = lane & 15;
    const int64_t gw = (int64_t)blockIdx.x * kTW + wq, nw = (int64_t)gridDim.x * kTW;
    const int64_t my = gw < a.n ? (a.n - 1 - gw) / nw + 1 : 0;
    const int steps = tb_steps(a, gw, nw, my, lane, wq, S.steps_w);

    uint32_t phase = 0;
    // slot schedule (consecutive bonds of consecutive centers, 16 per step):
    // lane i takes slot i's bond.  The next step's indices are fetched one
    // step ahead in three stages (bond edge; vector and source atom; source
    // row), each under the current step's work
    CenterMeta cmeta;
    int64_t jcur = -1;
    int b0 = 0, nb = 0, jpos = 0;
    auto schedule = [&](int& ns_o, int& myb_o) {
        ns_o = 0;
        myb_o = -1;
        while (ns_o < kSlots) {
            if (jpos >= nb) {
                if (jcur >= my) break;
                jcur = next_center(a, gw, nw, my, lane, cmeta, jcur + 1, b0, nb);
                jpos = 0;
                if (nb == 0) break;
                continue;
            }
            const int take = min(kSlots - ns_o, nb - jpos);
            if (lane >= ns_o && lane < ns_o + take) myb_o = b0 + jpos + (lane - ns_o);
            ns_o += take;
            jpos += take;
        }
    };
    int ns, myb;
    schedule(ns, myb);
    float4 qm = make_float4(0.f, 0.f, 0.f, 1.f);
    int rxm = 0;
    if (myb >= 0) {
        const int e = a.bedge[myb];
        qm = a.vd[e];
        const int x = a.esrc[e];
        rxm = a.crow ? a.crow[x] : x;
    }
    int nsn, mybn;
    schedule(nsn, mybn);
    int en = mybn >= 0 ? __ldg(a.bedge + mybn) : 0;
    for (int step = 0; step < steps; ++step) {
        // lane i: slot i's bond, its radial scalars into shared memory
        if (myb >= 0) {
            float fc, dfc, du[K];
            fcut3w(b3, qm.w, fc, dfc);
            u3w(b3, qm.w, du, true);
            S.du[wq][lane][0] = make_float4(du[0], du[1], du[2], du[3]);
            S.du[wq][lane][1] = make_float4(du[4], du[5], du[6], du[7]);
            S.fcd[wq][lane] = make_float2(fc, dfc);
            S.slot_b[wq][lane] = myb;
        }
        __syncwarp();
        // feature lanes: y rows (A operand) and this lane's share of
        // dbf + da per slot; one transposed reduction for the 16 slots
        float part[kSlots];
#pragma unroll
        for (int i0 = 0; i0 < kSlots; i0 += 4) {
            if (i0 < ns) {
                float2 tpb[4], th[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {  // four slots' rows in flight
                    const int i = i0 + jj;
                    const int rx = __shfl_sync(kFull, rxm, i), b = __shfl_sync(kFull, myb, i);
                    if (i < ns) {
                        tpb[jj] = __ldg(reinterpret_cast<const float2*>(QB + (size_t)rx * F) + lane);
                        th[jj] = reinterpret_cast<const float2*>(TH3 + (size_t)b * F)[lane];
                    }
                }
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int i = i0 + jj;
                    part[i] = 0.f;
                    if (i < ns) {
                        const float4 d0 = S.du[wq][i][0], d1 = S.du[wq][i][1];
                        const float du[K] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
                        const float2 fcd = S.fcd[wq][i];
                        const float2 ds = p3dot(P32, du);
                        const float dbf = fmaf(tpb[jj].x * th[jj].x, fcd.y, (tpb[jj].y * th[jj].y) * fcd.y);
                        const float da = fmaf(tpb[jj].x, ds.x, tpb[jj].y * ds.y);
                        part[i] = dbf + da;
                        const float2 y = make_float2(tpb[jj].x * fcd.x * (1.0f - th[jj].x * th[jj].x),
                                                     tpb[jj].y * fcd.x * (1.0f - th[jj].y * th[jj].y));
                        stage_row(S, row0 + i, lane, y);
                    }
                }
            } else {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) part[i0 + jj] = 0.f;
            }
        }
        // next step's vector and source atom (its bond edge has landed)
        float4 qn = make_float4(0.f, 0.f, 0.f, 1.f);
        int xn = 0;
        if (mybn >= 0) {
            qn = __ldg(a.vd + en);
            xn = __ldg(a.esrc + en);
        }
        {
            const float tot = transpose_reduce<kSlots>(part, lane);  // lanes i, i + 16: slot i
            if (myb >= 0) {
                const float c0 = -tot / qm.w;
                VOUT[myb] = make_float4(qm.x * c0, qm.y * c0, qm.z * c0, 0.f);
            }
        }
        __syncwarp();
        tb_mma(S, tmem, phase, 16);
        float ev[8];
        tmem_ld8(trow, ev);
        if (owner && oslot < ns) {
            float4* ep = reinterpret_cast<float4*>(EB + (size_t)S.slot_b[wq][oslot] * K);
            ep[0] = make_float4(ev[0], ev[1], ev[2], ev[3]);
            ep[1] = make_float4(ev[4], ev[5], ev[6], ev[7]);
        }
        // rotate the pipeline: next step's source row, then the step after's bond edge
        ns = nsn;
        myb = mybn;
        qm = qn;
        rxm = mybn >= 0 ? (a.crow ? __ldg(a.crow + xn) : xn) : 0;
        schedule(nsn, mybn);
        en = mybn >= 0 ? __ldg(a.bedge + mybn) : 0;
    }
    tc::fence_before();
    __syncthreads();
    if (wq == 0) tc::tmem_free(tmem, 32);
}

// backward phase 2 per center s, slot j: the line edges through s.
//   (a) (e_j, e'_o): tbar_j += c m_bar_3,o; cb = m_bar_3,o . t_j;
//       VIN_j += -(-v_o/d_o + v_j c / d_j) / d_j cb
//   (b) (e_o, e'_j): cb2 = m_bar_3,j . t_o; VOUT_j += -(v_o/d_o - v_j c/d_j)/d_j cb2
//   then VIN_j += v_j db / d_j with db = tbar_j . ds_j, ds_j = P3 u3'(d_j)
//   virial (VIN - VOUT) (x) v_j.
// With t = P3 u3 and E = P3^T m_bar_3 (from back1): cb = E_o . u3_j,
// cb2 = E_j . u3_o, db = sum_o c_oj E_o . u3'_j -- 8-wide products.  The
// center's per-bond E, u3, u3' and v are staged in shared memory (lane o),
// then lane j sums its pairs over ascending o (no cross-lane reductions).
constexpr int kB2Warps = 8;
constexpr int kB2Max = 64;  // bonds per center staged; larger centers stage in windows

struct __align__(16) Back2Smem {
    float4 q[kB2Warps][kB2Max];
    float4 e[kB2Warps][kB2Max][2];
    float4 u[kB2Warps][kB2Max][2];
};

__device__ __forceinline__ float dot8(float4 a0, float4 a1, const float b[K]) {
    return fmaf(a1.w, b[7], fmaf(a1.z, b[6], fmaf(a1.y, b[5], fmaf(a1.x, b[4],
           fmaf(a0.w, b[3], fmaf(a0.z, b[2], fmaf(a0.y, b[1], a0.x * b[0])))))));
}

__device__ __forceinline__ void u3both(const Basis3& b, float d, float u[K], float du[K]) {
    float fc, dfc;
    fcut3w(b, d, fc, dfc);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const float x = (d - b.mus3 * (float)k) * b.isg3;
        const float e = expf(-x * x);
        u[k] = fc * e;
        du[k] = e * (dfc - 2.0f * fc * x * b.isg3);
    }
}

__global__ void __launch_bounds__(kB2Warps * 32) k_wide_tb_back2(GenModel g, Basis3 b3, BondArgs a,
                                                                 const float* __restrict__ EB,
                                                                 float4* __restrict__ VIN,
                                                                 float4* __restrict__ VOUT,
                                                                 double* __restrict__ vir_part) {
    extern __shared__ __align__(16) unsigned char b2sm[];
    Back2Smem& S = *reinterpret_cast<Back2Smem*>(b2sm);
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    double vir[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t k = (int64_t)blockIdx.x * kB2Warps + wq; k < a.n; k += (int64_t)gridDim.x * kB2Warps) {
        const int64_t s = a.nodes ? (int64_t)a.nodes[k] : k;
        const int b0 = a.brow[s], nb = a.brow[s + 1] - b0;
        for (int jb = 0; jb < nb; jb += 32) {  // slots j = jb + lane
            const int j = jb + lane;
            float4 qj = make_float4(0.f, 0.f, 0.f, 1.f), ej0 = make_float4(0.f, 0.f, 0.f, 0.f), ej1 = ej0;
            float uj[K], duj[K];
            if (j < nb) {
                qj = a.vd[a.bedge[b0 + j]];
                ej0 = reinterpret_cast<const float4*>(EB + (size_t)(b0 + j) * K)[0];
                ej1 = reinterpret_cast<const float4*>(EB + (size_t)(b0 + j) * K)[1];
                u3both(b3, qj.w, uj, duj);
            } else {
#pragma unroll
                for (int kk = 0; kk < K; ++kk) uj[kk] = duj[kk] = 0.f;
            }
            const float idj = 1.0f / qj.w;
            float vi[3] = {0.f, 0.f, 0.f}, vo3[3] = {0.f, 0.f, 0.f}, db = 0.f;
            for (int ob = 0; ob < nb; ob += kB2Max) {  // window of staged bonds o
                const int on = min(kB2Max, nb - ob);
                __syncwarp();
                for (int o = lane; o < on; o += 32) {
                    const float4 qo = a.vd[a.bedge[b0 + ob + o]];
                    S.q[wq][o] = qo;
                    S.e[wq][o][0] = reinterpret_cast<const float4*>(EB + (size_t)(b0 + ob + o) * K)[0];
                    S.e[wq][o][1] = reinterpret_cast<const float4*>(EB + (size_t)(b0 + ob + o) * K)[1];
                    float uo[K], duo[K];
                    u3both(b3, qo.w, uo, duo);
                    S.u[wq][o][0] = make_float4(uo[0], uo[1], uo[2], uo[3]);
                    S.u[wq][o][1] = make_float4(uo[4], uo[5], uo[6], uo[7]);
                }
                __syncwarp();
                if (j < nb) {
                    for (int oo = 0; oo < on; ++oo) {
                        const int o = ob + oo;
                        if (o == j) continue;  // the reverse pair
                        const float4 qo = S.q[wq][oo];
                        const float ido = 1.0f / qo.w;
                        const float c = (qj.x * qo.x + qj.y * qo.y + qj.z * qo.z) * idj * ido;
                        const float4 eo0 = S.e[wq][oo][0], eo1 = S.e[wq][oo][1];
                        const float4 uo0 = S.u[wq][oo][0], uo1 = S.u[wq][oo][1];
                        const float uo[K] = {uo0.x, uo0.y, uo0.z, uo0.w, uo1.x, uo1.y, uo1.z, uo1.w};
                        const float cb = dot8(eo0, eo1, uj);    // m_bar_3,o . t_j
                        const float cb2 = dot8(ej0, ej1, uo);   // m_bar_3,j . t_o
                        db = fmaf(c, dot8(eo0, eo1, duj), db);  // c (m_bar_3,o . ds_j)
                        const float qv[3] = {qo.x, qo.y, qo.z}, qw[3] = {qj.x, qj.y, qj.z};
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            vi[d] += -(-qv[d] * ido + qw[d] * idj * c) * idj * cb;
                            vo3[d] += -(qv[d] * ido - qw[d] * idj * c) * idj * cb2;
                        }
                    }
                }
            }
            if (j < nb) {
                const float vix = vi[0] + qj.x * db * idj, viy = vi[1] + qj.y * db * idj,
                            viz = vi[2] + qj.z * db * idj;
                float4 vo = VOUT[b0 + j];
                vo.x += vo3[0];
                vo.y += vo3[1];
                vo.z += vo3[2];
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
        }
    }
    // per-warp virial: lanes' partials summed in lane order
#pragma unroll
    for (int c = 0; c < 9; ++c) {
        double acc = 0.0;
        for (int l = 0; l < 32; ++l) acc += __shfl_sync(kFull, vir[c], l);
        if (lane == 0) vir_part[((int64_t)blockIdx.x * kB2Warps + wq) * 9 + c] = acc;
    }
}

}  // namespace

int wide_conv_grid(int64_t n) {
    int64_t g = (n + kConvWarps - 1) / kConvWarps;
    if (g > 148 * 8) g = 148 * 8;
    return (int)(g > 0 ? g : 1);
}

// backward edge kernel (GMD_WIDE_BWD, read per call: tests switch families):
// "sm" (default) partials in shared memory, 4 rows in flight, 3 CTAs per SM;
// "sm8" 8 rows in flight, 2 CTAs; "ff" / "ff16" register partials with the
// transposed butterfly, 32 / 16-edge chunks; "tc" G = X P on tcgen05 (also
// GMD_WIDE_TC=1)
enum { kBwdSm4, kBwdSm8, kBwdFf32, kBwdFf16, kBwdTc };
static int bwd_variant() {
    const char* tc = std::getenv("GMD_WIDE_TC");
    if (tc && std::atoi(tc) == 1) return kBwdTc;
    const char* v = std::getenv("GMD_WIDE_BWD");
    if (!v) return kBwdSm4;
    const std::string s(v);
    return s == "sm8" ? kBwdSm8 : s == "ff" ? kBwdFf32 : s == "ff16" ? kBwdFf16 : s == "tc" ? kBwdTc : kBwdSm4;
}
static int bwd_ctas_per_sm() {
    const int v = bwd_variant();
    return v == kBwdSm4 || v == kBwdFf16 ? 3 : 2;
}

int wide_bwd_grid(int64_t n) {  // one wave
    int64_t g = (n + kBW - 1) / kBW;
    const int64_t cap = 148 * bwd_ctas_per_sm();
    if (g > cap) g = cap;
    return (int)(g > 0 ? g : 1);
}

void launch_wide_conv(const GenModel& g, const ConvArgs& a, int layer, const float* Hin, float* Hout,
                      float* TH, double* per_atom, cudaStream_t s, const uint8_t* zs,
                      const unsigned* zmask) {
    if (a.n <= 0) return;
    if (zs)
        k_wide_conv<true><<<wide_conv_grid(a.n), kConvWarps * 32, 0, s>>>(g, make_basis(g), a, layer, Hin, Hout,
                                                                      TH, per_atom, zs, zmask);
    else
        k_wide_conv<<<wide_conv_grid(a.n), kConvWarps * 32, 0, s>>>(g, make_basis(g), a, layer, Hin, Hout,
                                                                    TH, per_atom);
    GMD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Per-node W^T y on tcgen05 (bwd_node and the three-body q_bar, potential.cpp
// :816-822, :460-470): m_bar = W^T (h_bar (.) (1 - th^2)) for 128 nodes per
// tile, D[r][g] = sum_f y[r][f] W[f][g] as M = 128, N = 64, K = 64 3xTF32
// into TMEM; warps stage rows (lanes over feature pairs, coalesced row
// reads), thread r writes node r's row from its TMEM lane.  Every row is an
// independent dot product, so results do not depend on the tile a node lands
// in (partition-invariant).  Persistent CTAs, W staged once.
// ---------------------------------------------------------------------------
struct NodeTcSmem {
    unsigned char x_hi[kXBytes];
    unsigned char x_lo[kXBytes];
    unsigned char w_hi[kWBytes];
    unsigned char w_lo[kWBytes];
    uint64_t mbar;
    uint32_t tbase;
};
constexpr int kNodeTcRows = 8;  // rows a warp loads before staging them

__global__ void __launch_bounds__(128, 2) k_wide_node_tc(GenModel g, int64_t n, const int32_t* __restrict__ nodes,
                                                        const int32_t* __restrict__ crow,
                                                        const float* __restrict__ W, float* __restrict__ HB,
                                                        const float* __restrict__ TH, float* __restrict__ MB,
                                                        int init) {
    extern __shared__ __align__(1024) unsigned char wsm[];
    NodeTcSmem& S = *reinterpret_cast<NodeTcSmem*>(wsm);
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    // B[n][k] = W[k][n]: D[r][n] = sum_k y[r][k] W[k][n]
    for (int t = tid; t < F * F; t += blockDim.x) {
        const int nn = t / F, kk = t % F;
        float hv, lv;
        tc::split_tf32(W[kk * F + nn], hv, lv);
        *reinterpret_cast<float*>(S.w_hi + poff(nn, kk)) = hv;
        *reinterpret_cast<float*>(S.w_lo + poff(nn, kk)) = lv;
    }
    if (tid == 0) {
        tc::mbar_init(&S.mbar, 1);
        tc::fence_mbar_init();
    }
    if (wq == 0) tc::tmem_alloc(&S.tbase, F);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = S.tbase;
    const uint32_t trow = tmem + ((uint32_t)(32 * wq) << 16);
    const float2 ro2 = make_float2(g.ro[2 * lane], g.ro[2 * lane + 1]);
    uint32_t phase = 0;
    const int64_t ntiles = (n + 127) / 128;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t k0 = tile * 128;
        // warp wq stages rows 32 wq .. 32 wq + 31, kNodeTcRows rows' loads in flight
        for (int j0 = 0; j0 < 32; j0 += kNodeTcRows) {
            float2 hb[kNodeTcRows], th[kNodeTcRows];
#pragma unroll
            for (int j = 0; j < kNodeTcRows; ++j) {
                const int64_t k = k0 + wq * 32 + j0 + j;
                hb[j] = make_float2(0.f, 0.f);
                th[j] = make_float2(0.f, 0.f);
                if (k < n) {
                    hb[j] = init ? ro2 : reinterpret_cast<const float2*>(HB + (size_t)k * F)[lane];
                    th[j] = reinterpret_cast<const float2*>(TH + (size_t)k * F)[lane];
                }
            }
#pragma unroll
            for (int j = 0; j < kNodeTcRows; ++j) {
                const int row = wq * 32 + j0 + j;
                const int64_t k = k0 + row;
                if (init && k < n) reinterpret_cast<float2*>(HB + (size_t)k * F)[lane] = hb[j];
                const float2 y = make_float2(hb[j].x * (1.0f - th[j].x * th[j].x),
                                             hb[j].y * (1.0f - th[j].y * th[j].y));
                stage_row_x(S.x_hi, S.x_lo, row, lane, y);
            }
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (tid == 0) {
            const uint32_t idesc = tc::idesc_tf32(128, F);
#pragma unroll
            for (int ks = 0; ks < F / 8; ++ks) {
                const uint64_t ah = sdesc2(S.x_hi + ks * 2 * kXLbo, kXLbo, kXSbo);
                const uint64_t al = sdesc2(S.x_lo + ks * 2 * kXLbo, kXLbo, kXSbo);
                const uint64_t bh = sdesc2(S.w_hi + ks * 2 * kPLbo, kPLbo, kPSbo);
                const uint64_t bl = sdesc2(S.w_lo + ks * 2 * kPLbo, kPLbo, kPSbo);
                tc::mma_tf32(tmem, ah, bh, idesc, ks > 0);
                tc::mma_tf32(tmem, al, bh, idesc, true);
                tc::mma_tf32(tmem, ah, bl, idesc, true);
            }
            tc::commit(&S.mbar);
        }
        tc::mbar_wait(&S.mbar, phase);
        phase ^= 1u;
        tc::fence_after();
        // thread tid holds row tid of the tile in its TMEM lane
        float z[F];
        tc::tmem_ld32(trow, z);
        tc::tmem_ld32(trow + 32, z + 32);
        const int64_t k = k0 + tid;
        if (k < n) {
            const int64_t v = nodes ? (int64_t)nodes[k] : k;
            const int64_t r = crow ? (int64_t)crow[v] : v;
            float4* dst = reinterpret_cast<float4*>(MB + (size_t)r * F);
#pragma unroll
            for (int c = 0; c < F / 4; ++c) dst[c] = make_float4(z[4 * c], z[4 * c + 1], z[4 * c + 2], z[4 * c + 3]);
        }
        // the next tile restages x and overwrites TMEM
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
    }
    if (wq == 0) tc::tmem_free(tmem, F);
}

static bool node_tc() {  // GMD_WIDE_NODE_TC=0: the FFMA2 warp-per-node kernel (A/B, tests)
    const char* v = std::getenv("GMD_WIDE_NODE_TC");
    return !(v && v[0] == '0');
}

static void launch_node(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                        const float* W, float* HB, const float* TH, float* MB, bool init, cudaStream_t s) {
    if (node_tc()) {
        static bool attr[64] = {};
        int dev = 0;
        GMD_CUDA(cudaGetDevice(&dev));
        if (dev < 0 || dev >= 64 || !attr[dev]) {
            GMD_CUDA(cudaFuncSetAttribute(k_wide_node_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)sizeof(NodeTcSmem)));
            if (dev >= 0 && dev < 64) attr[dev] = true;
        }
        int64_t gr = (n + 127) / 128;
        if (gr > 148 * 2) gr = 148 * 2;
        k_wide_node_tc<<<(int)gr, 128, sizeof(NodeTcSmem), s>>>(g, n, nodes, crow, W, HB, TH, MB, init ? 1 : 0);
    } else {
        k_wide_bwd_node<<<wide_conv_grid(n), kConvWarps * 32, 0, s>>>(g, n, nodes, crow, W, HB, TH, MB,
                                                                      init ? 1 : 0);
    }
    GMD_LAUNCH_CHECK();
}

void launch_wide_bwd_node(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                          int layer, float* HB, const float* TH, float* MB, bool init, cudaStream_t s) {
    if (n <= 0) return;
    launch_node(g, n, nodes, crow, g.W + (size_t)layer * F * F, HB, TH, MB, init, s);
}

static int back2_grid(int64_t n) {  // four CTAs of 8 warps per SM, one wave
    int64_t gr = (n + kB2Warps - 1) / kB2Warps;
    if (gr > 148 * 4) gr = 148 * 4;
    return (int)(gr > 0 ? gr : 1);
}

int wide_tb_grid(int64_t n) {  // records of launch_wide_tb_backward's virial (9 doubles each)
    return back2_grid(n) * kB2Warps;
}

void launch_wide_tb_t(const GenModel& g, const BondArgs& a, float* TT, cudaStream_t s) {
    if (a.n <= 0) return;
    k_wide_tb_t<<<wide_conv_grid(a.n), kConvWarps * 32, 0, s>>>(g, make_basis3(g), a, TT);
    GMD_LAUNCH_CHECK();
}

void launch_wide_tb_inject(const GenModel& g, const BondArgs& a, const float* TP, float* H, float* TH4,
                           cudaStream_t s) {
    if (a.n <= 0) return;
    k_wide_tb_inject<<<wide_conv_grid(a.n), kConvWarps * 32, 0, s>>>(g, a, TP, H, TH4);
    GMD_LAUNCH_CHECK();
}

void launch_wide_tb_bwd_q(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                          const float* HB, const float* TH4, float* QB, cudaStream_t s) {
    if (n <= 0) return;
    launch_node(g, n, nodes, crow, g.W4, const_cast<float*>(HB), TH4, QB, false, s);
}

static int tb_tc_grid(int64_t n) {  // two CTAs per SM (shared memory), one wave
    int64_t gr = (n + kTW - 1) / kTW;
    if (gr > 148 * 2) gr = 148 * 2;
    return (int)(gr > 0 ? gr : 1);
}

void launch_wide_tb_forward(const GenModel& g, const BondArgs& a, const float* TT, float* TP, float* TH3,
                            cudaStream_t s) {
    if (a.n <= 0) return;
    static bool attr = false;
    if (!attr) {
        GMD_CUDA(cudaFuncSetAttribute(k_wide_tb_forward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(TbSmem)));
        attr = true;
    }
    k_wide_tb_forward<<<tb_tc_grid(a.n), kTW * 32, sizeof(TbSmem), s>>>(g, make_basis3(g), a, TT, TP, TH3);
    GMD_LAUNCH_CHECK();
}

void launch_wide_tb_backward(const GenModel& g, const BondArgs& a, const float* QB, const float* TH3,
                             const float* TT, float* SMR, float4* VIN, float4* VOUT, double* vir_part,
                             cudaStream_t s) {
    const int vg = wide_tb_grid(a.n);
    if (a.n <= 0) {
        GMD_CUDA(cudaMemsetAsync(vir_part, 0, sizeof(double) * 9 * vg, s));
        return;
    }
    static bool attr = false;
    if (!attr) {
        GMD_CUDA(cudaFuncSetAttribute(k_wide_tb_back1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(TbSmem)));
        attr = true;
    }
    float* EB = SMR;  // back1 writes E = P3^T m_bar_3 (8 floats per bond) in the scratch rows
    k_wide_tb_back1<<<tb_tc_grid(a.n), kTW * 32, sizeof(TbSmem), s>>>(g, make_basis3(g), a, QB, TH3, EB,
                                                                       VOUT);
    GMD_LAUNCH_CHECK();
    static bool attr2 = false;
    if (!attr2) {
        GMD_CUDA(cudaFuncSetAttribute(k_wide_tb_back2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(Back2Smem)));
        attr2 = true;
    }
    (void)TT;
    k_wide_tb_back2<<<back2_grid(a.n), kB2Warps * 32, sizeof(Back2Smem), s>>>(g, make_basis3(g), a, EB, VIN,
                                                                             VOUT, vir_part);
    GMD_LAUNCH_CHECK();
}

void launch_wide_bwd_edge(const GenModel& g, const ConvArgs& a, const float* MB, const float* Hl,
                          float* HB, double4* GRAD, double* vir_part, cudaStream_t s, bool hbar) {
    const int grid = wide_bwd_grid(a.n);
    if (a.n <= 0) {
        GMD_CUDA(cudaMemsetAsync(vir_part, 0, sizeof(double) * 6 * grid, s));
        return;
    }
    // edges whose neighbour rows are in flight per warp (A/B: GMD_WIDE_BATCH =
    // 8 | 12; 16 spills at the two-CTA register budget)
    static const int batch = [] {
        const char* v = std::getenv("GMD_WIDE_BATCH");
        return v && std::atoi(v) == 12 ? 12 : 8;
    }();
    static bool attr = false;
    if (!attr) {
        GMD_CUDA(cudaFuncSetAttribute(k_wide_bwd_edge<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(BwdSmem) + 1024));
        GMD_CUDA(cudaFuncSetAttribute(k_wide_bwd_edge<12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(BwdSmem) + 1024));
        attr = true;
    }
    const int var = bwd_variant();
    if (var != kBwdTc) {
        const Basis bs = make_basis(g);
        const size_t sm = sizeof(BwdSmSmem);
        static bool attr_sm = false;
        if (!attr_sm) {
            GMD_CUDA(cudaFuncSetAttribute(k_wide_bwd_edge_sm<4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            GMD_CUDA(cudaFuncSetAttribute(k_wide_bwd_edge_sm<4, 3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)sm));
            GMD_CUDA(cudaFuncSetAttribute(k_wide_bwd_edge_sm<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            attr_sm = true;
        }
        if (var == kBwdSm4 && !hbar)
            k_wide_bwd_edge_sm<4, 3, false><<<grid, kFW * 32, sm, s>>>(g, bs, a, MB, Hl, HB, GRAD, vir_part);
        else if (var == kBwdSm4)
            k_wide_bwd_edge_sm<4, 3><<<grid, kFW * 32, sm, s>>>(g, bs, a, MB, Hl, HB, GRAD, vir_part);
        else if (var == kBwdSm8)
            k_wide_bwd_edge_sm<8, 2><<<grid, kFW * 32, sm, s>>>(g, bs, a, MB, Hl, HB, GRAD, vir_part);
        else if (var == kBwdFf16)
            k_wide_bwd_edge_ff<16, 3><<<grid, kFW * 32, 0, s>>>(g, bs, a, MB, Hl, HB, GRAD, vir_part);
        else
            k_wide_bwd_edge_ff<32, 2><<<grid, kFW * 32, 0, s>>>(g, bs, a, MB, Hl, HB, GRAD, vir_part);
        GMD_LAUNCH_CHECK();
        return;
    }
    auto kern = batch == 8 ? k_wide_bwd_edge<8> : k_wide_bwd_edge<12>;
    kern<<<grid, kBW * 32, sizeof(BwdSmem) + 1024, s>>>(g, make_basis(g), a, MB, Hl, HB, GRAD, vir_part);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
