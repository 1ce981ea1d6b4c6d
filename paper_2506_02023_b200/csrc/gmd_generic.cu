// Width-generic model kernels (see gmd_generic.cuh).  Formulas follow the
// tuned kernels and proj/src/potential.cpp:19-78 (radial basis), 743-774
// (conv), 816-848 (backward):
//   u_k(d) = fc(d) exp(-((d - mu_k)/sigma)^2), fc = (cos(pi d/rc) + 1)/2
//   m_u    = sum_{e=(w->u)} (P u(d_e)) * h_w,   h_u' = h_u + tanh(W m_u + b)
//   backward per edge: ds_f = ca A_f + cb B_f (A = P phi, B = (kP) phi),
//   h_bar_u += m_bar_w * fc A, grad_u -= v (dself + drev) / d, virial from dself.
#include "gmd_generic.cuh"

namespace gmd {
namespace {

constexpr int kGenWarps = 8;              // warps per CTA, one node per warp
constexpr int kNJ = kGenMaxF / 32;        // feature slots per lane
constexpr unsigned kFull = 0xffffffffu;
constexpr int kTbCache = 64;  // bond vectors of a center cached per warp

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

// with zs: also each row's species byte and the species presence mask
// (warp OR -> block OR -> one global OR per word), for the F = 64 layer-0
// species-sum kernels
__global__ void k_gen_embed(GenModel g, int64_t rows, const int32_t* __restrict__ node_array,
                            const int32_t* __restrict__ Z, float* __restrict__ H0,
                            uint8_t* __restrict__ zs, unsigned* zmask) {
    __shared__ unsigned smask[4];
    if (threadIdx.x < 4) smask[threadIdx.x] = 0u;
    __syncthreads();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = t < rows * g.F;
    const int64_t r = t / g.F;
    const int f = (int)(t - r * g.F);
    int z = 0;
    if (live) {
        const int id = node_array ? node_array[r] : (int)r;
        z = Z[id];
        H0[t] = g.emb[(size_t)z * g.F + f];
        if (zs && f == 0) zs[r] = (uint8_t)z;
    }
    if (zs) {
        const bool mine = live && f == 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const unsigned v = __reduce_or_sync(0xffffffffu, mine && (z >> 5) == w ? 1u << (z & 31) : 0u);
            if ((threadIdx.x & 31) == 0 && v) atomicOr(&smask[w], v);
        }
        __syncthreads();
        if (threadIdx.x < 4 && smask[threadIdx.x]) atomicOr(zmask + threadIdx.x, smask[threadIdx.x]);
    }
}

__global__ void k_gen_init_hbar(GenModel g, int64_t n, float* __restrict__ HB) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n * g.F) HB[t] = g.ro[t % g.F];
}

// Edges in chunks of 32: lane i evaluates edge i's radial basis into shared
// memory, then the warp (lanes over features) consumes the chunk with
// independent row loads.  Dynamic shared memory: P (F x K) + per-warp
// basis rows [32][K + 1] + the m staging row.
__global__ void __launch_bounds__(kGenWarps * 32) k_gen_conv(GenModel g, ConvArgs a, int layer,
                                                             const float* __restrict__ Hin,
                                                             float* __restrict__ Hout,
                                                             float* __restrict__ TH,
                                                             double* __restrict__ per_atom) {
    extern __shared__ float gsm[];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, K = g.K, nj = (F + 31) / 32, K1 = K + 1;
    float* sP = gsm;                                         // F x K
    float* su = sP + F * K + (size_t)wq * (32 * K1 + 32 + kGenMaxF);  // [32][K1]
    int* sw = reinterpret_cast<int*>(su + 32 * K1);          // [32]
    float* sm = su + 32 * K1 + 32;                           // [kGenMaxF]
    for (int t = threadIdx.x; t < F * K; t += blockDim.x) sP[(t % K) * F + t / K] = g.P[t];  // [k][f]
    __syncthreads();
    const float* WT = g.WT + (size_t)layer * F * F;
    const float* bl = g.b + (size_t)layer * F;
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t r = a.crow ? (int64_t)a.crow[v] : v;
        const int e0 = a.row[v], e1 = a.row[v + 1];
        float m[kNJ] = {0.f, 0.f, 0.f, 0.f};
        for (int eb = e0; eb < e1; eb += 32) {
            const int ne = min(32, e1 - eb);
            if (lane < ne) {
                const float d = a.d[eb + lane];
                sw[lane] = a.lsrc[eb + lane];
                const float fc = d < g.rc ? 0.5f * (cospif(d * g.inv_rc) + 1.0f) : 0.0f;
#pragma unroll 4
                for (int kk = 0; kk < K; ++kk) {
                    const float x = (d - g.mu_step * (float)kk) * g.inv_sigma;
                    su[lane * K1 + kk] = fc * expf(-x * x);
                }
            }
            __syncwarp();
            for (int i = 0; i < ne; ++i) {
                const int w = sw[i];
                const float* ui = su + i * K1;
                for (int jj = 0; jj < nj; ++jj) {
                    const int f = lane + 32 * jj;
                    if (f < F) {
                        float s2 = 0.f;
#pragma unroll 4
                        for (int kk = 0; kk < K; ++kk) s2 = fmaf(sP[kk * F + f], ui[kk], s2);
                        m[jj] = fmaf(Hin[(size_t)w * F + f], s2, m[jj]);
                    }
                }
            }
            __syncwarp();
        }
        for (int jj = 0; jj < nj; ++jj) {
            const int f = lane + 32 * jj;
            if (f < F) sm[f] = m[jj];
        }
        __syncwarp();
        float ev = 0.f;
        for (int jj = 0; jj < nj; ++jj) {
            const int f = lane + 32 * jj;
            if (f < F) {
                float z = bl[f];
#pragma unroll 4
                for (int q = 0; q < F; ++q) z = fmaf(WT[(size_t)q * F + f], sm[q], z);
                const float th = tanhf(z);
                const float hn = Hin[(size_t)r * F + f] + th;
                Hout[(size_t)r * F + f] = hn;
                note_nonfinite(a, layer, r, hn);
                TH[(size_t)k * F + f] = th;
                ev = fmaf(g.ro[f], hn, ev);
            }
        }
        __syncwarp();
        if (per_atom) {
            ev = gwarp_sum(ev);
            if (lane == 0) per_atom[v] = (double)ev;
        }
    }
}

__global__ void __launch_bounds__(kGenWarps * 32) k_gen_bwd_node(GenModel g, int64_t n,
                                                                 const int32_t* __restrict__ nodes,
                                                                 const int32_t* __restrict__ crow,
                                                                 int layer,
                                                                 const float* __restrict__ HB,
                                                                 const float* __restrict__ TH,
                                                                 float* __restrict__ MB) {
    __shared__ float sy[kGenWarps][kGenMaxF];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, nj = (F + 31) / 32;
    const float* W = g.W + (size_t)layer * F * F;
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t v = nodes ? (int64_t)nodes[k] : k;
        const int64_t r = crow ? (int64_t)crow[v] : v;
        for (int j = 0; j < nj; ++j) {
            const int f = lane + 32 * j;
            if (f < F) {
                const float th = TH[(size_t)k * F + f];
                sy[wq][f] = HB[(size_t)k * F + f] * (1.0f - th * th);
            }
        }
        __syncwarp();
        for (int j = 0; j < nj; ++j) {
            const int q = lane + 32 * j;
            if (q < F) {
                float acc = 0.f;
#pragma unroll 4
                for (int f = 0; f < F; ++f) acc = fmaf(W[(size_t)f * F + q], sy[wq][f], acc);
                MB[(size_t)r * F + q] = acc;
            }
        }
        __syncwarp();
    }
}

// Edges in chunks of 32 as in k_gen_conv: lane i evaluates edge i's basis
// terms (phi_k, fc, ca, cb) into shared memory; lanes over features then
// accumulate h_bar and each edge's (dself, drev) partials, which lane i sums
// for its edge (fixed order) before the gradient and virial terms.
__global__ void __launch_bounds__(kGenWarps * 32) k_gen_bwd_edge(GenModel g, ConvArgs a,
                                                                 const float* __restrict__ MB,
                                                                 const float* __restrict__ Hl,
                                                                 float* __restrict__ HB,
                                                                 double4* __restrict__ GRAD,
                                                                 double* __restrict__ vir_part) {
    extern __shared__ float gsm[];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, K = g.K, nj = (F + 31) / 32, K1 = K + 1;
    float* sP = gsm;             // F x K
    float* sPk = sP + F * K;     // F x K
    float* base = sPk + F * K + (size_t)wq * (32 * (K1 + 4) + 2 * 32 * 33);
    float* sph = base;                         // [32][K1] phi
    float* scf = sph + 32 * K1;                // [32][4]: fc, ca, cb, src (as int)
    float* pself = scf + 32 * 4;               // [32 edges][33]
    float* prev = pself + 32 * 33;             // [32 edges][33]
    for (int t = threadIdx.x; t < F * K; t += blockDim.x) {  // [k][f]
        sP[(t % K) * F + t / K] = g.P[t];
        sPk[(t % K) * F + t / K] = g.Pk[t];
    }
    __syncthreads();
    const float isg = g.inv_sigma, mus = g.mu_step;
    double wvir[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t ru = a.crow ? (int64_t)a.crow[v] : v;
        const int e0 = a.row[v], e1 = a.row[v + 1];
        float mu[kNJ], hu[kNJ], hb[kNJ] = {0.f, 0.f, 0.f, 0.f};
        for (int jj = 0; jj < kNJ; ++jj) {
            const int f = lane + 32 * jj;
            mu[jj] = jj < nj && f < F ? MB[(size_t)ru * F + f] : 0.f;
            hu[jj] = jj < nj && f < F ? Hl[(size_t)ru * F + f] : 0.f;
        }
        double gx = 0.0, gy = 0.0, gz = 0.0;
        float vr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int eb = e0; eb < e1; eb += 32) {
            const int ne = min(32, e1 - eb);
            float4 qi = make_float4(0.f, 0.f, 0.f, 1.f);
            if (lane < ne) {
                qi = a.vd[eb + lane];
                const float d = qi.w;
                float sn, cs;
                sincospif(d * g.inv_rc, &sn, &cs);
                const bool in = d < g.rc;
                const float fc = in ? 0.5f * (cs + 1.0f) : 0.0f;
                const float dfc = in ? -0.5f * 3.14159265358979f * g.inv_rc * sn : 0.0f;
                const float x0 = d * isg, step = mus * isg;
                scf[lane * 4 + 0] = fc;
                scf[lane * 4 + 1] = dfc - 2.0f * fc * isg * x0;
                scf[lane * 4 + 2] = 2.0f * fc * isg * step;
                scf[lane * 4 + 3] = __int_as_float(a.lsrc[eb + lane]);
#pragma unroll 4
                for (int kk = 0; kk < K; ++kk) {
                    const float x = (d - mus * (float)kk) * isg;
                    sph[lane * K1 + kk] = expf(-x * x);
                }
            }
            __syncwarp();
            for (int i = 0; i < ne; ++i) {
                const float fc = scf[i * 4], ca = scf[i * 4 + 1], cb = scf[i * 4 + 2];
                const int w = __float_as_int(scf[i * 4 + 3]);
                const float* ph = sph + i * K1;
                float ds_self = 0.f, ds_rev = 0.f;
                for (int jj = 0; jj < nj; ++jj) {
                    const int f = lane + 32 * jj;
                    if (f < F) {
                        float A = 0.f, B = 0.f;
#pragma unroll 4
                        for (int kk = 0; kk < K; ++kk) {
                            A = fmaf(sP[kk * F + f], ph[kk], A);
                            B = fmaf(sPk[kk * F + f], ph[kk], B);
                        }
                        const float mw = MB[(size_t)w * F + f], hw = Hl[(size_t)w * F + f];
                        const float ds = fmaf(ca, A, cb * B);
                        hb[jj] = fmaf(mw, fc * A, hb[jj]);
                        ds_self = fmaf(mu[jj] * hw, ds, ds_self);
                        ds_rev = fmaf(mw * hu[jj], ds, ds_rev);
                    }
                }
                pself[i * 33 + lane] = ds_self;
                prev[i * 33 + lane] = ds_rev;
            }
            __syncwarp();
            if (lane < ne) {  // edge `lane`: its partials over the 32 feature lanes, in order
                float dself = 0.f, drev = 0.f;
                for (int l = 0; l < 32; ++l) {
                    dself += pself[lane * 33 + l];
                    drev += prev[lane * 33 + l];
                }
                const float invd = 1.0f / qi.w;
                const float coef = (dself + drev) * invd;  // swapped terms on the reverse edge
                gx -= (double)(qi.x * coef);
                gy -= (double)(qi.y * coef);
                gz -= (double)(qi.z * coef);
                const float cself = dself * invd;
                vr[0] = fmaf(cself * qi.x, qi.x, vr[0]);
                vr[1] = fmaf(cself * qi.y, qi.y, vr[1]);
                vr[2] = fmaf(cself * qi.z, qi.z, vr[2]);
                vr[3] = fmaf(cself * qi.x, qi.y, vr[3]);
                vr[4] = fmaf(cself * qi.x, qi.z, vr[4]);
                vr[5] = fmaf(cself * qi.y, qi.z, vr[5]);
            }
            __syncwarp();
        }
        for (int jj = 0; jj < nj; ++jj) {  // one writer per element
            const int f = lane + 32 * jj;
            if (f < F) HB[(size_t)k * F + f] += hb[jj];
        }
        gx = gwarp_sumd(gx);
        gy = gwarp_sumd(gy);
        gz = gwarp_sumd(gz);
#pragma unroll
        for (int c = 0; c < 6; ++c) vr[c] = gwarp_sum(vr[c]);
        if (lane == 0) {  // fp64, one writer per node (exact antisymmetric sums, gmd_model.cu)
            double4 gr = GRAD[k];
            gr.x += gx;
            gr.y += gy;
            gr.z += gz;
            GRAD[k] = gr;
#pragma unroll
            for (int c = 0; c < 6; ++c) wvir[c] += (double)vr[c];
        }
    }
    if (lane == 0) {
        const int64_t rec = (int64_t)blockIdx.x * kGenWarps + wq;
#pragma unroll
        for (int c = 0; c < 6; ++c) vir_part[rec * 6 + c] = wvir[c];
    }
}

// ---- three-body ----------------------------------------------------------
// lane k (< K) holds the three-body basis value u3_k(d) (with fc3) or phi_k
__device__ __forceinline__ void gen_fcut3(const GenModel& g, float d, float& fc, float& dfc) {
    float sn, cs;
    sincospif(d * g.inv_r3, &sn, &cs);
    const bool in = d < g.r3;
    fc = in ? 0.5f * (cs + 1.0f) : 0.0f;
    dfc = in ? -0.5f * 3.14159265358979f * g.inv_r3 * sn : 0.0f;
}
// t_f = sum_k P3[f][k] u3_k(d) into out[j] (features lane + 32 j)
__device__ __forceinline__ void gen_bond_t(const GenModel& g, float d, int lane, float out[kNJ]) {
    const int F = g.F, K = g.K, nj = (F + 31) / 32;
    float fc, dfc;
    gen_fcut3(g, d, fc, dfc);
    float u = 0.f;
    if (lane < K) {
        const float x = (d - g.mu_step3 * (float)lane) * g.inv_sigma3;
        u = fc * expf(-x * x);
    }
    for (int j = 0; j < kNJ; ++j) out[j] = 0.f;
#pragma unroll 4
    for (int kk = 0; kk < K; ++kk) {
        const float uk = __shfl_sync(kFull, u, kk);
        for (int j = 0; j < nj; ++j) {
            const int f = lane + 32 * j;
            if (f < F) out[j] = fmaf(g.P3T[kk * F + f], uk, out[j]);
        }
    }
}
// ds_f = sum_k P3[f][k] du3_k(d)
__device__ __forceinline__ void gen_bond_dt(const GenModel& g, float d, int lane, float out[kNJ]) {
    const int F = g.F, K = g.K, nj = (F + 31) / 32;
    float fc, dfc;
    gen_fcut3(g, d, fc, dfc);
    float du = 0.f;
    if (lane < K) {
        const float x = (d - g.mu_step3 * (float)lane) * g.inv_sigma3;
        du = expf(-x * x) * (dfc - 2.0f * fc * x * g.inv_sigma3);
    }
    for (int j = 0; j < kNJ; ++j) out[j] = 0.f;
#pragma unroll 4
    for (int kk = 0; kk < K; ++kk) {
        const float uk = __shfl_sync(kFull, du, kk);
        for (int j = 0; j < nj; ++j) {
            const int f = lane + 32 * j;
            if (f < F) out[j] = fmaf(g.P3T[kk * F + f], uk, out[j]);
        }
    }
}

// TT[b] = t of bond b for the bonds of every center
__global__ void __launch_bounds__(kGenWarps * 32) k_gen_tb_t(GenModel g, BondArgs a,
                                                             float* __restrict__ TT) {
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, nj = (F + 31) / 32;
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t s = a.nodes ? (int64_t)a.nodes[k] : k;
        for (int b = a.brow[s]; b < a.brow[s + 1]; ++b) {
            float t[kNJ];
            gen_bond_t(g, a.vd[a.bedge[b]].w, lane, t);
            for (int j = 0; j < nj; ++j) {
                const int f = lane + 32 * j;
                if (f < F) TT[(size_t)b * F + f] = t[j];
            }
        }
    }
}

// per center s, slot j: m3 = sum_{o != j} c(o, j) t_o (ascending o),
// t' = t_j + fc3(d_j) tanh(W3 m3) -> TP / TH3 slot j
__global__ void __launch_bounds__(kGenWarps * 32) k_gen_tb_forward(GenModel g, BondArgs a,
                                                                   const float* __restrict__ TT,
                                                                   float* __restrict__ TP,
                                                                   float* __restrict__ TH3) {
    __shared__ float sm[kGenWarps][kGenMaxF];
    __shared__ float4 sq[kGenWarps][kTbCache];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, nj = (F + 31) / 32;
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t s = a.nodes ? (int64_t)a.nodes[k] : k;
        const int b0 = a.brow[s], nbd = a.brow[s + 1] - b0;
        for (int o = lane; o < nbd && o < kTbCache; o += 32) sq[wq][o] = a.vd[a.bedge[b0 + o]];
        __syncwarp();
        auto qof = [&](int o) { return o < kTbCache ? sq[wq][o] : a.vd[a.bedge[b0 + o]]; };
        for (int j = 0; j < nbd; ++j) {
            const float4 qj = qof(j);
            float m3[kNJ] = {0.f, 0.f, 0.f, 0.f};
            for (int o = 0; o < nbd; ++o) {
                if (o == j) continue;  // the reverse pair (linegraph.cpp:16-21)
                const float4 q2 = qof(o);
                const float c = (q2.x * qj.x + q2.y * qj.y + q2.z * qj.z) / (q2.w * qj.w);
                for (int jj = 0; jj < nj; ++jj) {
                    const int f = lane + 32 * jj;
                    if (f < F) m3[jj] = fmaf(c, TT[(size_t)(b0 + o) * F + f], m3[jj]);
                }
            }
            for (int jj = 0; jj < nj; ++jj) {
                const int f = lane + 32 * jj;
                if (f < F) sm[wq][f] = m3[jj];
            }
            __syncwarp();
            float fc, dfc;
            gen_fcut3(g, qj.w, fc, dfc);
            for (int jj = 0; jj < nj; ++jj) {
                const int f = lane + 32 * jj;
                if (f < F) {
                    float z = 0.f;
#pragma unroll 4
                    for (int q = 0; q < F; ++q) z = fmaf(g.W3T[(size_t)q * F + f], sm[wq][q], z);
                    const float th = tanhf(z);
                    TP[(size_t)(b0 + j) * F + f] = TT[(size_t)(b0 + j) * F + f] + fc * th;
                    TH3[(size_t)(b0 + j) * F + f] = th;
                }
            }
            __syncwarp();
        }
        __syncwarp();
    }
}

// q_u = sum_{b into u} t'_rev(b) (ascending b), h_u += tanh(W4 q_u)
__global__ void __launch_bounds__(kGenWarps * 32) k_gen_tb_inject(GenModel g, BondArgs a,
                                                                  const float* __restrict__ TP,
                                                                  float* __restrict__ H,
                                                                  float* __restrict__ TH4) {
    __shared__ float sq[kGenWarps][kGenMaxF];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, nj = (F + 31) / 32;
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t u = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t r = a.crow ? (int64_t)a.crow[u] : u;
        float q[kNJ] = {0.f, 0.f, 0.f, 0.f};
        for (int b = a.brow[u]; b < a.brow[u + 1]; ++b) {
            const int rb = a.brev[b];
            for (int jj = 0; jj < nj; ++jj) {
                const int f = lane + 32 * jj;
                if (f < F) q[jj] += TP[(size_t)rb * F + f];
            }
        }
        for (int jj = 0; jj < nj; ++jj) {
            const int f = lane + 32 * jj;
            if (f < F) sq[wq][f] = q[jj];
        }
        __syncwarp();
        for (int jj = 0; jj < nj; ++jj) {
            const int f = lane + 32 * jj;
            if (f < F) {
                float z = 0.f;
#pragma unroll 4
                for (int q2 = 0; q2 < F; ++q2) z = fmaf(g.W4T[(size_t)q2 * F + f], sq[wq][q2], z);
                const float th = tanhf(z);
                H[(size_t)r * F + f] += th;
                TH4[(size_t)k * F + f] = th;
            }
        }
        __syncwarp();
    }
}

// QB[row(v)] = W4^T (HB * (1 - TH4^2))
__global__ void __launch_bounds__(kGenWarps * 32) k_gen_tb_bwd_q(GenModel g, int64_t n,
                                                                 const int32_t* __restrict__ nodes,
                                                                 const int32_t* __restrict__ crow,
                                                                 const float* __restrict__ HB,
                                                                 const float* __restrict__ TH4,
                                                                 float* __restrict__ QB) {
    __shared__ float sy[kGenWarps][kGenMaxF];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, nj = (F + 31) / 32;
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t v = nodes ? (int64_t)nodes[k] : k;
        const int64_t r = crow ? (int64_t)crow[v] : v;
        for (int jj = 0; jj < nj; ++jj) {
            const int f = lane + 32 * jj;
            if (f < F) {
                const float th = TH4[(size_t)k * F + f];
                sy[wq][f] = HB[(size_t)k * F + f] * (1.0f - th * th);
            }
        }
        __syncwarp();
        for (int jj = 0; jj < nj; ++jj) {
            const int q = lane + 32 * jj;
            if (q < F) {
                float acc = 0.f;
#pragma unroll 4
                for (int f = 0; f < F; ++f) acc = fmaf(g.W4[(size_t)f * F + q], sy[wq][f], acc);
                QB[(size_t)r * F + q] = acc;
            }
        }
        __syncwarp();
    }
}

// per center s (the tuned k_tb_backward's adjoint, lanes over features):
// phase 1 per slot j: adjoints of t'(e'_j) -> m_bar_3 (SMR), VOUT (fc3 and
// bond-init paths); phase 2: line-edge cosine gradients -> VIN / VOUT
__global__ void __launch_bounds__(kGenWarps * 32) k_gen_tb_backward(
    GenModel g, BondArgs a, const float* __restrict__ QB, const float* __restrict__ TH3,
    const float* __restrict__ TT, float* __restrict__ SMR, float4* __restrict__ VIN,
    float4* __restrict__ VOUT, double* __restrict__ vir_part) {
    __shared__ float sy[kGenWarps][kGenMaxF];
    __shared__ float4 sq[kGenWarps][kTbCache];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, nj = (F + 31) / 32;
    double vir[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t s = a.nodes ? (int64_t)a.nodes[k] : k;
        const int b0 = a.brow[s], nbd = a.brow[s + 1] - b0;
        __syncwarp();
        for (int o = lane; o < nbd && o < kTbCache; o += 32) sq[wq][o] = a.vd[a.bedge[b0 + o]];
        __syncwarp();
        auto qof = [&](int o) { return o < kTbCache ? sq[wq][o] : a.vd[a.bedge[b0 + o]]; };
        for (int j = 0; j < nbd; ++j) {  // phase 1
            const int e = a.bedge[b0 + j];
            const float4 q = a.vd[e];
            const int x = a.esrc[e];
            const int64_t rx = a.crow ? (int64_t)a.crow[x] : x;
            float fc, dfc, ds[kNJ];
            gen_fcut3(g, q.w, fc, dfc);
            gen_bond_dt(g, q.w, lane, ds);
            float dbf = 0.f, da = 0.f;
            for (int jj = 0; jj < nj; ++jj) {
                const int f = lane + 32 * jj;
                if (f < F) {
                    const float tpb = QB[(size_t)rx * F + f];
                    const float th = TH3[(size_t)(b0 + j) * F + f];
                    dbf = fmaf(tpb * th, dfc, dbf);
                    da = fmaf(tpb, ds[jj], da);
                    sy[wq][f] = tpb * fc * (1.0f - th * th);
                }
            }
            dbf = gwarp_sum(dbf);
            da = gwarp_sum(da);
            __syncwarp();
            for (int jj = 0; jj < nj; ++jj) {
                const int q2 = lane + 32 * jj;
                if (q2 < F) {
                    float acc = 0.f;
#pragma unroll 4
                    for (int f = 0; f < F; ++f) acc = fmaf(g.W3[(size_t)f * F + q2], sy[wq][f], acc);
                    SMR[(size_t)(b0 + j) * F + q2] = acc;
                }
            }
            __syncwarp();
            if (lane == 0) {
                const float c0 = -(dbf + da) / q.w;
                VOUT[b0 + j] = make_float4(q.x * c0, q.y * c0, q.z * c0, 0.f);
            }
        }
        __syncwarp();
        for (int j = 0; j < nbd; ++j) {  // phase 2
            const float4 qj = qof(j);
            const float idj = 1.0f / qj.w;
            float tb[kNJ] = {0.f, 0.f, 0.f, 0.f};
            float vix = 0.f, viy = 0.f, viz = 0.f;
            float4 vo = VOUT[b0 + j];
            for (int o = 0; o < nbd; ++o) {
                if (o == j) continue;
                const float4 qo = qof(o);
                const float ido = 1.0f / qo.w;
                const float c = (qj.x * qo.x + qj.y * qo.y + qj.z * qo.z) * idj * ido;
                float cb = 0.f, cb2 = 0.f;
                for (int jj = 0; jj < nj; ++jj) {
                    const int f = lane + 32 * jj;
                    if (f < F) {
                        const float smo = SMR[(size_t)(b0 + o) * F + f];
                        tb[jj] = fmaf(c, smo, tb[jj]);
                        cb = fmaf(smo, TT[(size_t)(b0 + j) * F + f], cb);
                        cb2 = fmaf(SMR[(size_t)(b0 + j) * F + f], TT[(size_t)(b0 + o) * F + f], cb2);
                    }
                }
                cb = gwarp_sum(cb);
                cb2 = gwarp_sum(cb2);
                // (a) line edge (e_j, e'_o): dc/da = -(b^ + a^ c)/|a|, a = v_j, b = -v_o
                vix += -(-qo.x * ido + qj.x * idj * c) * idj * cb;
                viy += -(-qo.y * ido + qj.y * idj * c) * idj * cb;
                viz += -(-qo.z * ido + qj.z * idj * c) * idj * cb;
                // (b) line edge (e_o, e'_j): dc/db = -(a^ + b^ c)/|b|, a = v_o, b = -v_j
                vo.x += -(qo.x * ido - qj.x * idj * c) * idj * cb2;
                vo.y += -(qo.y * ido - qj.y * idj * c) * idj * cb2;
                vo.z += -(qo.z * ido - qj.z * idj * c) * idj * cb2;
            }
            float dsj[kNJ];
            gen_bond_dt(g, qj.w, lane, dsj);
            float db = 0.f;
            for (int jj = 0; jj < nj; ++jj) db = fmaf(tb[jj], dsj[jj], db);
            db = gwarp_sum(db);
            vix += qj.x * db * idj;
            viy += qj.y * db * idj;
            viz += qj.z * db * idj;
            if (lane == 0) {
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
    if (lane == 0) {
        const int64_t rec = (int64_t)blockIdx.x * kGenWarps + wq;
#pragma unroll
        for (int c = 0; c < 9; ++c) vir_part[rec * 9 + c] = vir[c];
    }
}

}  // namespace

int gen_grid(int64_t n) {
    int64_t g = (n + kGenWarps - 1) / kGenWarps;
    if (g > 148 * 8) g = 148 * 8;
    return (int)(g > 0 ? g : 1);
}

void launch_gen_embed(const GenModel& g, int64_t rows, const int32_t* node_array, const int32_t* Z,
                      float* H0, cudaStream_t s, uint8_t* zs, unsigned* zmask) {
    if (rows == 0) return;
    if (zs) GMD_CUDA(cudaMemsetAsync(zmask, 0, 4 * sizeof(unsigned), s));
    k_gen_embed<<<div_up(rows * g.F, 256), 256, 0, s>>>(g, rows, node_array, Z, H0, zs, zmask);
    GMD_LAUNCH_CHECK();
}

void launch_gen_conv(const GenModel& g, const ConvArgs& a, int layer, const float* Hin, float* Hout,
                     float* TH, double* per_atom, cudaStream_t s) {
    if (a.n == 0) return;
    const int K1 = g.K + 1;
    const size_t smem = sizeof(float) * ((size_t)g.F * g.K + kGenWarps * (32 * K1 + 32 + kGenMaxF));
    GMD_CUDA(cudaFuncSetAttribute(k_gen_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_gen_conv<<<gen_grid(a.n), kGenWarps * 32, smem, s>>>(g, a, layer, Hin, Hout, TH, per_atom);
    GMD_LAUNCH_CHECK();
}

void launch_gen_init_hbar(const GenModel& g, int64_t n, float* HB, cudaStream_t s) {
    if (n == 0) return;
    k_gen_init_hbar<<<div_up(n * g.F, 256), 256, 0, s>>>(g, n, HB);
    GMD_LAUNCH_CHECK();
}

void launch_gen_bwd_node(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                         int layer, const float* HB, const float* TH, float* MB, cudaStream_t s) {
    if (n == 0) return;
    k_gen_bwd_node<<<gen_grid(n), kGenWarps * 32, 0, s>>>(g, n, nodes, crow, layer, HB, TH, MB);
    GMD_LAUNCH_CHECK();
}

void launch_gen_bwd_edge(const GenModel& g, const ConvArgs& a, const float* MB, const float* Hl,
                         float* HB, double4* GRAD, double* vir_part, cudaStream_t s) {
    if (a.n == 0) return;
    const int K1 = g.K + 1;
    const size_t smem =
        sizeof(float) * (2 * (size_t)g.F * g.K + kGenWarps * (32 * (K1 + 4) + 2 * 32 * 33));
    GMD_CUDA(cudaFuncSetAttribute(k_gen_bwd_edge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    k_gen_bwd_edge<<<gen_grid(a.n), kGenWarps * 32, smem, s>>>(g, a, MB, Hl, HB, GRAD, vir_part);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd

namespace gmd {

void launch_gen_tb_t(const GenModel& g, const BondArgs& a, int64_t, float* TT, cudaStream_t s) {
    if (a.n == 0) return;
    k_gen_tb_t<<<gen_grid(a.n), kGenWarps * 32, 0, s>>>(g, a, TT);
    GMD_LAUNCH_CHECK();
}

void launch_gen_tb_forward(const GenModel& g, const BondArgs& a, const float* TT, float* TP,
                           float* TH3, int32_t*, cudaStream_t s) {
    if (a.n == 0) return;
    k_gen_tb_forward<<<gen_grid(a.n), kGenWarps * 32, 0, s>>>(g, a, TT, TP, TH3);
    GMD_LAUNCH_CHECK();
}

void launch_gen_tb_inject(const GenModel& g, const BondArgs& a, const float* TP, float* H, float* TH4,
                          cudaStream_t s) {
    if (a.n == 0) return;
    k_gen_tb_inject<<<gen_grid(a.n), kGenWarps * 32, 0, s>>>(g, a, TP, H, TH4);
    GMD_LAUNCH_CHECK();
}

void launch_gen_tb_bwd_q(const GenModel& g, int64_t n, const int32_t* nodes, const int32_t* crow,
                         const float* HB, const float* TH4, float* QB, cudaStream_t s) {
    if (n == 0) return;
    k_gen_tb_bwd_q<<<gen_grid(n), kGenWarps * 32, 0, s>>>(g, n, nodes, crow, HB, TH4, QB);
    GMD_LAUNCH_CHECK();
}

void launch_gen_tb_backward(const GenModel& g, const BondArgs& a, const float* QB, const float* TH3,
                            const float* TT, float* SMR, float4* VIN, float4* VOUT, double* vir_part,
                            cudaStream_t s) {
    if (a.n == 0) return;
    k_gen_tb_backward<<<gen_grid(a.n), kGenWarps * 32, 0, s>>>(g, a, QB, TH3, TT, SMR, VIN, VOUT,
                                                               vir_part);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
