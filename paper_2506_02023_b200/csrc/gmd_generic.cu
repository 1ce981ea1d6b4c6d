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

__device__ __forceinline__ float gwarp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__global__ void k_gen_embed(GenModel g, int64_t rows, const int32_t* __restrict__ node_array,
                            const int32_t* __restrict__ Z, float* __restrict__ H0) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * g.F) return;
    const int64_t r = t / g.F;
    const int f = (int)(t - r * g.F);
    const int id = node_array ? node_array[r] : (int)r;
    H0[t] = g.emb[(size_t)Z[id] * g.F + f];
}

__global__ void k_gen_init_hbar(GenModel g, int64_t n, float* __restrict__ HB) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n * g.F) HB[t] = g.ro[t % g.F];
}

__global__ void __launch_bounds__(kGenWarps * 32) k_gen_conv(GenModel g, ConvArgs a, int layer,
                                                             const float* __restrict__ Hin,
                                                             float* __restrict__ Hout,
                                                             float* __restrict__ TH,
                                                             double* __restrict__ per_atom) {
    __shared__ float sm[kGenWarps][kGenMaxF];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, K = g.K, nj = (F + 31) / 32;
    const float* W = g.W + (size_t)layer * F * F;
    const float* bl = g.b + (size_t)layer * F;
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t r = a.crow ? (int64_t)a.crow[v] : v;
        float m[kNJ] = {0.f, 0.f, 0.f, 0.f};
        for (int e = a.row[v]; e < a.row[v + 1]; ++e) {
            const float d = a.d[e];
            const int w = a.lsrc[e];
            const float fc = d < g.rc ? 0.5f * (cospif(d * g.inv_rc) + 1.0f) : 0.0f;
            float u = 0.f;
            if (lane < K) {
                const float x = (d - g.mu_step * (float)lane) * g.inv_sigma;
                u = fc * expf(-x * x);
            }
            float s[kNJ] = {0.f, 0.f, 0.f, 0.f};
            for (int kk = 0; kk < K; ++kk) {
                const float uk = __shfl_sync(kFull, u, kk);
                for (int j = 0; j < nj; ++j) {
                    const int f = lane + 32 * j;
                    if (f < F) s[j] = fmaf(g.P[f * K + kk], uk, s[j]);
                }
            }
            for (int j = 0; j < nj; ++j) {
                const int f = lane + 32 * j;
                if (f < F) m[j] = fmaf(Hin[(size_t)w * F + f], s[j], m[j]);
            }
        }
        for (int j = 0; j < nj; ++j) {
            const int f = lane + 32 * j;
            if (f < F) sm[wq][f] = m[j];
        }
        __syncwarp();
        float ev = 0.f;
        for (int j = 0; j < nj; ++j) {
            const int f = lane + 32 * j;
            if (f < F) {
                float z = bl[f];
                for (int q = 0; q < F; ++q) z = fmaf(W[(size_t)f * F + q], sm[wq][q], z);
                const float th = tanhf(z);
                const float hn = Hin[(size_t)r * F + f] + th;
                Hout[(size_t)r * F + f] = hn;
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
                for (int f = 0; f < F; ++f) acc = fmaf(W[(size_t)f * F + q], sy[wq][f], acc);
                MB[(size_t)r * F + q] = acc;
            }
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kGenWarps * 32) k_gen_bwd_edge(GenModel g, ConvArgs a,
                                                                 const float* __restrict__ MB,
                                                                 const float* __restrict__ Hl,
                                                                 float* __restrict__ HB,
                                                                 float4* __restrict__ GRAD,
                                                                 double* __restrict__ vir_part) {
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int F = g.F, K = g.K, nj = (F + 31) / 32;
    const float isg = g.inv_sigma, mus = g.mu_step;
    double wvir[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t k = (int64_t)blockIdx.x * kGenWarps + wq; k < a.n;
         k += (int64_t)gridDim.x * kGenWarps) {
        const int64_t v = a.nodes ? (int64_t)a.nodes[k] : k;
        const int64_t ru = a.crow ? (int64_t)a.crow[v] : v;
        float mu[kNJ], hu[kNJ], hb[kNJ] = {0.f, 0.f, 0.f, 0.f};
        for (int j = 0; j < kNJ; ++j) {
            const int f = lane + 32 * j;
            mu[j] = j < nj && f < F ? MB[(size_t)ru * F + f] : 0.f;
            hu[j] = j < nj && f < F ? Hl[(size_t)ru * F + f] : 0.f;
        }
        float gx = 0.f, gy = 0.f, gz = 0.f;
        float vr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int e = a.row[v]; e < a.row[v + 1]; ++e) {
            const float4 q = a.vd[e];
            const int w = a.lsrc[e];
            const float d = q.w;
            float sn, cs;
            sincospif(d * g.inv_rc, &sn, &cs);
            const bool in = d < g.rc;
            const float fc = in ? 0.5f * (cs + 1.0f) : 0.0f;
            const float dfc = in ? -0.5f * 3.14159265358979f * g.inv_rc * sn : 0.0f;
            float ph = 0.f;
            if (lane < K) {
                const float x = (d - mus * (float)lane) * isg;
                ph = expf(-x * x);
            }
            const float x0 = d * isg, step = mus * isg;
            const float ca = dfc - 2.0f * fc * isg * x0, cb = 2.0f * fc * isg * step;
            float A[kNJ] = {0.f, 0.f, 0.f, 0.f}, B[kNJ] = {0.f, 0.f, 0.f, 0.f};
            for (int kk = 0; kk < K; ++kk) {
                const float pk = __shfl_sync(kFull, ph, kk);
                for (int j = 0; j < nj; ++j) {
                    const int f = lane + 32 * j;
                    if (f < F) {
                        A[j] = fmaf(g.P[f * K + kk], pk, A[j]);
                        B[j] = fmaf(g.Pk[f * K + kk], pk, B[j]);
                    }
                }
            }
            float dself = 0.f, drev = 0.f;
            for (int j = 0; j < nj; ++j) {
                const int f = lane + 32 * j;
                if (f < F) {
                    const float mw = MB[(size_t)w * F + f], hw = Hl[(size_t)w * F + f];
                    const float ds = fmaf(ca, A[j], cb * B[j]);
                    hb[j] = fmaf(mw, fc * A[j], hb[j]);
                    dself = fmaf(mu[j] * hw, ds, dself);
                    drev = fmaf(mw * hu[j], ds, drev);
                }
            }
            dself = gwarp_sum(dself);
            drev = gwarp_sum(drev);
            const float invd = 1.0f / d;
            const float coef = (dself + drev) * invd;
            gx -= q.x * coef;
            gy -= q.y * coef;
            gz -= q.z * coef;
            const float cself = dself * invd;
            vr[0] = fmaf(cself * q.x, q.x, vr[0]);
            vr[1] = fmaf(cself * q.y, q.y, vr[1]);
            vr[2] = fmaf(cself * q.z, q.z, vr[2]);
            vr[3] = fmaf(cself * q.x, q.y, vr[3]);
            vr[4] = fmaf(cself * q.x, q.z, vr[4]);
            vr[5] = fmaf(cself * q.y, q.z, vr[5]);
        }
        for (int j = 0; j < nj; ++j) {  // one writer per element
            const int f = lane + 32 * j;
            if (f < F) HB[(size_t)k * F + f] += hb[j];
        }
        if (lane == 0) {
            float4 gr = GRAD[k];
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

}  // namespace

int gen_grid(int64_t n) {
    int64_t g = (n + kGenWarps - 1) / kGenWarps;
    if (g > 148 * 8) g = 148 * 8;
    return (int)(g > 0 ? g : 1);
}

void launch_gen_embed(const GenModel& g, int64_t rows, const int32_t* node_array, const int32_t* Z,
                      float* H0, cudaStream_t s) {
    if (rows == 0) return;
    k_gen_embed<<<div_up(rows * g.F, 256), 256, 0, s>>>(g, rows, node_array, Z, H0);
    GMD_LAUNCH_CHECK();
}

void launch_gen_conv(const GenModel& g, const ConvArgs& a, int layer, const float* Hin, float* Hout,
                     float* TH, double* per_atom, cudaStream_t s) {
    if (a.n == 0) return;
    k_gen_conv<<<gen_grid(a.n), kGenWarps * 32, 0, s>>>(g, a, layer, Hin, Hout, TH, per_atom);
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
                         float* HB, float4* GRAD, double* vir_part, cudaStream_t s) {
    if (a.n == 0) return;
    k_gen_bwd_edge<<<gen_grid(a.n), kGenWarps * 32, 0, s>>>(g, a, MB, Hl, HB, GRAD, vir_part);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
