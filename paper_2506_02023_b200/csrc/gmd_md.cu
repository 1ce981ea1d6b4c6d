// On-device velocity-Verlet MD (proj/src/md.cpp:55-160): the caller of the
// hot path.  Positions, velocities, forces and masses stay in HBM across
// steps; each step is kick+drift -> wrap_positions -> graph rebuild + forward
// (gmd_build / gmd_forward on device buffers) -> kick.  The fp64 update
// expressions follow md.cpp:94-108 in operand order (unfused, like the
// reference's x86-64 build); observables use fixed-order reductions.
#include "gmd_md.cuh"

namespace gmd {
namespace {

constexpr int kThreads = 256;
constexpr int kObsGrid = 148 * 4;  // fixed grid -> deterministic reductions

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// a = f * (kAccel / m); v += a * (0.5 dt); x += v * dt   (md.cpp:94-98)
__global__ void k_kick_drift(int64_t n, double* __restrict__ pos, double* __restrict__ vel,
                             const double* __restrict__ frc, const double* __restrict__ mass,
                             double dt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double s = kAccel / mass[i], h = 0.5 * dt;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double v = dadd(vel[3 * i + k], dmul(dmul(frc[3 * i + k], s), h));
        vel[3 * i + k] = v;
        pos[3 * i + k] = dadd(pos[3 * i + k], dmul(v, dt));
    }
}

// wrap_positions (system.cpp:216-229): f = r L^-1, f -= floor(f) (>= 1 -> 0),
// r = f L, rows evaluated as (a*x + b*y) + c*z
__global__ void k_wrap_positions(int64_t n, double* __restrict__ pos, Mat9 L, Mat9 inv) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
    double f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double v = dadd(dadd(dmul(inv.m[k], x), dmul(inv.m[3 + k], y)), dmul(inv.m[6 + k], z));
        v = __dsub_rn(v, floor(v));
        f[k] = v >= 1.0 ? 0.0 : v;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
        pos[3 * i + k] =
            dadd(dadd(dmul(L.m[k], f[0]), dmul(L.m[3 + k], f[1])), dmul(L.m[6 + k], f[2]));
}

// second half-kick with the non-finite check of md.cpp:100-106 (first
// offending atom = minimum index, independent of scheduling)
__global__ void k_kick(int64_t n, double* __restrict__ vel, const double* __restrict__ frc,
                       const double* __restrict__ mass, double dt,
                       unsigned long long* __restrict__ bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double f0 = frc[3 * i], f1 = frc[3 * i + 1], f2 = frc[3 * i + 2];
    if (!isfinite(f0) || !isfinite(f1) || !isfinite(f2)) atomicMin(bad, (unsigned long long)i);
    const double s = kAccel / mass[i], h = 0.5 * dt;
    const double f[3] = {f0, f1, f2};
#pragma unroll
    for (int k = 0; k < 3; ++k) vel[3 * i + k] = dadd(vel[3 * i + k], dmul(dmul(f[k], s), h));
}

// per-CTA partials of sum 0.5 m |v|^2 and max |f| (MDState::kinetic_energy,
// MDStepRecord::max_force, md.cpp:11-16, :128-130)
__global__ void k_observe(int64_t n, const double* __restrict__ vel,
                          const double* __restrict__ mass, const double* __restrict__ frc,
                          double* __restrict__ part) {
    __shared__ double sk[kThreads], sf[kThreads];
    double ke = 0.0, fm = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double vx = vel[3 * i], vy = vel[3 * i + 1], vz = vel[3 * i + 2];
        const double v2 = dadd(dadd(dmul(vx, vx), dmul(vy, vy)), dmul(vz, vz));
        ke = dadd(ke, dmul(dmul(0.5, mass[i]), v2));
        if (frc) {
            const double fx = frc[3 * i], fy = frc[3 * i + 1], fz = frc[3 * i + 2];
            const double f = __dsqrt_rn(dadd(dadd(dmul(fx, fx), dmul(fy, fy)), dmul(fz, fz)));
            fm = f > fm ? f : fm;
        }
    }
    sk[threadIdx.x] = ke;
    sf[threadIdx.x] = fm;
    __syncthreads();
    for (int o = kThreads / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sk[threadIdx.x] = dadd(sk[threadIdx.x], sk[threadIdx.x + o]);
            sf[threadIdx.x] = sf[threadIdx.x] > sf[threadIdx.x + o] ? sf[threadIdx.x] : sf[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = sk[0];
        part[2 * blockIdx.x + 1] = sf[0];
    }
}

__global__ void k_observe_final(int nparts, const double* __restrict__ part, double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double ke = 0.0, fm = 0.0;
    for (int b = 0; b < nparts; ++b) {
        ke = dadd(ke, part[2 * b]);
        fm = part[2 * b + 1] > fm ? part[2 * b + 1] : fm;
    }
    out[0] = dmul(ke, kKinetic);
    out[1] = fm;
}

int blocks(int64_t n) { return (int)((n + kThreads - 1) / kThreads); }

}  // namespace

void launch_md_kick_drift(int64_t n, double* pos, double* vel, const double* frc, const double* mass,
                          double dt, cudaStream_t s) {
    if (n == 0) return;
    k_kick_drift<<<blocks(n), kThreads, 0, s>>>(n, pos, vel, frc, mass, dt);
    GMD_LAUNCH_CHECK();
}

void launch_md_wrap(int64_t n, double* pos, const Mat9& L, const Mat9& inv, cudaStream_t s) {
    if (n == 0) return;
    k_wrap_positions<<<blocks(n), kThreads, 0, s>>>(n, pos, L, inv);
    GMD_LAUNCH_CHECK();
}

void launch_md_kick(int64_t n, double* vel, const double* frc, const double* mass, double dt,
                    unsigned long long* bad, cudaStream_t s) {
    if (n == 0) return;
    k_kick<<<blocks(n), kThreads, 0, s>>>(n, vel, frc, mass, dt, bad);
    GMD_LAUNCH_CHECK();
}

int md_observe_parts() { return kObsGrid; }

void launch_md_observe(int64_t n, const double* vel, const double* mass, const double* frc,
                       double* part, double* out, cudaStream_t s) {
    k_observe<<<kObsGrid, kThreads, 0, s>>>(n, vel, mass, frc, part);
    GMD_LAUNCH_CHECK();
    k_observe_final<<<1, 32, 0, s>>>(kObsGrid, part, out);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
