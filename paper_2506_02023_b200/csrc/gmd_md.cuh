// On-device velocity-Verlet MD step kernels (proj/src/md.cpp:55-160).
#pragma once
#include "gmd_common.cuh"

namespace gmd {

// md.hpp:14-21 unit constants (eV / A / fs / amu)
constexpr double kAccel = 9.648533212e-3;  // (eV/A)/amu -> A/fs^2
constexpr double kKinetic = 103.642697;    // amu (A/fs)^2 -> eV
constexpr double kBoltzmann = 8.617333262e-5;

struct Mat9 {
    double m[9];  // row-major 3 x 3
};

void launch_md_kick_drift(int64_t n, double* pos, double* vel, const double* frc, const double* mass,
                          double dt, cudaStream_t s);
void launch_md_wrap(int64_t n, double* pos, const Mat9& L, const Mat9& inv, cudaStream_t s);
void launch_md_kick(int64_t n, double* vel, const double* frc, const double* mass, double dt,
                    unsigned long long* bad, cudaStream_t s);
// kinetic energy (eV) and max |f| into out[0..1] (device); part holds
// 2 * md_observe_parts() doubles
int md_observe_parts();
void launch_md_observe(int64_t n, const double* vel, const double* mass, const double* frc,
                       double* part, double* out, cudaStream_t s);

}  // namespace gmd
