// Host-side Störmer-Verlet update for the host-resident drop-in path
// (HostForceCalculator driving the reference loop on host arrays).
//
// Same split and the same rounding as the device kernels and the reference's
// numpy sequence (integrator.py:31-44, :47-51, :98-128): built with
// -ffp-contract=off, so no multiply-add is fused.  OpenMP over particles.
#include <math.h>
#include <stdint.h>

#include "../../include/mdg.h"

namespace {

inline size_t idx(int layout, int64_t i, int k, int64_t n) {
    return layout == MDG_AOS ? (size_t)(3 * i + k) : (size_t)(k * n + i);
}

// np.mod(x, L): fmod with sign fix, +0.0 for exact zeros (integrator.py:118).
// Inside [-L, 2L] (every non-blow-up coordinate) the result needs no fmod:
// [0, L) -> x (+0.0 for -0.0); [L, 2L] -> x - L, exact by Sterbenz (2L -> 0);
// [-L, 0) -> x + L, the same rounded addition numpy's sign fix performs.
inline double np_mod(double x, double L) {
    if (x >= 0.0 && x < L) return x + 0.0;
    if (x >= L && x <= 2.0 * L) return x == 2.0 * L ? 0.0 : x - L;
    if (x >= -L && x < 0.0) return x + L;
    double r = fmod(x, L);
    if (r != 0.0) {
        if ((r < 0.0) != (L < 0.0)) r += L;
    } else {
        r = 0.0;
    }
    return r;
}

}  // namespace

extern "C" {

int mdg_host_drift_wrap_range(int64_t n, int64_t begin, int64_t end, int layout, double* pos,
                              double* vel, const double* force, double* old_force,
                              const int32_t* type_id, const double* mass, const double domain[3],
                              const int periodic[3], double dt, int* blowup) {
    if (n < 0 || begin < 0 || end > n || begin > end || (layout != MDG_AOS && layout != MDG_SOA))
        return MDG_EINVAL;
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t i = begin; i < end; ++i) {
        double m = mass[type_id ? type_id[i] : 0];
        double c = 0.5 * dt * dt / m;
        for (int k = 0; k < 3; ++k) {
            size_t a = idx(layout, i, k, n);
            double f = force[a];
            double x = pos[a] + vel[a] * dt;
            x = x + f * c;
            double L = domain[k];
            if (!(x >= -L && x <= 2.0 * L)) bad = 1;
            if (periodic[k]) {
                x = np_mod(x, L);
            } else if (x < 0.0) {
                x = -x;
                vel[a] = -vel[a];
            } else if (x > L) {
                x = 2.0 * L - x;
                vel[a] = -vel[a];
            }
            pos[a] = x;
            old_force[a] = f;
        }
    }
    if (blowup) *blowup = bad;
    return MDG_OK;
}

int mdg_host_drift_wrap(int64_t n, int layout, double* pos, double* vel, const double* force,
                        double* old_force, const int32_t* type_id, const double* mass,
                        const double domain[3], const int periodic[3], double dt, int* blowup) {
    return mdg_host_drift_wrap_range(n, 0, n, layout, pos, vel, force, old_force, type_id, mass,
                                     domain, periodic, dt, blowup);
}

int mdg_host_finish_kick_range(int64_t n, int64_t begin, int64_t end, int layout, double* vel,
                               double* force, const double* old_force, const int32_t* type_id,
                               const double* mass, double dt, int has_gravity, double gravity) {
    if (n < 0 || begin < 0 || end > n || begin > end || (layout != MDG_AOS && layout != MDG_SOA))
        return MDG_EINVAL;
#pragma omp parallel for schedule(static)
    for (int64_t i = begin; i < end; ++i) {
        double m = mass[type_id ? type_id[i] : 0];
        if (has_gravity) {
            size_t a = idx(layout, i, 2, n);
            force[a] = force[a] + m * gravity;
        }
        double c = 0.5 * dt / m;
        for (int k = 0; k < 3; ++k) {
            size_t a = idx(layout, i, k, n);
            vel[a] = vel[a] + (force[a] + old_force[a]) * c;
        }
    }
    return MDG_OK;
}

int mdg_host_finish_kick(int64_t n, int layout, double* vel, double* force, const double* old_force,
                         const int32_t* type_id, const double* mass, double dt, int has_gravity,
                         double gravity) {
    return mdg_host_finish_kick_range(n, 0, n, layout, vel, force, old_force, type_id, mass, dt,
                                      has_gravity, gravity);
}

}  // extern "C"
