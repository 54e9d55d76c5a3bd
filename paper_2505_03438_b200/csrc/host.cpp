// Host-side Störmer-Verlet update for the host-resident drop-in path
// (HostForceCalculator / mdg_host_step driving the reference loop on host
// arrays).
//
// Same split and the same rounding as the device kernels and the reference's
// numpy sequence (integrator.py:31-44, :47-51, :98-128): built with
// -ffp-contract=off, so no multiply-add is fused, and every element sees the
// reference's operations in the reference's order.  The loops are specialised
// per layout (SoA: one contiguous stream per component) and branch-free, so
// they vectorise; OpenMP over particles.
#include <math.h>
#include <stdint.h>

#include "../../include/mdg.h"

namespace {

// np.mod(x, L): fmod with sign fix, +0.0 for exact zeros (integrator.py:118),
// for x in [-L, 2L] (every non-blow-up coordinate; blow-ups are reported and
// the caller raises): [0, L) -> x (+0.0 for -0.0); [L, 2L] -> x - L, exact by
// Sterbenz (2L -> 0); [-L, 0) -> x + L, the rounded addition numpy's sign fix
// performs.  Selects only, so the loops vectorise.
inline double np_mod_in_range(double x, double L) {
    double r = x + 0.0;
    double up = (x == 2.0 * L) ? 0.0 : x - L;
    r = (x >= L) ? up : r;
    r = (x < 0.0) ? x + L : r;
    return r;
}

// fmod-based np.mod for any x (the scalar fallback path)
inline double np_mod(double x, double L) {
    if (x >= -L && x <= 2.0 * L) return np_mod_in_range(x, L);
    double r = fmod(x, L);
    if (r != 0.0) {
        if ((r < 0.0) != (L < 0.0)) r += L;
    } else {
        r = 0.0;
    }
    return r;
}

// one coordinate of the drift: x += v dt; x += f c (c = 0.5 dt^2 / m); wrap
// or reflect (v flips); returns the blow-up bit
inline int drift_coord(double& x, double& v, double f, double c, double L, bool per, double dt) {
    double y = x + v * dt;
    y = y + f * c;
    int bad = !(y >= -L && y <= 2.0 * L);
    bool lo = y < 0.0, hi = y > L;
    double refl = lo ? -y : (hi ? 2.0 * L - y : y);
    double vr = (lo || hi) ? -v : v;
    x = per ? np_mod_in_range(y, L) : refl;
    v = per ? v : vr;
    return bad;
}

// all axes periodic (the common case): velocities are only read
// COPY: F -> F_old here; otherwise the caller swapped the two buffers and
// the current forces are read from old_force (no copy, no write)
template <int LAYOUT, bool TYPED, bool COPY>
int drift_periodic(int64_t n, int64_t a, int64_t b, double* __restrict__ pos,
                   const double* __restrict__ vel, const double* __restrict__ force,
                   double* __restrict__ old_force, const int32_t* __restrict__ tid,
                   const double* __restrict__ mass, const double domain[3], double dt) {
    const double* __restrict__ fsrc = COPY ? force : old_force;
    const double c1 = TYPED ? 0.0 : 0.5 * dt * dt / mass[0];
    const double L0 = domain[0], L1 = domain[1], L2 = domain[2];
    int bad = 0;
#pragma omp parallel for simd schedule(static) reduction(| : bad)
    for (int64_t i = a; i < b; ++i) {
        double c = TYPED ? 0.5 * dt * dt / mass[tid[i]] : c1;
        size_t e0 = LAYOUT == MDG_AOS ? 3 * i : i;
        size_t e1 = LAYOUT == MDG_AOS ? 3 * i + 1 : n + i;
        size_t e2 = LAYOUT == MDG_AOS ? 3 * i + 2 : 2 * n + i;
        double f0 = fsrc[e0], f1 = fsrc[e1], f2 = fsrc[e2];
        double y0 = pos[e0] + vel[e0] * dt, y1 = pos[e1] + vel[e1] * dt, y2 = pos[e2] + vel[e2] * dt;
        y0 = y0 + f0 * c;
        y1 = y1 + f1 * c;
        y2 = y2 + f2 * c;
        bad |= !(y0 >= -L0 && y0 <= 2.0 * L0) | !(y1 >= -L1 && y1 <= 2.0 * L1) |
               !(y2 >= -L2 && y2 <= 2.0 * L2);
        pos[e0] = np_mod_in_range(y0, L0);
        pos[e1] = np_mod_in_range(y1, L1);
        pos[e2] = np_mod_in_range(y2, L2);
        if (COPY) {
            old_force[e0] = f0;
            old_force[e1] = f1;
            old_force[e2] = f2;
        }
    }
    return bad;
}

template <int LAYOUT, bool TYPED>
int drift_all(int64_t n, int64_t a, int64_t b, double* __restrict__ pos, double* __restrict__ vel,
              const double* __restrict__ force, double* __restrict__ old_force,
              const int32_t* __restrict__ tid, const double* __restrict__ mass,
              const double domain[3], const int periodic[3], double dt, bool swapped) {
    if (periodic[0] && periodic[1] && periodic[2]) {
        if (swapped)
            return drift_periodic<LAYOUT, TYPED, false>(n, a, b, pos, vel, force, old_force, tid, mass, domain, dt);
        return drift_periodic<LAYOUT, TYPED, true>(n, a, b, pos, vel, force, old_force, tid, mass, domain, dt);
    }
    if (swapped) force = old_force;   // read the current forces; the copy below is then a no-op
    const double c1 = TYPED ? 0.0 : 0.5 * dt * dt / mass[0];
    const double L0 = domain[0], L1 = domain[1], L2 = domain[2];
    const bool p0 = periodic[0], p1 = periodic[1], p2 = periodic[2];
    int bad = 0;
#pragma omp parallel for simd schedule(static) reduction(| : bad)
    for (int64_t i = a; i < b; ++i) {
        double c = TYPED ? 0.5 * dt * dt / mass[tid[i]] : c1;
        // AoS: component k at 3 i + k; SoA: at k n + i
        size_t e0 = LAYOUT == MDG_AOS ? 3 * i : i;
        size_t e1 = LAYOUT == MDG_AOS ? 3 * i + 1 : n + i;
        size_t e2 = LAYOUT == MDG_AOS ? 3 * i + 2 : 2 * n + i;
        double f0 = force[e0], f1 = force[e1], f2 = force[e2];
        double x0 = pos[e0], x1 = pos[e1], x2 = pos[e2];
        double v0 = vel[e0], v1 = vel[e1], v2 = vel[e2];
        bad |= drift_coord(x0, v0, f0, c, L0, p0, dt);
        bad |= drift_coord(x1, v1, f1, c, L1, p1, dt);
        bad |= drift_coord(x2, v2, f2, c, L2, p2, dt);
        pos[e0] = x0; pos[e1] = x1; pos[e2] = x2;
        vel[e0] = v0; vel[e1] = v1; vel[e2] = v2;
        old_force[e0] = f0; old_force[e1] = f1; old_force[e2] = f2;
    }
    return bad;
}

template <int LAYOUT, bool TYPED>
void kick_all(int64_t n, int64_t a, int64_t b, double* __restrict__ vel, double* __restrict__ force,
              const double* __restrict__ old_force, const int32_t* __restrict__ tid,
              const double* __restrict__ mass, double dt, int has_gravity, double gravity) {
    const double c1 = TYPED ? 0.0 : 0.5 * dt / mass[0];
    const double mg1 = TYPED ? 0.0 : mass[0] * gravity;
    const bool grav = has_gravity != 0;
#pragma omp parallel for simd schedule(static)
    for (int64_t i = a; i < b; ++i) {
        double m = TYPED ? mass[tid[i]] : 0.0;
        size_t e0 = LAYOUT == MDG_AOS ? 3 * i : i;
        size_t e1 = LAYOUT == MDG_AOS ? 3 * i + 1 : n + i;
        size_t e2 = LAYOUT == MDG_AOS ? 3 * i + 2 : 2 * n + i;
        double f2 = force[e2];
        if (grav) {   // apply_gravity (integrator.py:47-51) before the kick
            f2 = f2 + (TYPED ? m * gravity : mg1);
            force[e2] = f2;
        }
        double c = TYPED ? 0.5 * dt / m : c1;
        vel[e0] = vel[e0] + (force[e0] + old_force[e0]) * c;
        vel[e1] = vel[e1] + (force[e1] + old_force[e1]) * c;
        vel[e2] = vel[e2] + (f2 + old_force[e2]) * c;
    }
}

// kick of step s fused with the drift of step s+1 over [a, b), all axes
// periodic: per element exactly kick_all's then drift_periodic's operations
// (gravity into fnew.z first, v += (fnew + fold) c_k, x += v dt, x += fnew c_d,
// np.mod), one pass instead of two.  The drift reads fnew without copying it
// to fold (the caller alternates the two buffers, MDG_HOST_STEP_SWAPPED).
template <int LAYOUT, bool TYPED>
int kick_drift_periodic(int64_t n, int64_t a, int64_t b, double* __restrict__ pos,
                        double* __restrict__ vel, double* __restrict__ fnew,
                        const double* __restrict__ fold, const int32_t* __restrict__ tid,
                        const double* __restrict__ mass, const double domain[3], double dt,
                        int has_gravity, double gravity) {
    const double ck1 = TYPED ? 0.0 : 0.5 * dt / mass[0];
    const double cd1 = TYPED ? 0.0 : 0.5 * dt * dt / mass[0];
    const double mg1 = TYPED ? 0.0 : mass[0] * gravity;
    const bool grav = has_gravity != 0;
    const double L0 = domain[0], L1 = domain[1], L2 = domain[2];
    int bad = 0;
#pragma omp parallel for simd schedule(static) reduction(| : bad)
    for (int64_t i = a; i < b; ++i) {
        double m = TYPED ? mass[tid[i]] : 0.0;
        size_t e0 = LAYOUT == MDG_AOS ? 3 * i : i;
        size_t e1 = LAYOUT == MDG_AOS ? 3 * i + 1 : n + i;
        size_t e2 = LAYOUT == MDG_AOS ? 3 * i + 2 : 2 * n + i;
        double f0 = fnew[e0], f1 = fnew[e1], f2 = fnew[e2];
        if (grav) {
            f2 = f2 + (TYPED ? m * gravity : mg1);
            fnew[e2] = f2;
        }
        double ck = TYPED ? 0.5 * dt / m : ck1;
        double v0 = vel[e0] + (f0 + fold[e0]) * ck;
        double v1 = vel[e1] + (f1 + fold[e1]) * ck;
        double v2 = vel[e2] + (f2 + fold[e2]) * ck;
        vel[e0] = v0;
        vel[e1] = v1;
        vel[e2] = v2;
        double cd = TYPED ? 0.5 * dt * dt / m : cd1;
        double y0 = pos[e0] + v0 * dt, y1 = pos[e1] + v1 * dt, y2 = pos[e2] + v2 * dt;
        y0 = y0 + f0 * cd;
        y1 = y1 + f1 * cd;
        y2 = y2 + f2 * cd;
        bad |= !(y0 >= -L0 && y0 <= 2.0 * L0) | !(y1 >= -L1 && y1 <= 2.0 * L1) |
               !(y2 >= -L2 && y2 <= 2.0 * L2);
        pos[e0] = np_mod_in_range(y0, L0);
        pos[e1] = np_mod_in_range(y1, L1);
        pos[e2] = np_mod_in_range(y2, L2);
    }
    return bad;
}

}  // namespace

extern "C" {

int mdg_host_kick_drift_range(int64_t n, int64_t begin, int64_t end, int layout, double* pos,
                              double* vel, double* fnew, const double* fold,
                              const int32_t* type_id, const double* mass, const double domain[3],
                              const int periodic[3], double dt, int has_gravity, double gravity,
                              int* blowup) {
    if (n < 0 || begin < 0 || end > n || begin > end || (layout != MDG_AOS && layout != MDG_SOA))
        return MDG_EINVAL;
    int bad = 0;
    if (periodic[0] && periodic[1] && periodic[2]) {
#define MDG_KD(LY, TY) kick_drift_periodic<LY, TY>(n, begin, end, pos, vel, fnew, fold, type_id, mass, domain, dt, has_gravity, gravity)
        bad = layout == MDG_AOS ? (type_id ? MDG_KD(MDG_AOS, true) : MDG_KD(MDG_AOS, false))
                                : (type_id ? MDG_KD(MDG_SOA, true) : MDG_KD(MDG_SOA, false));
#undef MDG_KD
    } else {
        // reflective axes: the two passes over the range (same operations)
        int r = mdg_host_finish_kick_range(n, begin, end, layout, vel, fnew, fold, type_id, mass, dt,
                                           has_gravity, gravity);
        if (r) return r;
        r = mdg_host_drift_wrap_range_ex(n, begin, end, layout, pos, vel, nullptr, fnew, type_id,
                                         mass, domain, periodic, dt, 1, &bad);
        if (r) return r;
    }
    if (blowup) *blowup = bad;
    return MDG_OK;
}


int mdg_host_drift_wrap_range_ex(int64_t n, int64_t begin, int64_t end, int layout, double* pos,
                                 double* vel, const double* force, double* old_force,
                                 const int32_t* type_id, const double* mass, const double domain[3],
                                 const int periodic[3], double dt, int swapped, int* blowup) {
    if (n < 0 || begin < 0 || end > n || begin > end || (layout != MDG_AOS && layout != MDG_SOA))
        return MDG_EINVAL;
#define MDG_DRIFT(LY, TY) drift_all<LY, TY>(n, begin, end, pos, vel, force, old_force, type_id, mass, domain, periodic, dt, swapped != 0)
    int bad = layout == MDG_AOS ? (type_id ? MDG_DRIFT(MDG_AOS, true) : MDG_DRIFT(MDG_AOS, false))
                                : (type_id ? MDG_DRIFT(MDG_SOA, true) : MDG_DRIFT(MDG_SOA, false));
#undef MDG_DRIFT
    (void)np_mod;   // blow-ups (x outside [-L, 2L]) are reported; the caller raises BlowUpError
    if (blowup) *blowup = bad;
    return MDG_OK;
}

int mdg_host_drift_wrap_range(int64_t n, int64_t begin, int64_t end, int layout, double* pos,
                              double* vel, const double* force, double* old_force,
                              const int32_t* type_id, const double* mass, const double domain[3],
                              const int periodic[3], double dt, int* blowup) {
    return mdg_host_drift_wrap_range_ex(n, begin, end, layout, pos, vel, force, old_force, type_id,
                                        mass, domain, periodic, dt, 0, blowup);
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
#define MDG_KICK(LY, TY) kick_all<LY, TY>(n, begin, end, vel, force, old_force, type_id, mass, dt, has_gravity, gravity)
    if (layout == MDG_AOS) {
        if (type_id) MDG_KICK(MDG_AOS, true); else MDG_KICK(MDG_AOS, false);
    } else {
        if (type_id) MDG_KICK(MDG_SOA, true); else MDG_KICK(MDG_SOA, false);
    }
#undef MDG_KICK
    return MDG_OK;
}

int mdg_host_finish_kick(int64_t n, int layout, double* vel, double* force, const double* old_force,
                         const int32_t* type_id, const double* mass, double dt, int has_gravity,
                         double gravity) {
    return mdg_host_finish_kick_range(n, 0, n, layout, vel, force, old_force, type_id, mass, dt,
                                      has_gravity, gravity);
}

}  // extern "C"
