// Störmer-Verlet update split the reference's way, on device.
//
// Reference: integrator.py:31-44 (drift_with_force, finish_kick), :47-51
// (gravity), :98-128 (boundaries + BlowUpError), simulation.py:151-153,177,185
// (loop order: drift, boundaries, F -> F_old, ..., gravity, finish_kick).
// Arithmetic uses explicit round-to-nearest intrinsics so no multiply-add is
// contracted: the update is bit-identical to the reference's numpy sequence.
#include <cstddef>
#include <type_traits>

#include "device.cuh"

namespace mdg {

struct BoxParams {
    double L[3];
    int periodic[3];
    double dt;
    int64_t n;
    // the loop iteration this drift belongs to (mdg_set_iteration) and the
    // slot that keeps the first one whose drift raised the blow-up flag
    unsigned long long tag;
    unsigned long long* first;
};

// BlowUpError (integrator.py:108-116): the status bit, plus the earliest
// iteration that raised it, so the loop can report the reference's iteration
__device__ __forceinline__ void flag_blowup(const BoxParams& p, unsigned long long* blowup) {
    atomicOr(blowup, 1ull);
    atomicMin(p.first, p.tag);
}

// np.mod(x, L) (integrator.py:118): fmod with sign fix, +0.0 for exact zeros.
// Inside [-L, 2L] no fmod is needed: [0, L) -> x (+0.0 for -0.0); [L, 2L] ->
// x - L, exact by Sterbenz (2L -> 0); [-L, 0) -> x + L, the rounded addition
// numpy's sign fix performs.
__device__ __forceinline__ double np_mod(double x, double L) {
    if (x >= 0.0 && x < L) return __dadd_rn(x, 0.0);
    if (x >= L && x <= 2.0 * L) return x == 2.0 * L ? 0.0 : __dadd_rn(x, -L);
    if (x >= -L && x < 0.0) return __dadd_rn(x, L);
    double r = fmod(x, L);
    if (r != 0.0) {
        if ((r < 0.0) != (L < 0.0)) r = __dadd_rn(r, L);
    } else {
        r = 0.0;
    }
    return r;
}

template <int LAYOUT>
__global__ void drift_wrap_kernel(BoxParams p, const int* __restrict__ tid,
                                  const double* __restrict__ mass, double* __restrict__ pos,
                                  double* __restrict__ vel, const double* __restrict__ force,
                                  double* __restrict__ old_force, unsigned long long* blowup) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    double m = mass[tid ? tid[i] : 0];
    double c = __ddiv_rn(__dmul_rn(__dmul_rn(0.5, p.dt), p.dt), m);
    bool bad = false;
    for (int k = 0; k < 3; ++k) {
        size_t a = pidx<LAYOUT>(i, k, p.n);
        double f = force[a];
        double x = __dadd_rn(pos[a], __dmul_rn(vel[a], p.dt));
        x = __dadd_rn(x, __dmul_rn(f, c));
        double L = p.L[k];
        if (!(x >= -L && x <= 2.0 * L)) bad = true;
        if (p.periodic[k]) {
            x = np_mod(x, L);
        } else if (x < 0.0) {
            x = -x;
            vel[a] = -vel[a];
        } else if (x > L) {
            x = __dadd_rn(2.0 * L, -x);
            vel[a] = -vel[a];
        }
        pos[a] = x;
        old_force[a] = f;
    }
    if (bad) flag_blowup(p, blowup);
}

template <int LAYOUT>
__global__ void finish_kick_kernel(BoxParams p, const int* __restrict__ tid,
                                   const double* __restrict__ mass, double* __restrict__ vel,
                                   double* __restrict__ force, const double* __restrict__ old_force,
                                   int has_gravity, double g) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    double m = mass[tid ? tid[i] : 0];
    if (has_gravity) {
        size_t a = pidx<LAYOUT>(i, 2, p.n);
        force[a] = __dadd_rn(force[a], __dmul_rn(m, g));
    }
    double c = __ddiv_rn(__dmul_rn(0.5, p.dt), m);
    for (int k = 0; k < 3; ++k) {
        size_t a = pidx<LAYOUT>(i, k, p.n);
        vel[a] = __dadd_rn(vel[a], __dmul_rn(__dadd_rn(force[a], old_force[a]), c));
    }
}

// finish_kick of step s fused with the drift + boundaries of step s+1: per
// element exactly finish_kick_kernel's operations, then drift_wrap_kernel's
// (gravity into F_z, v += (F + F_old) dt/(2m), x += v dt, x += F dt^2/(2m),
// wrap / reflect with the velocity flip, blow-up test), one pass over the
// particle state instead of two.  COPY: F -> F_old as drift_wrap does;
// otherwise the caller swaps its force / old_force buffers afterwards.
template <int LAYOUT, bool COPY>
__global__ void kick_drift_kernel(BoxParams p, const int* __restrict__ tid,
                                  const double* __restrict__ mass, double* __restrict__ pos,
                                  double* __restrict__ vel, double* __restrict__ force,
                                  double* __restrict__ old_force, int has_gravity, double g,
                                  unsigned long long* blowup) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    double m = mass[tid ? tid[i] : 0];
    double ck = __ddiv_rn(__dmul_rn(0.5, p.dt), m);
    double cd = __ddiv_rn(__dmul_rn(__dmul_rn(0.5, p.dt), p.dt), m);
    bool bad = false;
    for (int k = 0; k < 3; ++k) {
        size_t a = pidx<LAYOUT>(i, k, p.n);
        double f = force[a];
        if (k == 2 && has_gravity) {
            f = __dadd_rn(f, __dmul_rn(m, g));
            force[a] = f;
        }
        double v = __dadd_rn(vel[a], __dmul_rn(__dadd_rn(f, old_force[a]), ck));
        double x = __dadd_rn(pos[a], __dmul_rn(v, p.dt));
        x = __dadd_rn(x, __dmul_rn(f, cd));
        double L = p.L[k];
        if (!(x >= -L && x <= 2.0 * L)) bad = true;
        if (p.periodic[k]) {
            x = np_mod(x, L);
        } else if (x < 0.0) {
            x = -x;
            v = -v;
        } else if (x > L) {
            x = __dadd_rn(2.0 * L, -x);
            v = -v;
        }
        pos[a] = x;
        vel[a] = v;
        if (COPY) old_force[a] = f;
    }
    if (bad) flag_blowup(p, blowup);
}

// Capped steepest descent used to relax overlapping random inputs (BASELINE
// configs 2 and 4; no reference counterpart): x += F/|F| * min(gamma|F|, dmax),
// then the boundary rule of the axis.
template <int LAYOUT>
__global__ void sd_step_kernel(BoxParams p, double* __restrict__ pos, double* __restrict__ vel,
                               const double* __restrict__ force, double gamma, double dmax,
                               unsigned long long* blowup) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    double f[3];
    for (int k = 0; k < 3; ++k) f[k] = force[pidx<LAYOUT>(i, k, p.n)];
    double fn = sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
    double scale = 0.0;
    if (fn > 0.0) {
        double d = gamma * fn;
        if (d > dmax) d = dmax;
        scale = d / fn;
    }
    bool bad = false;
    for (int k = 0; k < 3; ++k) {
        size_t a = pidx<LAYOUT>(i, k, p.n);
        double x = pos[a] + scale * f[k];
        double L = p.L[k];
        if (!(x >= -L && x <= 2.0 * L)) bad = true;
        if (p.periodic[k]) x = np_mod(x, L);
        else if (x < 0.0) x = -x;
        else if (x > L) x = 2.0 * L - x;
        pos[a] = x;
    }
    if (bad) flag_blowup(p, blowup);
}

static BoxParams box(const Context& c, double dt) {
    BoxParams p;
    for (int k = 0; k < 3; ++k) {
        p.L[k] = c.L[k];
        p.periodic[k] = c.periodic[k];
    }
    p.dt = dt;
    p.n = c.n;
    p.tag = (unsigned long long)c.iter_tag;
    p.first = c.scal.p + 8;
    return p;
}

void integ_drift_wrap(Context& c, double dt) {
    if (c.n == 0) return;
    BoxParams p = box(c, dt);
    dim3 b(blocks_for(c.n, 256)), t(256);
    if (c.layout == AOS)
        drift_wrap_kernel<AOS><<<b, t, 0, c.stream>>>(p, c.tid, c.d_mass.p, c.pos, c.vel, c.force, c.old_force, c.scal.p + 2), note_launch();
    else
        drift_wrap_kernel<SOA><<<b, t, 0, c.stream>>>(p, c.tid, c.d_mass.p, c.pos, c.vel, c.force, c.old_force, c.scal.p + 2), note_launch();
}

void integ_finish_kick(Context& c, double dt, int has_gravity, double gravity) {
    if (c.n == 0) return;
    BoxParams p = box(c, dt);
    dim3 b(blocks_for(c.n, 256)), t(256);
    if (c.layout == AOS)
        finish_kick_kernel<AOS><<<b, t, 0, c.stream>>>(p, c.tid, c.d_mass.p, c.vel, c.force, c.old_force, has_gravity, gravity), note_launch();
    else
        finish_kick_kernel<SOA><<<b, t, 0, c.stream>>>(p, c.tid, c.d_mass.p, c.vel, c.force, c.old_force, has_gravity, gravity), note_launch();
}

void integ_kick_drift(Context& c, double dt, int has_gravity, double gravity, bool copy) {
    if (c.n == 0) return;
    BoxParams p = box(c, dt);
    dim3 b(blocks_for(c.n, 256)), t(256);
#define MDG_KD(LY, CP) kick_drift_kernel<LY, CP><<<b, t, 0, c.stream>>>(p, c.tid, c.d_mass.p, c.pos, c.vel, c.force, c.old_force, has_gravity, gravity, c.scal.p + 2), note_launch()
    if (c.layout == AOS) {
        if (copy) MDG_KD(AOS, true); else MDG_KD(AOS, false);
    } else {
        if (copy) MDG_KD(SOA, true); else MDG_KD(SOA, false);
    }
#undef MDG_KD
}

// mdg_run's graph replays patch the iteration tag of the captured kick_drift
// launch (its first parameter, a BoxParams)
template <class... A>
constexpr int kernel_nparams(void (*)(A...)) { return (int)sizeof...(A); }
static_assert(std::is_same<decltype(kick_drift_kernel<AOS, false>),
                           void(BoxParams, const int*, const double*, double*, double*, double*,
                                double*, int, double, unsigned long long*)>::value,
              "mdg_run patches kick_drift_kernel's first parameter (a BoxParams) per graph replay");
size_t integ_box_size() { return sizeof(BoxParams); }
size_t integ_box_tag_offset() { return offsetof(BoxParams, tag); }
int integ_kick_drift_nparams() { return kernel_nparams(&kick_drift_kernel<AOS, false>); }

void integ_sd_step(Context& c, double gamma, double dmax) {
    if (c.n == 0) return;
    BoxParams p = box(c, 0.0);
    dim3 b(blocks_for(c.n, 256)), t(256);
    if (c.layout == AOS)
        sd_step_kernel<AOS><<<b, t, 0, c.stream>>>(p, c.pos, c.vel, c.force, gamma, dmax, c.scal.p + 2), note_launch();
    else
        sd_step_kernel<SOA><<<b, t, 0, c.stream>>>(p, c.pos, c.vel, c.force, gamma, dmax, c.scal.p + 2), note_launch();
}

}  // namespace mdg
