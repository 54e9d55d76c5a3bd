// Device-side helpers shared by the kernels of libmdg.
#pragma once

#include "mdg.cuh"

namespace mdg {

// LJ 12-6 scalar of the reference pair blocks (kernels.py:41-45):
//   inv = 1/r2; a = sig2*inv; a6 = a^3; fs = eps24*(2 a6 a6 - a6)*inv
// F_i += fs * (x_i - x_j).
__device__ __forceinline__ double lj_fs(double r2, double s2, double e24) {
    double inv = 1.0 / r2;
    double a = s2 * inv;
    double a6 = a * a * a;
    return e24 * (2.0 * a6 * a6 - a6) * inv;
}

// 1/x: MUFU.RCP64H seed (~2^-22) + one cubically convergent correction
// y(1 + e + e^2), e = 1 - x y: three DFMAs to full double precision (the LJ
// minimum cancels 2 a6 - 1, so a single Newton step's 1e-13 is visible
// there), instead of the IEEE division sequence with its slow-path branch.
__device__ __forceinline__ double fast_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    double t = fma(e, e, e);
    return fma(y, t, y);
}

__device__ __forceinline__ double lj_fs_fast(double r2, double s2, double e24) {
    double y = fast_rcp(r2);
    double a = s2 * y;
    double a6 = a * a * a;
    return (e24 * y) * (a6 * fma(2.0, a6, -1.0));
}

template <bool MT>
__device__ __forceinline__ void lj_params(const LJTab& t, int ti, int tj, double& s2, double& e24) {
    if (MT) {
        s2 = t.sig2[ti * t.T + tj];
        e24 = t.eps24[ti * t.T + tj];
    } else {
        s2 = t.sig2[0];
        e24 = t.eps24[0];
    }
}

// One 256-bit read-only load of a 32-byte record (LDG.E.ENL2.256 on sm_100a):
// a gathered double4 costs one L1 wavefront instead of LDG.128 + LDG.64.
__device__ __forceinline__ double4 ldg256(const double4* p) {
    double4 v;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
        : "l"(p));
    return v;
}

// Cell-sorted scratch positions (LayoutBuffers.pos, containers.py:126-154).
// AoS: one 32-byte record {x, y, z, type}; SoA: three component arrays + types.
template <int LAYOUT>
struct ScratchPos {
    const double4* __restrict__ p4;
    const double* __restrict__ x;
    const double* __restrict__ y;
    const double* __restrict__ z;
    const int* __restrict__ tid;
    __device__ __forceinline__ void load(int r, double& px, double& py, double& pz, int& t) const {
        if (LAYOUT == AOS) {
            double4 v = ldg256(p4 + r);
            px = v.x; py = v.y; pz = v.z; t = (int)v.w;
        } else {
            px = x[r]; py = y[r]; pz = z[r]; t = tid[r];
        }
    }
};

// Scratch forces: AoS (m,3) interleaved, SoA (3,m).
template <int LAYOUT>
struct ScratchForce {
    double* __restrict__ f;
    int m;
    __device__ __forceinline__ double* at(int r, int k) const {
        return LAYOUT == AOS ? f + 3 * (size_t)r + k : f + (size_t)k * m + r;
    }
};

// Particle arrays owned by the caller: AoS (N,3), SoA (3,N).
template <int LAYOUT>
__device__ __forceinline__ size_t pidx(int64_t i, int k, int64_t n) {
    return LAYOUT == AOS ? (size_t)(3 * i + k) : (size_t)(k * n + i);
}

struct GridView {
    int D0, D1, D2;
    int H0, H1, H2;
    int S0, S1, S2;
    const int* __restrict__ start;   // ncells + 1 (end = start[c+1])
    const int* __restrict__ row_cell;
    int m;
    __device__ __forceinline__ void decode(int c, int& x, int& y, int& z) const {
        z = c % D2;
        int t = c / D2;
        y = t % D1;
        x = t / D1;
    }
    __device__ __forceinline__ bool owned(int x, int y, int z) const {
        return x >= H0 && x < H0 + S0 && y >= H1 && y < H1 + S1 && z >= H2 && z < H2 + S2;
    }
    __device__ __forceinline__ bool in_grid(int x, int y, int z) const {
        return x >= 0 && x < D0 && y >= 0 && y < D1 && z >= 0 && z < D2;
    }
    __device__ __forceinline__ int flat(int x, int y, int z) const { return (x * D1 + y) * D2 + z; }
};

inline GridView make_view(const Grid& gr) {
    GridView v;
    v.D0 = gr.g.D[0]; v.D1 = gr.g.D[1]; v.D2 = gr.g.D[2];
    v.H0 = gr.g.H[0]; v.H1 = gr.g.H[1]; v.H2 = gr.g.H[2];
    v.S0 = gr.g.S[0]; v.S1 = gr.g.S[1]; v.S2 = gr.g.S[2];
    v.start = gr.cell_start.p;
    v.row_cell = gr.row_cell.p;
    v.m = (int)gr.m;
    return v;
}

// Warp-aggregated 64-bit counter update (within-cutoff evaluation count,
// kernels.py:9-11).  Must be called by all lanes of the warp.
__device__ __forceinline__ void warp_count(unsigned long long* counter, unsigned cnt) {
    unsigned s = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(counter, (unsigned long long)s);
}

}  // namespace mdg
