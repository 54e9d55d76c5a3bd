// Linked-cells force traversals on the cell-sorted scratch arrays.
//
// Reference: kernels.py:24-725 (pair blocks, C08/forward/directed sweeps) and
// the schedules of containers.py:176-335.  GPU realisation per traversal:
//
//   C01  thread per owned row, gathers own cell + full pruned stencil, writes
//        only its own row (no atomics)                      kernels.py:584-725
//   SLI  thread per owned row, own cell (j>i) + forward stencil, all writes
//        through fp64 RED (the lock-free analogue of the seam locks,
//        containers.py:288-322)                             kernels.py:493-579
//   C18  default: every base cell in ONE launch, S row-slot threads per base
//        cell (own cell j>i + forward stencil), writes through fp64 RED --
//        on the GPU the colour barriers only serialise work the atomics
//        already make safe (CSF 0.5: 75 launches 14.9 ms -> 1.0 ms).
//        MDG_LC_ROWS=0: one launch per base colour (strides o+1, 2o+1, 2o+1),
//        warp per base cell, 32x32 rotation tiles (lane l pairs its i with
//        j=(l+k) mod P at step k, so j-side updates never collide), plain
//        stores: same-colour bases touch disjoint cells  containers.py:269-287
//   C08  one launch per anchor colour (stride o+1 per axis), the schedule
//        kept.  Dense cells (>= 8 rows): warp per anchor block, rotation tiles,
//        plain stores.  Sparse cells: thread per (anchor, block cell, row
//        slot) over the pairs whose first cell is that block cell (C08Table),
//        fp64 RED (CSF 0.5: 11.8 -> 4.5 ms).  MDG_LC_C08=0 tiles always,
//        =2 every anchor in one launch                 kernels.py:373-488
//
// N3L: one evaluation per pair, reaction subtracted from j (count 1).
// NoN3L: both directions evaluated separately, each counted (count 2), exactly
// as the reference's _pair_no3/_intra_no3 blocks.
#include "device.cuh"

namespace mdg {

enum Traversal { T_C01 = 0, T_C08 = 1, T_C18 = 2, T_SLI = 3 };

template <int LAYOUT, bool MT>
__device__ __forceinline__ bool pair_force(const ScratchPos<LAYOUT>& sp, const LJTab& tab, int j,
                                           double xi, double yi, double zi, int ti, double& dx,
                                           double& dy, double& dz, double& fs, int& tj) {
    double xj, yj, zj;
    sp.load(j, xj, yj, zj, tj);
    dx = xi - xj;
    dy = yi - yj;
    dz = zi - zj;
    double r2 = dx * dx + dy * dy + dz * dz;
    if (!(r2 < tab.rc2)) return false;
    double s2, e24;
    lj_params<MT>(tab, ti, tj, s2, e24);
    fs = lj_fs(r2, s2, e24);
    return true;
}

// ------------------------------------------------------------------ C01

template <int LAYOUT, bool MT>
__global__ void __launch_bounds__(128) lc_c01_kernel(GridView gv, ScratchPos<LAYOUT> sp,
                                                     ScratchForce<LAYOUT> sf, LJTab tab, Stencil st,
                                                     unsigned long long* counter) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned cnt = 0;
    if (r < gv.m) {
        int cell = gv.row_cell[r], cx, cy, cz;
        gv.decode(cell, cx, cy, cz);
        if (gv.owned(cx, cy, cz)) {
            double xi, yi, zi;
            int ti;
            sp.load(r, xi, yi, zi, ti);
            double fx = 0.0, fy = 0.0, fz = 0.0;
            auto visit = [&](int j) {
                double dx, dy, dz, fs;
                int tj;
                if (pair_force<LAYOUT, MT>(sp, tab, j, xi, yi, zi, ti, dx, dy, dz, fs, tj)) {
                    ++cnt;
                    fx += fs * dx;
                    fy += fs * dy;
                    fz += fs * dz;
                }
            };
            int s = gv.start[cell], e = gv.start[cell + 1];
            for (int j = s; j < e; ++j)
                if (j != r) visit(j);
            for (int k = 0; k < st.n; ++k) {
                int x2 = cx + st.d[k][0], y2 = cy + st.d[k][1], z2 = cz + st.d[k][2];
                if (!gv.in_grid(x2, y2, z2)) continue;
                int c2 = gv.flat(x2, y2, z2);
                int e2 = gv.start[c2 + 1];
                for (int j = gv.start[c2]; j < e2; ++j) visit(j);
            }
            *sf.at(r, 0) = fx;
            *sf.at(r, 1) = fy;
            *sf.at(r, 2) = fz;
        }
    }
    warp_count(counter, cnt);
}

// ------------------------------------------------------------------ SLI (atomics)

template <int LAYOUT, bool MT, bool N3L>
__global__ void __launch_bounds__(128) lc_fwd_atomic_kernel(GridView gv, ScratchPos<LAYOUT> sp,
                                                            ScratchForce<LAYOUT> sf, LJTab tab,
                                                            Stencil st,
                                                            unsigned long long* counter) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned cnt = 0;
    if (r < gv.m) {
        int cell = gv.row_cell[r], cx, cy, cz;
        gv.decode(cell, cx, cy, cz);
        if (gv.owned(cx, cy, cz)) {
            double xi, yi, zi;
            int ti;
            sp.load(r, xi, yi, zi, ti);
            double fx = 0.0, fy = 0.0, fz = 0.0;
            auto visit = [&](int j) {
                double dx, dy, dz, fs;
                int tj;
                if (pair_force<LAYOUT, MT>(sp, tab, j, xi, yi, zi, ti, dx, dy, dz, fs, tj)) {
                    fx += fs * dx;
                    fy += fs * dy;
                    fz += fs * dz;
                    if (N3L) {
                        ++cnt;
                        atomicAdd(sf.at(j, 0), -(fs * dx));
                        atomicAdd(sf.at(j, 1), -(fs * dy));
                        atomicAdd(sf.at(j, 2), -(fs * dz));
                    } else {
                        // reverse direction evaluated on its own (kernels.py:86-98)
                        double bx = -dx, by = -dy, bz = -dz;
                        double s2, e24;
                        lj_params<MT>(tab, tj, ti, s2, e24);
                        double gs = lj_fs(bx * bx + by * by + bz * bz, s2, e24);
                        cnt += 2;
                        atomicAdd(sf.at(j, 0), gs * bx);
                        atomicAdd(sf.at(j, 1), gs * by);
                        atomicAdd(sf.at(j, 2), gs * bz);
                    }
                }
            };
            int e = gv.start[cell + 1];
            for (int j = r + 1; j < e; ++j) visit(j);
            for (int k = 0; k < st.n; ++k) {
                int x2 = cx + st.d[k][0], y2 = cy + st.d[k][1], z2 = cz + st.d[k][2];
                if (!gv.in_grid(x2, y2, z2)) continue;
                int c2 = gv.flat(x2, y2, z2);
                int e2 = gv.start[c2 + 1];
                for (int j = gv.start[c2]; j < e2; ++j) visit(j);
            }
            atomicAdd(sf.at(r, 0), fx);
            atomicAdd(sf.at(r, 1), fy);
            atomicAdd(sf.at(r, 2), fz);
        }
    }
    warp_count(counter, cnt);
}

// ------------------------------------------------------------------ colour tiles

struct WarpTile {
    double x[32], y[32], z[32];
    double fx[32], fy[32], fz[32];
    int t[32];
};

// i-rows i0..i0+ni-1 sit in the lanes (registers), j-rows j0..j0+nj-1 are
// staged in shared memory.  tri: same chunk, pairs j > i only.
template <int LAYOUT, bool MT, bool N3L>
__device__ __forceinline__ void tile(WarpTile& w, const ScratchPos<LAYOUT>& sp,
                                     const ScratchForce<LAYOUT>& sf, const LJTab& tab, int ni,
                                     int j0, int nj, bool tri, double xi, double yi, double zi,
                                     int ti, double& fx, double& fy, double& fz, unsigned& cnt) {
    int lane = threadIdx.x & 31;
    if (lane < nj) {
        double x, y, z;
        int t;
        sp.load(j0 + lane, x, y, z, t);
        w.x[lane] = x; w.y[lane] = y; w.z[lane] = z; w.t[lane] = t;
        w.fx[lane] = 0.0; w.fy[lane] = 0.0; w.fz[lane] = 0.0;
    }
    __syncwarp();
    auto body = [&](int j) {
        double dx = xi - w.x[j], dy = yi - w.y[j], dz = zi - w.z[j];
        double r2 = dx * dx + dy * dy + dz * dz;
        if (r2 < tab.rc2) {
            int tj = w.t[j];
            double s2, e24;
            lj_params<MT>(tab, ti, tj, s2, e24);
            double fs = lj_fs(r2, s2, e24);
            fx += fs * dx;
            fy += fs * dy;
            fz += fs * dz;
            if (N3L) {
                ++cnt;
                w.fx[j] -= fs * dx;
                w.fy[j] -= fs * dy;
                w.fz[j] -= fs * dz;
            } else {
                double bx = -dx, by = -dy, bz = -dz;
                lj_params<MT>(tab, tj, ti, s2, e24);
                double gs = lj_fs(bx * bx + by * by + bz * bz, s2, e24);
                cnt += 2;
                w.fx[j] += gs * bx;
                w.fy[j] += gs * by;
                w.fz[j] += gs * bz;
            }
        }
    };
    if (tri) {
        for (int k = 1; k < ni; ++k) {
            int j = lane + k;
            if (j < ni) body(j);
            __syncwarp();
        }
    } else {
        int P = ni > nj ? ni : nj;
        for (int k = 0; k < P; ++k) {
            int j = lane + k;
            if (j >= P) j -= P;
            if (lane < ni && j < nj) body(j);
            __syncwarp();
        }
    }
    if (lane < nj) {
        *sf.at(j0 + lane, 0) += w.fx[lane];
        *sf.at(j0 + lane, 1) += w.fy[lane];
        *sf.at(j0 + lane, 2) += w.fz[lane];
    }
    __syncwarp();
}

// All pairs of cell c1 (i side) against cell c2 (j side), or the intra pairs
// of c1 when c2 < 0.  Plain read-modify-write stores: the colour schedule
// guarantees that no other warp of the launch touches these rows.
template <int LAYOUT, bool MT, bool N3L>
__device__ __forceinline__ void cell_pair(WarpTile& w, const GridView& gv,
                                          const ScratchPos<LAYOUT>& sp,
                                          const ScratchForce<LAYOUT>& sf, const LJTab& tab, int c1,
                                          int c2, unsigned& cnt) {
    int lane = threadIdx.x & 31;
    int s1 = gv.start[c1], e1 = gv.start[c1 + 1];
    bool intra = c2 < 0;
    int s2 = intra ? s1 : gv.start[c2], e2 = intra ? e1 : gv.start[c2 + 1];
    if (e1 <= s1 || e2 <= s2) return;
    for (int i0 = s1; i0 < e1; i0 += 32) {
        int ni = min(32, e1 - i0);
        double xi = 0.0, yi = 0.0, zi = 0.0;
        int ti = 0;
        if (lane < ni) sp.load(i0 + lane, xi, yi, zi, ti);
        double fx = 0.0, fy = 0.0, fz = 0.0;
        for (int j0 = intra ? i0 : s2; j0 < e2; j0 += 32) {
            int nj = min(32, e2 - j0);
            tile<LAYOUT, MT, N3L>(w, sp, sf, tab, ni, j0, nj, intra && j0 == i0, xi, yi, zi, ti, fx,
                                  fy, fz, cnt);
        }
        if (lane < ni) {
            *sf.at(i0 + lane, 0) += fx;
            *sf.at(i0 + lane, 1) += fy;
            *sf.at(i0 + lane, 2) += fz;
        }
        __syncwarp();
    }
}

struct ColourLaunch {
    int p[3];        // colour phase per axis
    int stride[3];
    int lo[3];       // first base/anchor per axis (before phase)
    int hi[3];       // exclusive bound per axis
    int cnt[3];      // bases/anchors per axis in this colour
};

// C18: one warp per base cell of one colour (kernels.py:493-537 driven by
// containers.py:269-287).
template <int LAYOUT, bool MT, bool N3L>
__global__ void __launch_bounds__(128) lc_c18_kernel(GridView gv, ScratchPos<LAYOUT> sp,
                                                     ScratchForce<LAYOUT> sf, LJTab tab, Stencil st,
                                                     ColourLaunch cl,
                                                     unsigned long long* counter) {
    __shared__ WarpTile tiles[4];
    WarpTile& w = tiles[threadIdx.x >> 5];
    int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned cnt = 0;
    int total = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
    if (wid < total) {
        int kz = wid % cl.cnt[2], t = wid / cl.cnt[2];
        int ky = t % cl.cnt[1], kx = t / cl.cnt[1];
        int bx = cl.lo[0] + cl.p[0] + kx * cl.stride[0];
        int by = cl.lo[1] + cl.p[1] + ky * cl.stride[1];
        int bz = cl.lo[2] + cl.p[2] + kz * cl.stride[2];
        int c1 = gv.flat(bx, by, bz);
        if (gv.start[c1 + 1] > gv.start[c1]) {
            cell_pair<LAYOUT, MT, N3L>(w, gv, sp, sf, tab, c1, -1, cnt);
            for (int k = 0; k < st.n; ++k) {
                int x2 = bx + st.d[k][0], y2 = by + st.d[k][1], z2 = bz + st.d[k][2];
                if (!gv.in_grid(x2, y2, z2)) continue;
                cell_pair<LAYOUT, MT, N3L>(w, gv, sp, sf, tab, c1, gv.flat(x2, y2, z2), cnt);
            }
        }
    }
    warp_count(counter, cnt);
}

// C08: one warp per anchor of one colour (kernels.py:373-433).
template <int LAYOUT, bool MT, bool N3L>
__global__ void __launch_bounds__(128) lc_c08_kernel(GridView gv, ScratchPos<LAYOUT> sp,
                                                     ScratchForce<LAYOUT> sf, LJTab tab, Stencil st,
                                                     ColourLaunch cl,
                                                     unsigned long long* counter) {
    __shared__ WarpTile tiles[4];
    WarpTile& w = tiles[threadIdx.x >> 5];
    int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned cnt = 0;
    int total = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
    if (wid < total) {
        int kz = wid % cl.cnt[2], t = wid / cl.cnt[2];
        int ky = t % cl.cnt[1], kx = t / cl.cnt[1];
        int ax = cl.p[0] + kx * cl.stride[0];
        int ay = cl.p[1] + ky * cl.stride[1];
        int az = cl.p[2] + kz * cl.stride[2];
        if (gv.owned(ax, ay, az)) cell_pair<LAYOUT, MT, N3L>(w, gv, sp, sf, tab, gv.flat(ax, ay, az), -1, cnt);
        for (int k = 0; k < st.n; ++k) {
            int dx = st.d[k][0], dy = st.d[k][1], dz = st.d[k][2];
            int c1x = dx < 0 ? ax - dx : ax, c1y = dy < 0 ? ay - dy : ay, c1z = dz < 0 ? az - dz : az;
            if (!gv.owned(c1x, c1y, c1z)) continue;
            int c2x = c1x + dx, c2y = c1y + dy, c2z = c1z + dz;
            if (!gv.in_grid(c2x, c2y, c2z)) continue;
            cell_pair<LAYOUT, MT, N3L>(w, gv, sp, sf, tab, gv.flat(c1x, c1y, c1z),
                                       gv.flat(c2x, c2y, c2z), cnt);
        }
    }
    warp_count(counter, cnt);
}

// ------------------------------------------------------------------ colour rows
//
// The same colour schedules with row-level threads instead of warp tiles:
// thread = (unit of the colour, row slot), unit = a C18 base cell or a C08
// anchor block.  A row walks exactly the cell pairs its unit assigns to its
// cell, keeps f_i in registers and adds the reactions (N3L) / reverse
// evaluations (NoN3L) with fp64 atomics; same-colour units touch disjoint
// cells, so the atomics never collide across units.  Pair sets and counts are
// those of the tiles; with small cells (CSF 0.5: ~2 rows per cell) a 32x32
// tile keeps 2-3 lanes busy, a row slot keeps all of them.

template <int LAYOUT, bool MT, bool N3L>
__device__ __forceinline__ void row_vs_range(const ScratchPos<LAYOUT>& sp, const ScratchForce<LAYOUT>& sf,
                                             const LJTab& tab, int j0, int j1, double xi, double yi,
                                             double zi, int ti, double& fx, double& fy, double& fz,
                                             unsigned& cnt) {
    for (int j = j0; j < j1; ++j) {
        double dx, dy, dz, fs;
        int tj;
        if (pair_force<LAYOUT, MT>(sp, tab, j, xi, yi, zi, ti, dx, dy, dz, fs, tj)) {
            fx += fs * dx;
            fy += fs * dy;
            fz += fs * dz;
            if (N3L) {
                ++cnt;
                atomicAdd(sf.at(j, 0), -(fs * dx));
                atomicAdd(sf.at(j, 1), -(fs * dy));
                atomicAdd(sf.at(j, 2), -(fs * dz));
            } else {
                double bx = -dx, by = -dy, bz = -dz;
                double s2, e24;
                lj_params<MT>(tab, tj, ti, s2, e24);
                double gs = lj_fs(bx * bx + by * by + bz * bz, s2, e24);
                cnt += 2;
                atomicAdd(sf.at(j, 0), gs * bx);
                atomicAdd(sf.at(j, 1), gs * by);
                atomicAdd(sf.at(j, 2), gs * bz);
            }
        }
    }
}

// C18 rows: unit = base cell of the colour (kernels.py:493-537 per base).
template <int LAYOUT, bool MT, bool N3L>
__global__ void __launch_bounds__(128) lc_c18_rows_kernel(GridView gv, ScratchPos<LAYOUT> sp,
                                                          ScratchForce<LAYOUT> sf, LJTab tab,
                                                          Stencil st, ColourLaunch cl, int S,
                                                          unsigned long long* counter) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    int unit = t / S, slot = t % S;
    unsigned cnt = 0;
    int total = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
    if (unit < total) {
        int kz = unit % cl.cnt[2], u2 = unit / cl.cnt[2];
        int ky = u2 % cl.cnt[1], kx = u2 / cl.cnt[1];
        int bx = cl.lo[0] + cl.p[0] + kx * cl.stride[0];
        int by = cl.lo[1] + cl.p[1] + ky * cl.stride[1];
        int bz = cl.lo[2] + cl.p[2] + kz * cl.stride[2];
        int c1 = gv.flat(bx, by, bz);
        int s1 = gv.start[c1], e1 = gv.start[c1 + 1];
        for (int r = s1 + slot; r < e1; r += S) {
            double xi, yi, zi;
            int ti;
            sp.load(r, xi, yi, zi, ti);
            double fx = 0.0, fy = 0.0, fz = 0.0;
            row_vs_range<LAYOUT, MT, N3L>(sp, sf, tab, r + 1, e1, xi, yi, zi, ti, fx, fy, fz, cnt);
            for (int k = 0; k < st.n; ++k) {
                int x2 = bx + st.d[k][0], y2 = by + st.d[k][1], z2 = bz + st.d[k][2];
                if (!gv.in_grid(x2, y2, z2)) continue;
                int c2 = gv.flat(x2, y2, z2);
                row_vs_range<LAYOUT, MT, N3L>(sp, sf, tab, gv.start[c2], gv.start[c2 + 1], xi, yi, zi,
                                              ti, fx, fy, fz, cnt);
            }
            atomicAdd(sf.at(r, 0), fx);
            atomicAdd(sf.at(r, 1), fy);
            atomicAdd(sf.at(r, 2), fz);
        }
    }
    warp_count(counter, cnt);
}

// C08 rows: unit = anchor block of the colour (kernels.py:373-433): the
// anchor's intra pairs (owned anchor) and, per forward offset d, the pair
// (anchor + max(0, -d), that + d); a row of block cell c walks the pairs whose
// first cell is c.
// stencil entries grouped by the block offset of their first cell
// (max(0, -d) per axis), so a row visits only the pairs of its own cell
struct C08Table {
    int start[28];
    signed char d[kMaxStencil][3];
};

template <int LAYOUT, bool MT, bool N3L>
__global__ void __launch_bounds__(128) lc_c08_rows_kernel(GridView gv, ScratchPos<LAYOUT> sp,
                                                          ScratchForce<LAYOUT> sf, LJTab tab,
                                                          C08Table tb, ColourLaunch cl, int o0,
                                                          int o1, int o2, int S,
                                                          unsigned long long* counter) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    int unit = t / S, slot = t % S;
    unsigned cnt = 0;
    int total = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
    if (unit < total) {
        int kz = unit % cl.cnt[2], u2 = unit / cl.cnt[2];
        int ky = u2 % cl.cnt[1], kx = u2 / cl.cnt[1];
        int ax = cl.p[0] + kx * cl.stride[0];
        int ay = cl.p[1] + ky * cl.stride[1];
        int az = cl.p[2] + kz * cl.stride[2];
        // block cells anchor + [0, o]^3 (inside the grid), rows enumerated cell by cell
        int nb0 = min(o0 + 1, gv.D0 - ax), nb1 = min(o1 + 1, gv.D1 - ay), nb2 = min(o2 + 1, gv.D2 - az);
        int q = slot;
        for (int bi = 0; bi < nb0; ++bi)
            for (int bj = 0; bj < nb1; ++bj)
                for (int bk = 0; bk < nb2; ++bk) {
                    int cx = ax + bi, cy = ay + bj, cz = az + bk;
                    int c = gv.flat(cx, cy, cz);
                    int s1 = gv.start[c], e1 = gv.start[c + 1];
                    int nrow = e1 - s1;
                    if (!gv.owned(cx, cy, cz)) {   // a first cell must be owned
                        while (q < nrow) q += S;
                        q -= nrow;
                        continue;
                    }
                    for (; q < nrow; q += S) {
                        int r = s1 + q;
                        double xi, yi, zi;
                        int ti;
                        sp.load(r, xi, yi, zi, ti);
                        double fx = 0.0, fy = 0.0, fz = 0.0;
                        if (bi == 0 && bj == 0 && bk == 0)
                            row_vs_range<LAYOUT, MT, N3L>(sp, sf, tab, r + 1, e1, xi, yi, zi, ti, fx, fy, fz, cnt);
                        int slot_b = (bi * (o1 + 1) + bj) * (o2 + 1) + bk;
                        for (int e = tb.start[slot_b]; e < tb.start[slot_b + 1]; ++e) {
                            int dx = tb.d[e][0], dy = tb.d[e][1], dz = tb.d[e][2];
                            int x2 = cx + dx, y2 = cy + dy, z2 = cz + dz;
                            if (!gv.in_grid(x2, y2, z2)) continue;
                            int c2 = gv.flat(x2, y2, z2);
                            row_vs_range<LAYOUT, MT, N3L>(sp, sf, tab, gv.start[c2], gv.start[c2 + 1], xi, yi,
                                                          zi, ti, fx, fy, fz, cnt);
                        }
                        atomicAdd(sf.at(r, 0), fx);
                        atomicAdd(sf.at(r, 1), fy);
                        atomicAdd(sf.at(r, 2), fz);
                    }
                    q -= nrow;
                }
    }
    warp_count(counter, cnt);
}

// C08 with the colour schedule kept: one launch per anchor colour, thread per
// (anchor, block cell, row slot); a thread walks its rows of that cell against
// the pairs whose first cell is that block cell (C08Table) plus, in the anchor
// cell, the intra pairs.
template <int LAYOUT, bool MT, bool N3L>
__global__ void __launch_bounds__(128) lc_c08_cells_kernel(GridView gv, ScratchPos<LAYOUT> sp,
                                                           ScratchForce<LAYOUT> sf, LJTab tab,
                                                           C08Table tb, ColourLaunch cl, int o0,
                                                           int o1, int o2, int S,
                                                           unsigned long long* counter) {
    int nb = (o0 + 1) * (o1 + 1) * (o2 + 1);
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int slot = (int)(t % S);
    int64_t ub = t / S;
    int unit = (int)(ub / nb), b = (int)(ub % nb);
    unsigned cnt = 0;
    int total = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
    if (unit < total) {
        int kz = unit % cl.cnt[2], u2 = unit / cl.cnt[2];
        int ky = u2 % cl.cnt[1], kx = u2 / cl.cnt[1];
        int bi = b / ((o1 + 1) * (o2 + 1)), bj = (b / (o2 + 1)) % (o1 + 1), bk = b % (o2 + 1);
        int cx = cl.p[0] + kx * cl.stride[0] + bi;
        int cy = cl.p[1] + ky * cl.stride[1] + bj;
        int cz = cl.p[2] + kz * cl.stride[2] + bk;
        if (gv.in_grid(cx, cy, cz) && gv.owned(cx, cy, cz)) {
            int c = gv.flat(cx, cy, cz);
            int s1 = gv.start[c], e1 = gv.start[c + 1];
            for (int r = s1 + slot; r < e1; r += S) {
                double xi, yi, zi;
                int ti;
                sp.load(r, xi, yi, zi, ti);
                double fx = 0.0, fy = 0.0, fz = 0.0;
                unsigned before = cnt;
                if (b == 0)
                    row_vs_range<LAYOUT, MT, N3L>(sp, sf, tab, r + 1, e1, xi, yi, zi, ti, fx, fy, fz, cnt);
                for (int e = tb.start[b]; e < tb.start[b + 1]; ++e) {
                    int x2 = cx + tb.d[e][0], y2 = cy + tb.d[e][1], z2 = cz + tb.d[e][2];
                    if (!gv.in_grid(x2, y2, z2)) continue;
                    int c2 = gv.flat(x2, y2, z2);
                    row_vs_range<LAYOUT, MT, N3L>(sp, sf, tab, gv.start[c2], gv.start[c2 + 1], xi, yi, zi,
                                                  ti, fx, fy, fz, cnt);
                }
                if (cnt != before) {   // a row meets most block cells with no partner
                    atomicAdd(sf.at(r, 0), fx);
                    atomicAdd(sf.at(r, 1), fy);
                    atomicAdd(sf.at(r, 2), fz);
                }
            }
        }
    }
    warp_count(counter, cnt);
}

// C08 for small systems, deterministic: one warp per (anchor, block cell) of
// a colour, lanes = rows of that cell.  The warp evaluates, for its rows,
// every pair of the anchor that touches its cell -- as the first cell
// (partners c + d, d in t1[cell]), as the second (partners c - d, d in
// t2[cell]) and the anchor's intra pairs -- and writes only its own rows, so
// no two warps of a launch write the same row and no atomics are needed.
// Each pair is evaluated from both sides (F(j,i) = -F(i,j) bit for bit); the
// count is taken once per pair for N3L (first-cell side, j > i within a cell)
// and per direction for NoN3L, as the reference counts.  Twice the pair
// arithmetic of the tiles, 8 (27) times their warps: BASELINE config 1 has ~90
// anchors per colour, which leave a one-warp-per-anchor launch latency-bound.
//
// WPU > 1 (round 2): a CTA of WPU warps per (anchor, block cell) unit.  The
// unit's partner rows (its cell, the forward cells, the backward cells, in
// that order) are cut into 4-row rounds dealt round-robin to the warps; each
// warp keeps per-row partial sums, and warp 0 adds the WPU partials in warp
// order -- deterministic, no atomics, WPU times the parallelism of a colour
// (BASELINE config 1: 24 -> ~7 us per colour launch).
// ALL (WPU > 1): every colour in one launch.  Unit u of the launch belongs to
// the colour k with ca.ustart[k] <= u < ca.ustart[k + 1]; within a colour no
// two units share a cell, so each unit STORES its rows' sums into colour k's
// partial buffer (colours x 3m, zeroed first), and c08_colour_sum_kernel then
// adds a row's partials in colour order -- the same additions, in the same
// order, as the colour-by-colour launches accumulating into the scratch
// forces, so the result is bit-identical with 1 launch instead of 8.
struct C08All {
    ColourLaunch cl[8];
    int ustart[9];
    int ncol;
};

// The staged partner list of every unit (C08All launches), built once per
// grid rebuild by the LM = 1 instantiation and read by LM = 2: the per-step
// kernel then skips the range lookups, the length scan and the per-row range
// search (two CTA barriers and a chain of dependent loads per unit).  tot[u]
// = the unit's staged rows (-1: more than the staging capacity, the unit takes
// the unstaged path), j / f: staged row and flags, kStage per unit.
struct C08Lists {
    int* tot;
    int* j;
    unsigned char* f;
};
constexpr int kC08Stage = 512;

template <int LAYOUT, bool MT, bool N3L, int WPU, bool ALL = false, int LM = 0>
__global__ void __launch_bounds__(WPU == 1 ? 128 : 32 * WPU, ALL ? 32 / WPU : 1) lc_c08_cellwarp_kernel(
    GridView gv, ScratchPos<LAYOUT> sp, ScratchForce<LAYOUT> sf, LJTab tab, C08Table t1, C08Table t2,
    ColourLaunch cl, int o0, int o1, int o2, unsigned long long* counter, C08All ca = {},
    double* cpart = nullptr, C08Lists ul = {}) {
    int nb = (o0 + 1) * (o1 + 1) * (o2 + 1);
    int gw = WPU == 1 ? (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) : (int)blockIdx.x;
    if (ALL) {
        static_assert(!ALL || WPU > 1, "one launch of all colours: CTA units only");
        int k = 0;
        while (k + 1 < ca.ncol && gw >= ca.ustart[k + 1]) ++k;
        gw -= ca.ustart[k];
        cl = ca.cl[k];
        sf.f = cpart + (size_t)k * 3 * sf.m;
    }
    int lane = threadIdx.x & 31;
    const int w = WPU == 1 ? 0 : (int)(threadIdx.x >> 5);
    __shared__ double red[WPU > 1 ? WPU : 1][3][32];
    // WPU > 1: the unit's partner ranges and their rows, staged
    constexpr int kStage = WPU > 1 ? kC08Stage : 1;
    constexpr int kRng = WPU > 1 ? 2 * kMaxStencil + 2 : 1;
    __shared__ double st_x[kStage], st_y[kStage], st_z[kStage];
    __shared__ int st_t[kStage], st_j[kStage];
    __shared__ unsigned char st_f[kStage];
    __shared__ int st_a[kRng], st_off[kRng + 1], st_fl[kRng], st_n[2];
    // per warp and lane: the queued partners (staged indices) of one segment
    constexpr int kSeg = WPU > 1 ? 32 : 1;
    __shared__ unsigned short qbuf[WPU > 1 ? WPU : 1][kSeg][32];
    unsigned cnt = 0;
    int total = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
    int unit = gw / nb, beta = gw % nb;
    if (unit < total) {
        int kz = unit % cl.cnt[2], u2 = unit / cl.cnt[2];
        int ky = u2 % cl.cnt[1], kx = u2 / cl.cnt[1];
        int bi = beta / ((o1 + 1) * (o2 + 1)), bj = (beta / (o2 + 1)) % (o1 + 1), bk = beta % (o2 + 1);
        int cx = cl.p[0] + kx * cl.stride[0] + bi;
        int cy = cl.p[1] + ky * cl.stride[1] + bj;
        int cz = cl.p[2] + kz * cl.stride[2] + bk;
        if (WPU > 1 && gv.in_grid(cx, cy, cz)) {
            // the unit's partner rows staged in shared memory once (one round
            // of global loads for the whole CTA), then read as broadcasts
            int c = gv.flat(cx, cy, cz);
            int s1 = gv.start[c], e1 = gv.start[c + 1];
            bool own = gv.owned(cx, cy, cz);
            int tot = 0;
            bool staged = false;
            if (LM == 2) {   // the unit's list of this grid (C08Lists)
                tot = ul.tot[blockIdx.x];
                staged = tot >= 0;
                const size_t o = (size_t)blockIdx.x * kStage;
                for (int q = threadIdx.x; q < tot; q += blockDim.x) {
                    const int j = ul.j[o + q];
                    double xj, yj, zj;
                    int tj;
                    sp.load(j, xj, yj, zj, tj);
                    st_x[q] = xj;
                    st_y[q] = yj;
                    st_z[q] = zj;
                    st_t[q] = MT ? tj : 0;
                    st_j[q] = j;
                    st_f[q] = ul.f[o + q];
                }
            } else {
            // one partner range per thread (slot 0: the intra range, then the
            // forward entries whose first cell is this one, then the backward
            // ones), lengths scanned by one warp: no serial chain of loads
            const int nt1 = own ? t1.start[beta + 1] - t1.start[beta] : 0;
            const int nt2 = t2.start[beta + 1] - t2.start[beta];
            const int nrng = 1 + nt1 + nt2;
            for (int k = threadIdx.x; k < nrng; k += blockDim.x) {
                int a = 0, len = 0, fl = 0;
                if (k == 0) {
                    if (beta == 0 && own) { a = s1; len = e1 - s1; fl = 3; }   // counted | intra
                } else if (k <= nt1) {
                    int e = t1.start[beta] + k - 1;
                    int x2 = cx + t1.d[e][0], y2 = cy + t1.d[e][1], z2 = cz + t1.d[e][2];
                    if (gv.in_grid(x2, y2, z2)) {
                        int c2 = gv.flat(x2, y2, z2);
                        a = gv.start[c2];
                        len = gv.start[c2 + 1] - a;
                        fl = 1;
                    }
                } else {
                    int e = t2.start[beta] + k - 1 - nt1;
                    int x1 = cx - t2.d[e][0], y1 = cy - t2.d[e][1], z1 = cz - t2.d[e][2];
                    if (gv.in_grid(x1, y1, z1) && gv.owned(x1, y1, z1)) {
                        int c1 = gv.flat(x1, y1, z1);
                        a = gv.start[c1];
                        len = gv.start[c1 + 1] - a;
                    }
                }
                st_a[k] = a;
                st_off[k] = len;
                st_fl[k] = fl;
            }
            __syncthreads();
            if (threadIdx.x < 32) {   // exclusive scan of the lengths
                int carry = 0;
                for (int k0 = 0; k0 < nrng; k0 += 32) {
                    int k = k0 + lane;
                    int v = k < nrng ? st_off[k] : 0, x = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        int t = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += t;
                    }
                    if (k < nrng) st_off[k] = carry + x - v;
                    carry += __shfl_sync(0xffffffffu, x, 31);
                }
                if (lane == 0) {
                    st_off[nrng] = carry;
                    st_n[0] = nrng;
                    st_n[1] = carry;
                }
            }
            __syncthreads();
            const int nr = st_n[0];
            tot = st_n[1];
            staged = tot <= kStage;
            if (staged) {
                for (int q = threadIdx.x; q < tot; q += blockDim.x) {
                    int lo = 0, hi = nr - 1;   // the last range starting at or before q
                    while (lo < hi) {
                        int mid = (lo + hi + 1) >> 1;
                        if (st_off[mid] <= q) lo = mid; else hi = mid - 1;
                    }
                    int k = lo;
                    int j = st_a[k] + (q - st_off[k]);
                    if (LM == 1) {
                        ul.j[(size_t)blockIdx.x * kStage + q] = j;
                        ul.f[(size_t)blockIdx.x * kStage + q] = (unsigned char)st_fl[k];
                        continue;
                    }
                    double xj, yj, zj;
                    int tj;
                    sp.load(j, xj, yj, zj, tj);
                    st_x[q] = xj;
                    st_y[q] = yj;
                    st_z[q] = zj;
                    st_t[q] = MT ? tj : 0;
                    st_j[q] = j;
                    st_f[q] = (unsigned char)st_fl[k];
                }
            }
            if (LM == 1) {
                if (threadIdx.x == 0) ul.tot[blockIdx.x] = staged ? tot : -1;
                return;
            }
            }
            if (staged) {
                __syncthreads();
                for (int i0 = s1; i0 < e1; i0 += 32) {
                    int i = i0 + lane;
                    bool act = i < e1;
                    double xi = 0.0, yi = 0.0, zi = 0.0;
                    int ti = 0;
                    if (act) sp.load(i, xi, yi, zi, ti);
                    double fx = 0.0, fy = 0.0, fz = 0.0;
                    // this warp's staged partners: 4-row rounds dealt round-robin
                    // (candidate s of the warp is q = 4w + 4 WPU (s/4) + s%4), in
                    // segments of kSeg: first the exact r^2 < rc^2 test of every
                    // candidate (the reference's test, kernels.py:36-40), the
                    // passing ones queued per lane; then the force of the queued
                    // partners only, four at a time with one batched reciprocal
                    // -- ~8% of the candidates of a 27-cell neighbourhood are
                    // within rc, so the force arithmetic no longer runs on every
                    // candidate.  Sums in candidate order (deterministic).
                    for (int s0 = 0;; s0 += kSeg) {
                        if (4 * w + 4 * WPU * (s0 >> 2) >= tot) break;
                        int nq = 0;
                        for (int s = s0; s < s0 + kSeg; ++s) {
                            const int q = 4 * w + 4 * WPU * (s >> 2) + (s & 3);
                            if (q >= tot) break;
                            const double dx = xi - st_x[q], dy = yi - st_y[q], dz = zi - st_z[q];
                            const double r2 = dx * dx + dy * dy + dz * dz;
                            const int fl = st_f[q];
                            if (act && (!(fl & 2) || st_j[q] != i) && r2 < tab.rc2) {
                                qbuf[w][nq][lane] = (unsigned short)q;
                                ++nq;
                                cnt += (N3L ? ((fl & 1) && (!(fl & 2) || st_j[q] > i)) : 1) ? 1u : 0u;
                            }
                        }
                        const int nmax = __reduce_max_sync(0xffffffffu, (unsigned)nq);
                        for (int k0 = 0; k0 < nmax; k0 += 4) {
                            double dx[4], dy[4], dz[4], qq[4];
                            int tj[4];
                            bool ok[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                ok[u] = k0 + u < nq;
                                const int q = ok[u] ? qbuf[w][k0 + u][lane] : 0;
                                dx[u] = xi - st_x[q];
                                dy[u] = yi - st_y[q];
                                dz[u] = zi - st_z[q];
                                tj[u] = st_t[q];
                                const double r2 = dx[u] * dx[u] + dy[u] * dy[u] + dz[u] * dz[u];
                                qq[u] = ok[u] ? r2 : 1.0;
                            }
                            double p01 = qq[0] * qq[1], p23 = qq[2] * qq[3];
                            double y = fast_rcp(p01 * p23);
                            double y01 = y * p23, y23 = y * p01;
                            double inv[4] = {y01 * qq[1], y01 * qq[0], y23 * qq[3], y23 * qq[2]};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                double s2, e24;
                                lj_params<MT>(tab, ti, tj[u], s2, e24);
                                double aa = s2 * inv[u];
                                double a6 = aa * aa * aa;
                                double fs = (e24 * inv[u]) * (a6 * fma(2.0, a6, -1.0));
                                fs = ok[u] ? fs : 0.0;
                                fx += fs * dx[u];
                                fy += fs * dy[u];
                                fz += fs * dz[u];
                            }
                        }
                    }
                    red[w][0][lane] = fx;
                    red[w][1][lane] = fy;
                    red[w][2][lane] = fz;
                    __syncthreads();
                    if (w == 0 && act) {
                        double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
                        for (int q = 0; q < WPU; ++q) {
                            gx += red[q][0][lane];
                            gy += red[q][1][lane];
                            gz += red[q][2][lane];
                        }
                        if (ALL) {
                            *sf.at(i, 0) = gx;
                            *sf.at(i, 1) = gy;
                            *sf.at(i, 2) = gz;
                        } else {
                            *sf.at(i, 0) += gx;
                            *sf.at(i, 1) += gy;
                            *sf.at(i, 2) += gz;
                        }
                    }
                    __syncthreads();
                }
                warp_count(counter, cnt);
                return;
            }
        }
        if (LM == 1) return;   // list build: no force work
        if (gv.in_grid(cx, cy, cz)) {
            int c = gv.flat(cx, cy, cz);
            int s1 = gv.start[c], e1 = gv.start[c + 1];
            bool own = gv.owned(cx, cy, cz);
            for (int i0 = s1; i0 < e1; i0 += 32) {
                int i = i0 + lane;
                bool act = i < e1;
                double xi = 0.0, yi = 0.0, zi = 0.0;
                int ti = 0;
                if (act) sp.load(i, xi, yi, zi, ti);
                double fx = 0.0, fy = 0.0, fz = 0.0;
                int gk = 0;   // rounds met so far in this unit: warp w takes gk % WPU == w
                // four partners per round (independent loads and one batched
                // reciprocal, as in the Verlet walk), accumulated in order
                auto run = [&](int a, int b, bool counted, bool intra) {
                    for (int j0 = a; j0 < b; j0 += 4) {
                        if (WPU > 1 && (gk++ % WPU) != w) continue;
                        double dx[4], dy[4], dz[4], qq[4];
                        int tj[4];
                        bool ok[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            int j = min(j0 + u, b - 1);
                            double xj, yj, zj;
                            sp.load(j, xj, yj, zj, tj[u]);
                            dx[u] = xi - xj;
                            dy[u] = yi - yj;
                            dz[u] = zi - zj;
                            double r2 = dx[u] * dx[u] + dy[u] * dy[u] + dz[u] * dz[u];
                            ok[u] = act && j0 + u < b && (!intra || j0 + u != i) && r2 < tab.rc2;
                            qq[u] = ok[u] ? r2 : 1.0;
                        }
                        double p01 = qq[0] * qq[1], p23 = qq[2] * qq[3];
                        double y = fast_rcp(p01 * p23);
                        double y01 = y * p23, y23 = y * p01;
                        double inv[4] = {y01 * qq[1], y01 * qq[0], y23 * qq[3], y23 * qq[2]};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (ok[u]) {
                                double s2, e24;
                                lj_params<MT>(tab, ti, tj[u], s2, e24);
                                double aa = s2 * inv[u];
                                double a6 = aa * aa * aa;
                                double fs = (e24 * inv[u]) * (a6 * fma(2.0, a6, -1.0));
                                fx += fs * dx[u];
                                fy += fs * dy[u];
                                fz += fs * dz[u];
                                cnt += (N3L ? (counted && (!intra || j0 + u > i)) : 1) ? 1u : 0u;
                            }
                        }
                    }
                };
                if (beta == 0 && own) run(s1, e1, true, true);
                if (own)
                    for (int e = t1.start[beta]; e < t1.start[beta + 1]; ++e) {
                        int x2 = cx + t1.d[e][0], y2 = cy + t1.d[e][1], z2 = cz + t1.d[e][2];
                        if (!gv.in_grid(x2, y2, z2)) continue;
                        int c2 = gv.flat(x2, y2, z2);
                        run(gv.start[c2], gv.start[c2 + 1], true, false);
                    }
                for (int e = t2.start[beta]; e < t2.start[beta + 1]; ++e) {
                    int x1 = cx - t2.d[e][0], y1 = cy - t2.d[e][1], z1 = cz - t2.d[e][2];
                    if (!gv.in_grid(x1, y1, z1) || !gv.owned(x1, y1, z1)) continue;
                    int c1 = gv.flat(x1, y1, z1);
                    run(gv.start[c1], gv.start[c1 + 1], false, false);
                }
                if (WPU > 1) {   // the partials of the unit's warps, added in warp order
                    red[w][0][lane] = fx;
                    red[w][1][lane] = fy;
                    red[w][2][lane] = fz;
                    __syncthreads();
                    if (w == 0) {
                        fx = fy = fz = 0.0;
#pragma unroll
                        for (int q = 0; q < WPU; ++q) {
                            fx += red[q][0][lane];
                            fy += red[q][1][lane];
                            fz += red[q][2][lane];
                        }
                    }
                    __syncthreads();
                }
                if (act && w == 0) {
                    if (ALL) {
                        *sf.at(i, 0) = fx;
                        *sf.at(i, 1) = fy;
                        *sf.at(i, 2) = fz;
                    } else {
                        *sf.at(i, 0) += fx;
                        *sf.at(i, 1) += fy;
                        *sf.at(i, 2) += fz;
                    }
                }
            }
        }
    }
    warp_count(counter, cnt);
}

// scratch force = the colour partials added in colour order (C08All)
// (the partials are zeroed behind the read, ready for the next compute: no
// memset launch per step)
__global__ void c08_colour_sum_kernel(int64_t len, int ncol, double* __restrict__ cpart,
                                      double* __restrict__ sforce) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= len) return;
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = k < ncol ? cpart[(size_t)k * len + e] : 0.0;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (k < ncol) {
            s += v[k];
            cpart[(size_t)k * len + e] = 0.0;
        }
    sforce[e] = s;
}

// MDG_LC_C08_ALL: 1 (default) the small-system C08 runs every colour in one
// launch (C08All), 0 one launch per colour, 3 the colour partials added in the fold
static int lc_env_c08_all() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_LC_C08_ALL");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// MDG_LC_C08_LISTS: 1 (default) the one-launch C08 reads per-unit partner
// lists built once per grid rebuild (C08Lists), 0 looks the ranges up every step
static int lc_env_c08_lists() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_LC_C08_LISTS");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// warps per unit of the one-launch small-system C08 (2, 4, 8; MDG_LC_C08_ALL_WPU)
static int lc_env_c08_all_wpu() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_LC_C08_ALL_WPU");
        v = e ? atoi(e) : 4;
    }
    return v;
}

// warps per (anchor, block cell) unit of the small-system C08 kernel (1, 4, 8)
static int lc_env_c08_wpu() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_LC_C08_WPU");
        v = e ? atoi(e) : 8;
    }
    return v;
}

static int lc_env_rows() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_LC_ROWS");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// C08 realisation: 1 (default) per colour -- warp per (anchor, block cell)
// when a colour has fewer than 4 anchors per SM (small systems), else
// row-slot threads for sparse cells and warp tiles for dense ones; 0 warp
// tiles per colour always; 2 every anchor in one launch (row slots, fp64
// atomics, not run-to-run deterministic); 3 warp per (anchor, block cell)
// always
static int lc_env_c08() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_LC_C08");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// second = false: entries grouped by the block offset of their FIRST cell,
// max(0, -d); true: by that of their SECOND cell, max(0, d)
static C08Table make_c08_table(const Geom& g, const Stencil& fwd, bool second = false) {
    C08Table tb{};
    int nb = (g.overlap[0] + 1) * (g.overlap[1] + 1) * (g.overlap[2] + 1);
    int e = 0;
    for (int b = 0; b < nb; ++b) {
        int bi = b / ((g.overlap[1] + 1) * (g.overlap[2] + 1));
        int bj = (b / (g.overlap[2] + 1)) % (g.overlap[1] + 1), bk = b % (g.overlap[2] + 1);
        tb.start[b] = e;
        for (int k = 0; k < fwd.n; ++k) {
            const int* d = fwd.d[k];
            int o[3];
            for (int a = 0; a < 3; ++a) o[a] = second ? (d[a] > 0 ? d[a] : 0) : (d[a] < 0 ? -d[a] : 0);
            if (o[0] == bi && o[1] == bj && o[2] == bk) {
                for (int a = 0; a < 3; ++a) tb.d[e][a] = (signed char)d[a];
                ++e;
            }
        }
    }
    tb.start[nb] = e;
    return tb;
}

// row slots per unit: the power of two at or above the mean rows per unit (4..32)
static int slot_width(double rows_per_unit) {
    int S = 4;
    while (S < 32 && S < rows_per_unit) S <<= 1;
    return S;
}

// ------------------------------------------------------------------ dispatch

// too few anchors per colour to fill the GPU with anchor warps (small
// systems): the (anchor, block cell) unit kernel, deterministic
static bool lc_c08_cellwarp_applies(const Context& c, const Geom& g) {
    int64_t anchors_per_colour = (int64_t)g.D[0] * g.D[1] * g.D[2] /
                                 ((g.overlap[0] + 1) * (g.overlap[1] + 1) * (g.overlap[2] + 1));
    return lc_env_c08() == 3 || (lc_env_c08() == 1 && anchors_per_colour < 4 * c.sm_count);
}

// ... and all its colours in one launch (C08All)
static bool lc_c08_all_applies(const Context& c, const Grid& gr, int traversal) {
    const Geom& g = gr.g;
    const int nbc = (g.overlap[0] + 1) * (g.overlap[1] + 1) * (g.overlap[2] + 1);
    return traversal == T_C08 && lc_env_c08() != 2 && lc_c08_cellwarp_applies(c, g) && lc_env_c08_all() &&
           nbc <= 8;
}

template <int LAYOUT, bool MT>
static void lc_launch(Context& c, Grid& gr, int traversal, int newton3) {
    GridView gv = make_view(gr);
    ScratchPos<LAYOUT> sp{gr.spos4.p, gr.spos3.p, gr.spos3.p + gr.m, gr.spos3.p + 2 * gr.m,
                          gr.row_tid.p};
    ScratchForce<LAYOUT> sf{gr.sforce.p, (int)gr.m};
    unsigned long long* counter = c.scal.p;
    cudaStream_t s = c.stream;
    int m = (int)gr.m;
    const Geom& g = gr.g;
    if (traversal == T_C01) {
        lc_c01_kernel<LAYOUT, MT><<<blocks_for(m, 128), 128, 0, s>>>(gv, sp, sf, c.tab, gr.pruned, counter), note_launch();
        return;
    }
    if (traversal == T_SLI) {
        if (newton3)
            lc_fwd_atomic_kernel<LAYOUT, MT, true><<<blocks_for(m, 128), 128, 0, s>>>(gv, sp, sf, c.tab, gr.fwd_sli, counter), note_launch();
        else
            lc_fwd_atomic_kernel<LAYOUT, MT, false><<<blocks_for(m, 128), 128, 0, s>>>(gv, sp, sf, c.tab, gr.fwd_sli, counter), note_launch();
        return;
    }
    ColourLaunch cl;
    double rows_per_cell = (double)gr.m / (double)std::max<int64_t>(1, g.ncells);
    if ((traversal == T_C18 && lc_env_rows()) || (traversal == T_C08 && lc_env_c08() == 2)) {
        // every unit of every colour in one launch (the row kernels resolve the
        // write races with atomics, which is what the colours are for on a CPU)
        for (int k = 0; k < 3; ++k) {
            cl.p[k] = 0;
            cl.stride[k] = 1;
            cl.lo[k] = traversal == T_C18 ? g.H[k] : 0;
            cl.hi[k] = traversal == T_C18 ? g.H[k] + g.S[k] : g.D[k];
            cl.cnt[k] = cl.hi[k] - cl.lo[k];
        }
        int units = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
        if (traversal == T_C18) {
            int S = slot_width(rows_per_cell);
            int64_t threads = (int64_t)units * S;
            if (newton3)
                lc_c18_rows_kernel<LAYOUT, MT, true><<<blocks_for(threads, 128), 128, 0, s>>>(gv, sp, sf, c.tab, gr.fwd, cl, S, counter), note_launch();
            else
                lc_c18_rows_kernel<LAYOUT, MT, false><<<blocks_for(threads, 128), 128, 0, s>>>(gv, sp, sf, c.tab, gr.fwd, cl, S, counter), note_launch();
        } else {
            int block_cells = (g.overlap[0] + 1) * (g.overlap[1] + 1) * (g.overlap[2] + 1);
            C08Table tb = make_c08_table(g, gr.fwd);
            int S = slot_width(rows_per_cell * block_cells);
            int64_t threads = (int64_t)units * S;
            if (newton3)
                lc_c08_rows_kernel<LAYOUT, MT, true><<<blocks_for(threads, 128), 128, 0, s>>>(gv, sp, sf, c.tab, tb, cl, g.overlap[0], g.overlap[1], g.overlap[2], S, counter), note_launch();
            else
                lc_c08_rows_kernel<LAYOUT, MT, false><<<blocks_for(threads, 128), 128, 0, s>>>(gv, sp, sf, c.tab, tb, cl, g.overlap[0], g.overlap[1], g.overlap[2], S, counter), note_launch();
        }
        return;
    }
    if (traversal == T_C18) {
        int strides[3] = {g.overlap[0] + 1, 2 * g.overlap[1] + 1, 2 * g.overlap[2] + 1};
        for (int px = 0; px < strides[0]; ++px)
            for (int py = 0; py < strides[1]; ++py)
                for (int pz = 0; pz < strides[2]; ++pz) {
                    int ph[3] = {px, py, pz};
                    bool empty = false;
                    for (int k = 0; k < 3; ++k) {
                        cl.p[k] = ph[k];
                        cl.stride[k] = strides[k];
                        cl.lo[k] = g.H[k];
                        cl.hi[k] = g.H[k] + g.S[k];
                        int first = g.H[k] + ph[k];
                        cl.cnt[k] = first >= cl.hi[k] ? 0 : (cl.hi[k] - first + strides[k] - 1) / strides[k];
                        if (!cl.cnt[k]) empty = true;
                    }
                    if (empty) continue;
                    int warps = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
                    if (newton3)
                        lc_c18_kernel<LAYOUT, MT, true><<<blocks_for(warps, 4), 128, 0, s>>>(gv, sp, sf, c.tab, gr.fwd, cl, counter), note_launch();
                    else
                        lc_c18_kernel<LAYOUT, MT, false><<<blocks_for(warps, 4), 128, 0, s>>>(gv, sp, sf, c.tab, gr.fwd, cl, counter), note_launch();
                }
        return;
    }
    // C08: anchors over the whole padded grid, stride overlap+1 per axis
    // dense cells (CSF 1): warp tiles; sparse cells: row-slot threads
    bool c08_cells = lc_env_c08() == 1 && rows_per_cell < 8.0;
    bool c08_cellwarp = lc_c08_cellwarp_applies(c, g);
    C08Table c08t2 = make_c08_table(g, gr.fwd, true);
    C08Table c08tb = make_c08_table(g, gr.fwd);
    int strides[3] = {g.overlap[0] + 1, g.overlap[1] + 1, g.overlap[2] + 1};
    const int nbc = strides[0] * strides[1] * strides[2];
    const bool c08_all = lc_c08_all_applies(c, gr, traversal);
    C08All ca{};
    ca.ncol = 0;
    for (int px = 0; px < strides[0]; ++px)
        for (int py = 0; py < strides[1]; ++py)
            for (int pz = 0; pz < strides[2]; ++pz) {
                int ph[3] = {px, py, pz};
                bool empty = false;
                for (int k = 0; k < 3; ++k) {
                    cl.p[k] = ph[k];
                    cl.stride[k] = strides[k];
                    cl.lo[k] = 0;
                    cl.hi[k] = g.D[k];
                    cl.cnt[k] = ph[k] >= g.D[k] ? 0 : (g.D[k] - ph[k] + strides[k] - 1) / strides[k];
                    if (!cl.cnt[k]) empty = true;
                }
                if (empty) continue;
                int warps = cl.cnt[0] * cl.cnt[1] * cl.cnt[2];
                if (c08_all) {   // collected, one launch below
                    ca.cl[ca.ncol] = cl;
                    ca.ustart[ca.ncol + 1] = ca.ustart[ca.ncol] + warps * nbc;
                    ++ca.ncol;
                } else if (c08_cellwarp) {
                    int nb = (g.overlap[0] + 1) * (g.overlap[1] + 1) * (g.overlap[2] + 1);
                    int64_t units = (int64_t)warps * nb;
                    int wpu = lc_env_c08_wpu();
#define MDG_C08W(N3, W) lc_c08_cellwarp_kernel<LAYOUT, MT, N3, W><<<W == 1 ? blocks_for(units * 32, 128) : (unsigned)units, W == 1 ? 128 : 32 * W, 0, s>>>(gv, sp, sf, c.tab, c08tb, c08t2, cl, g.overlap[0], g.overlap[1], g.overlap[2], counter), note_launch()
                    if (newton3) {
                        if (wpu >= 8) MDG_C08W(true, 8); else if (wpu >= 4) MDG_C08W(true, 4); else MDG_C08W(true, 1);
                    } else {
                        if (wpu >= 8) MDG_C08W(false, 8); else if (wpu >= 4) MDG_C08W(false, 4); else MDG_C08W(false, 1);
                    }
#undef MDG_C08W
                } else if (c08_cells) {
                    int nb = (g.overlap[0] + 1) * (g.overlap[1] + 1) * (g.overlap[2] + 1);
                    int S = slot_width(rows_per_cell);
                    int64_t threads = (int64_t)warps * nb * S;
                    if (newton3)
                        lc_c08_cells_kernel<LAYOUT, MT, true><<<blocks_for(threads, 128), 128, 0, s>>>(gv, sp, sf, c.tab, c08tb, cl, g.overlap[0], g.overlap[1], g.overlap[2], S, counter), note_launch();
                    else
                        lc_c08_cells_kernel<LAYOUT, MT, false><<<blocks_for(threads, 128), 128, 0, s>>>(gv, sp, sf, c.tab, c08tb, cl, g.overlap[0], g.overlap[1], g.overlap[2], S, counter), note_launch();
                } else if (newton3)
                    lc_c08_kernel<LAYOUT, MT, true><<<blocks_for(warps, 4), 128, 0, s>>>(gv, sp, sf, c.tab, gr.fwd, cl, counter), note_launch();
                else
                    lc_c08_kernel<LAYOUT, MT, false><<<blocks_for(warps, 4), 128, 0, s>>>(gv, sp, sf, c.tab, gr.fwd, cl, counter), note_launch();
            }
    if (c08_all && ca.ncol > 0) {
        const size_t len = 3 * (size_t)m;
        const double* before = gr.cpart.p;
        gr.cpart.ensure(len * ca.ncol + 1);
        if (!gr.cpart.p) return;   // out of memory: no forces (the caller's status check reports it)
        if (gr.cpart.p != before) gr.cpart_zero = 0;
        // the sum pass leaves the partials zeroed; the fold-fused variant does not
        if (gr.cpart_zero < len * ca.ncol || lc_env_c08_all() == 3) {
            cudaMemsetAsync(gr.cpart.p, 0, len * ca.ncol * sizeof(double), s);
            gr.cpart_zero = len * ca.ncol;
        }
        const unsigned units = (unsigned)ca.ustart[ca.ncol];
        const int wpu = lc_env_c08_all_wpu();
        // the units' staged partner lists, once per grid build
        C08Lists ul{};
        bool lists = lc_env_c08_lists() != 0;
        if (lists) {
            gr.c08l_tot.ensure(units + 1);
            gr.c08l_j.ensure((size_t)units * kC08Stage + 1);
            gr.c08l_f.ensure((size_t)units * kC08Stage + 1);
            lists = gr.c08l_tot.p && gr.c08l_j.p && gr.c08l_f.p;
            ul = C08Lists{gr.c08l_tot.p, gr.c08l_j.p, gr.c08l_f.p};
        }
        if (lists && gr.c08l_for != gr.build_id) {
#define MDG_C08L(W) lc_c08_cellwarp_kernel<LAYOUT, MT, true, W, true, 1><<<units, 32 * W, 0, s>>>(gv, sp, sf, c.tab, c08tb, c08t2, cl, g.overlap[0], g.overlap[1], g.overlap[2], counter, ca, gr.cpart.p, ul), note_launch()
            if (wpu >= 8) MDG_C08L(8); else if (wpu >= 4) MDG_C08L(4); else MDG_C08L(2);
#undef MDG_C08L
            gr.c08l_for = gr.build_id;
        }
#define MDG_C08A(N3, W, LM) lc_c08_cellwarp_kernel<LAYOUT, MT, N3, W, true, LM><<<units, 32 * W, 0, s>>>(gv, sp, sf, c.tab, c08tb, c08t2, cl, g.overlap[0], g.overlap[1], g.overlap[2], counter, ca, gr.cpart.p, ul), note_launch()
        if (lists) {
            if (newton3) {
                if (wpu >= 8) MDG_C08A(true, 8, 2); else if (wpu >= 4) MDG_C08A(true, 4, 2); else MDG_C08A(true, 2, 2);
            } else {
                if (wpu >= 8) MDG_C08A(false, 8, 2); else if (wpu >= 4) MDG_C08A(false, 4, 2); else MDG_C08A(false, 2, 2);
            }
        } else {
            if (newton3) {
                if (wpu >= 8) MDG_C08A(true, 8, 0); else if (wpu >= 4) MDG_C08A(true, 4, 0); else MDG_C08A(true, 2, 0);
            } else {
                if (wpu >= 8) MDG_C08A(false, 8, 0); else if (wpu >= 4) MDG_C08A(false, 4, 0); else MDG_C08A(false, 2, 0);
            }
        }
#undef MDG_C08A
        // the colour sums as their own element-parallel pass (the fold then
        // runs as for every LC traversal): measured faster than adding the
        // partials inside the fold, whose thread-per-particle chains of
        // dependent image loads then carry 8 loads per row (5.5 + 2.1 us
        // against 16.7 us at BASELINE config 1)
        if (lc_env_c08_all() == 3) {
            gr.cpart_ncol = ca.ncol;   // the fold adds the partials
            gr.cpart_zero = 0;
        }
        else
            c08_colour_sum_kernel<<<blocks_for((int64_t)len, 256), 256, 0, s>>>((int64_t)len, ca.ncol, gr.cpart.p, gr.sforce.p), note_launch();
    }
}

// ---------------------------------------------------------------- pair export
//
// The set of pairs every LC traversal evaluates within rc on this grid (the
// reference's r^2 < rc^2 on pos[src] + shift, kernels.py:36-40), as owner
// pairs (src_i, src_j) with src_i < src_j: a thread per owned row walks its own
// cell and the full pruned stencil (each unordered owner pair is met from at
// least one side).  Parity export only.
__global__ void lc_pairs_kernel(GridView gv, const double4* __restrict__ spos, const int* __restrict__ src,
                                Stencil st, double rc2, unsigned long long* counter, int2* out,
                                long long cap) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= gv.m) return;
    int cell = gv.row_cell[r], cx, cy, cz;
    gv.decode(cell, cx, cy, cz);
    if (!gv.owned(cx, cy, cz)) return;
    double4 pi = spos[r];
    int si = src[r];
    auto visit = [&](int j) {
        if (j == r) return;
        int sj = src[j];
        if (sj <= si) return;
        double4 pj = spos[j];
        double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
        if (dx * dx + dy * dy + dz * dz < rc2) {
            unsigned long long k = atomicAdd(counter, 1ull);
            if (out && (long long)k < cap) out[k] = make_int2(si, sj);
        }
    };
    for (int j = gv.start[cell]; j < gv.start[cell + 1]; ++j) visit(j);
    for (int k = 0; k < st.n; ++k) {
        int x2 = cx + st.d[k][0], y2 = cy + st.d[k][1], z2 = cz + st.d[k][2];
        if (!gv.in_grid(x2, y2, z2)) continue;
        int c2 = gv.flat(x2, y2, z2);
        for (int j = gv.start[c2]; j < gv.start[c2 + 1]; ++j) visit(j);
    }
}

int lc_pairs(Context& c, Grid& gr, long long cap, int2* dev_out, long long* count) {
    grid_bind_scratch(c, gr, AOS);
    grid_refresh(c, gr, AOS);
    unsigned long long* counter = c.scal.p + 4;
    if (cudaMemsetAsync(counter, 0, sizeof(unsigned long long), c.stream) != cudaSuccess) return -1;
    if (gr.m > 0)
        lc_pairs_kernel<<<blocks_for(gr.m, 128), 128, 0, c.stream>>>(make_view(gr), gr.spos4.p, gr.row_src.p,
                                                                     gr.pruned, c.tab.rc2, counter, dev_out, cap), note_launch();
    unsigned long long h = 0;
    if (cudaMemcpyAsync(&h, counter, sizeof(h), cudaMemcpyDeviceToHost, c.stream) != cudaSuccess ||
        cudaStreamSynchronize(c.stream) != cudaSuccess)
        return -1;
    *count = (long long)h;
    return 0;
}

void lc_compute(Context& c, Grid& gr, int traversal, int newton3, int layout) {
    gr.cpart_ncol = 0;
    if (gr.m == 0) return;
    if (traversal != T_C01 && !lc_c08_all_applies(c, gr, traversal))
        cudaMemsetAsync(gr.sforce.p, 0, 3 * (size_t)gr.m * sizeof(double), c.stream);
    bool mt = c.tab.T > 1;
    c.prof_mark();
    if (layout == AOS) {
        if (mt) lc_launch<AOS, true>(c, gr, traversal, newton3);
        else lc_launch<AOS, false>(c, gr, traversal, newton3);
    } else {
        if (mt) lc_launch<SOA, true>(c, gr, traversal, newton3);
        else lc_launch<SOA, false>(c, gr, traversal, newton3);
    }
    c.prof_mark();
}

}  // namespace mdg
