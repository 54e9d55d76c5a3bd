/*
 * ORACLE / TEST INFRASTRUCTURE — not product code.
 *
 * CPU restatement, in plain C, of the reference's numba pair kernels
 * (/root/reference/pkg/src/mdtune/kernels.py).  Only tests/, bench.py's
 * cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load
 * this library, and only as the checker or the timed CPU baseline.
 *
 * Arithmetic follows the reference expression by expression and the file is
 * compiled with -ffp-contract=off (numba/LLVM does not contract without
 * fastmath), so results reproduce the numba kernels bit for bit on the same
 * inputs.  Every entry point releases nothing and allocates nothing; callers
 * (oracle/port.py) run them from a thread pool exactly like the reference's
 * Workforce does with its GIL-free numba kernels (containers.py:50-73).
 *
 * Layout: positions/forces are addressed as P[i*si + k*sk]; AoS (M,3) has
 * si=3, sk=1 and SoA (3,M) has si=1, sk=M (particles.py:31-98).
 * Type tables are T x T row-major (forces.py:12-22).
 */
#include <math.h>
#include <stdint.h>

typedef int64_t i64;

#define PX(p, i) (p)[(i) * si]
#define PY(p, i) (p)[(i) * si + sk]
#define PZ(p, i) (p)[(i) * si + 2 * sk]

/* LJ scalar: kernels.py:41-45 (fs = eps24*(2 a6 a6 - a6)*inv). */
static inline double lj_scalar(double r2, double s2, double e24) {
    double inv = 1.0 / r2;
    double a = s2 * inv;
    double a6 = a * a * a;
    return e24 * (2.0 * a6 * a6 - a6) * inv;
}

/* Cell-pair block with Newton-3 writes: kernels.py:24-56 / :187-225. */
static i64 pair_n3l(const double* pos, double* f, i64 si, i64 sk,
                    const i64* tid, const double* sig2, const double* eps24,
                    i64 T, double rc2, i64 s1, i64 e1, i64 s2, i64 e2) {
    i64 count = 0;
    for (i64 i = s1; i < e1; ++i) {
        double xi = PX(pos, i), yi = PY(pos, i), zi = PZ(pos, i);
        i64 ti = tid[i];
        double fxi = 0.0, fyi = 0.0, fzi = 0.0;
        for (i64 j = s2; j < e2; ++j) {
            double dx = xi - PX(pos, j);
            double dy = yi - PY(pos, j);
            double dz = zi - PZ(pos, j);
            double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 < rc2) {
                i64 tj = tid[j];
                double fs = lj_scalar(r2, sig2[ti * T + tj], eps24[ti * T + tj]);
                count += 1;
                fxi += fs * dx;
                fyi += fs * dy;
                fzi += fs * dz;
                PX(f, j) -= fs * dx;
                PY(f, j) -= fs * dy;
                PZ(f, j) -= fs * dz;
            }
        }
        PX(f, i) += fxi;
        PY(f, i) += fyi;
        PZ(f, i) += fzi;
    }
    return count;
}

/* Both directions evaluated separately: kernels.py:59-102 / :228-276. */
static i64 pair_no3(const double* pos, double* f, i64 si, i64 sk,
                    const i64* tid, const double* sig2, const double* eps24,
                    i64 T, double rc2, i64 s1, i64 e1, i64 s2, i64 e2) {
    i64 count = 0;
    for (i64 i = s1; i < e1; ++i) {
        double xi = PX(pos, i), yi = PY(pos, i), zi = PZ(pos, i);
        i64 ti = tid[i];
        double fxi = 0.0, fyi = 0.0, fzi = 0.0;
        for (i64 j = s2; j < e2; ++j) {
            double dx = xi - PX(pos, j);
            double dy = yi - PY(pos, j);
            double dz = zi - PZ(pos, j);
            double r2 = dx * dx + dy * dy + dz * dz;
            i64 tj = tid[j];
            if (r2 < rc2) {
                double fs = lj_scalar(r2, sig2[ti * T + tj], eps24[ti * T + tj]);
                count += 1;
                fxi += fs * dx;
                fyi += fs * dy;
                fzi += fs * dz;
            }
            double bx = PX(pos, j) - xi;
            double by = PY(pos, j) - yi;
            double bz = PZ(pos, j) - zi;
            double q2 = bx * bx + by * by + bz * bz;
            if (q2 < rc2) {
                double gs = lj_scalar(q2, sig2[tj * T + ti], eps24[tj * T + ti]);
                count += 1;
                PX(f, j) += gs * bx;
                PY(f, j) += gs * by;
                PZ(f, j) += gs * bz;
            }
        }
        PX(f, i) += fxi;
        PY(f, i) += fyi;
        PZ(f, i) += fzi;
    }
    return count;
}

/* Same-cell pairs j > i: kernels.py:105-182 / :279-368. */
static i64 intra_n3l(const double* pos, double* f, i64 si, i64 sk,
                     const i64* tid, const double* sig2, const double* eps24,
                     i64 T, double rc2, i64 s, i64 e) {
    i64 count = 0;
    for (i64 i = s; i < e; ++i) {
        double xi = PX(pos, i), yi = PY(pos, i), zi = PZ(pos, i);
        i64 ti = tid[i];
        double fxi = 0.0, fyi = 0.0, fzi = 0.0;
        for (i64 j = i + 1; j < e; ++j) {
            double dx = xi - PX(pos, j);
            double dy = yi - PY(pos, j);
            double dz = zi - PZ(pos, j);
            double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 < rc2) {
                i64 tj = tid[j];
                double fs = lj_scalar(r2, sig2[ti * T + tj], eps24[ti * T + tj]);
                count += 1;
                fxi += fs * dx;
                fyi += fs * dy;
                fzi += fs * dz;
                PX(f, j) -= fs * dx;
                PY(f, j) -= fs * dy;
                PZ(f, j) -= fs * dz;
            }
        }
        PX(f, i) += fxi;
        PY(f, i) += fyi;
        PZ(f, i) += fzi;
    }
    return count;
}

static i64 intra_no3(const double* pos, double* f, i64 si, i64 sk,
                     const i64* tid, const double* sig2, const double* eps24,
                     i64 T, double rc2, i64 s, i64 e) {
    i64 count = 0;
    for (i64 i = s; i < e; ++i) {
        double xi = PX(pos, i), yi = PY(pos, i), zi = PZ(pos, i);
        i64 ti = tid[i];
        double fxi = 0.0, fyi = 0.0, fzi = 0.0;
        for (i64 j = i + 1; j < e; ++j) {
            double dx = xi - PX(pos, j);
            double dy = yi - PY(pos, j);
            double dz = zi - PZ(pos, j);
            double r2 = dx * dx + dy * dy + dz * dz;
            i64 tj = tid[j];
            if (r2 < rc2) {
                double fs = lj_scalar(r2, sig2[ti * T + tj], eps24[ti * T + tj]);
                count += 1;
                fxi += fs * dx;
                fyi += fs * dy;
                fzi += fs * dz;
            }
            double bx = PX(pos, j) - xi;
            double by = PY(pos, j) - yi;
            double bz = PZ(pos, j) - zi;
            double q2 = bx * bx + by * by + bz * bz;
            if (q2 < rc2) {
                double gs = lj_scalar(q2, sig2[tj * T + ti], eps24[tj * T + ti]);
                count += 1;
                PX(f, j) += gs * bx;
                PY(f, j) += gs * by;
                PZ(f, j) += gs * bz;
            }
        }
        PX(f, i) += fxi;
        PY(f, i) += fyi;
        PZ(f, i) += fzi;
    }
    return count;
}

#define FLAT(x, y, z) (((x) * ny + (y)) * nz + (z))
#define IN_GRID(x, y, z) (0 <= (x) && (x) < nx && 0 <= (y) && (y) < ny && 0 <= (z) && (z) < nz)

/* C08 anchor sweep for one colour: kernels.py:373-433 (AoS) / :436-488 (SoA). */
i64 ljp_c08_sweep(const double* pos, double* f, i64 si, i64 sk, const i64* tid,
                  const i64* start, const i64* end, const double* sig2,
                  const double* eps24, i64 T, double rc2, i64 nx, i64 ny, i64 nz,
                  i64 olx, i64 oly, i64 olz, i64 ohx, i64 ohy, i64 ohz,
                  const i64* deltas, i64 nd, i64 sx, i64 sy, i64 sz, i64 py,
                  i64 pz, i64 x_begin, i64 x_end, int newton3) {
    i64 count = 0;
    for (i64 ax = x_begin; ax < x_end; ax += sx)
        for (i64 ay = py; ay < ny; ay += sy)
            for (i64 az = pz; az < nz; az += sz) {
                if (olx <= ax && ax < ohx && oly <= ay && ay < ohy && olz <= az && az < ohz) {
                    i64 c = FLAT(ax, ay, az);
                    i64 s = start[c], e = end[c];
                    if (e - s > 1)
                        count += newton3 ? intra_n3l(pos, f, si, sk, tid, sig2, eps24, T, rc2, s, e)
                                         : intra_no3(pos, f, si, sk, tid, sig2, eps24, T, rc2, s, e);
                }
                for (i64 k = 0; k < nd; ++k) {
                    i64 dx = deltas[3 * k], dy = deltas[3 * k + 1], dz = deltas[3 * k + 2];
                    i64 c1x = dx < 0 ? ax - dx : ax;
                    i64 c1y = dy < 0 ? ay - dy : ay;
                    i64 c1z = dz < 0 ? az - dz : az;
                    i64 c2x = c1x + dx, c2y = c1y + dy, c2z = c1z + dz;
                    if (!(olx <= c1x && c1x < ohx && oly <= c1y && c1y < ohy && olz <= c1z && c1z < ohz))
                        continue;
                    if (!IN_GRID(c2x, c2y, c2z)) continue;
                    i64 c1 = FLAT(c1x, c1y, c1z), c2 = FLAT(c2x, c2y, c2z);
                    i64 s1 = start[c1], e1 = end[c1];
                    if (e1 <= s1) continue;
                    i64 s2 = start[c2], e2 = end[c2];
                    if (e2 <= s2) continue;
                    count += newton3 ? pair_n3l(pos, f, si, sk, tid, sig2, eps24, T, rc2, s1, e1, s2, e2)
                                     : pair_no3(pos, f, si, sk, tid, sig2, eps24, T, rc2, s1, e1, s2, e2);
                }
            }
    return count;
}

/* Forward base sweep (C18 colours, SLI layers): kernels.py:493-579. */
i64 ljp_fwd_sweep(const double* pos, double* f, i64 si, i64 sk, const i64* tid,
                  const i64* start, const i64* end, const double* sig2,
                  const double* eps24, i64 T, double rc2, i64 nx, i64 ny, i64 nz,
                  const i64* deltas, i64 nd, i64 x0, i64 x1, i64 sx, i64 y0,
                  i64 y1, i64 sy, i64 z0, i64 z1, i64 sz, int newton3) {
    i64 count = 0;
    for (i64 bx = x0; bx < x1; bx += sx)
        for (i64 by = y0; by < y1; by += sy)
            for (i64 bz = z0; bz < z1; bz += sz) {
                i64 c1 = FLAT(bx, by, bz);
                i64 s1 = start[c1], e1 = end[c1];
                if (e1 <= s1) continue;
                if (e1 - s1 > 1)
                    count += newton3 ? intra_n3l(pos, f, si, sk, tid, sig2, eps24, T, rc2, s1, e1)
                                     : intra_no3(pos, f, si, sk, tid, sig2, eps24, T, rc2, s1, e1);
                for (i64 k = 0; k < nd; ++k) {
                    i64 c2x = bx + deltas[3 * k], c2y = by + deltas[3 * k + 1], c2z = bz + deltas[3 * k + 2];
                    if (!IN_GRID(c2x, c2y, c2z)) continue;
                    i64 c2 = FLAT(c2x, c2y, c2z);
                    i64 s2 = start[c2], e2 = end[c2];
                    if (e2 <= s2) continue;
                    count += newton3 ? pair_n3l(pos, f, si, sk, tid, sig2, eps24, T, rc2, s1, e1, s2, e2)
                                     : pair_no3(pos, f, si, sk, tid, sig2, eps24, T, rc2, s1, e1, s2, e2);
                }
            }
    return count;
}

/* C01 directed sweep, writes only base rows: kernels.py:584-725. */
i64 ljp_directed_sweep(const double* pos, double* f, i64 si, i64 sk, const i64* tid,
                       const i64* start, const i64* end, const double* sig2,
                       const double* eps24, i64 T, double rc2, i64 nx, i64 ny,
                       i64 nz, const i64* deltas, i64 nd, i64 x0, i64 x1, i64 y0,
                       i64 y1, i64 z0, i64 z1) {
    i64 count = 0;
    for (i64 bx = x0; bx < x1; ++bx)
        for (i64 by = y0; by < y1; ++by)
            for (i64 bz = z0; bz < z1; ++bz) {
                i64 c1 = FLAT(bx, by, bz);
                i64 s1 = start[c1], e1 = end[c1];
                if (e1 <= s1) continue;
                for (i64 i = s1; i < e1; ++i) {
                    double xi = PX(pos, i), yi = PY(pos, i), zi = PZ(pos, i);
                    i64 ti = tid[i];
                    double fxi = 0.0, fyi = 0.0, fzi = 0.0;
                    for (i64 j = s1; j < e1; ++j) {
                        if (j == i) continue;
                        double dx = xi - PX(pos, j), dy = yi - PY(pos, j), dz = zi - PZ(pos, j);
                        double r2 = dx * dx + dy * dy + dz * dz;
                        if (r2 < rc2) {
                            i64 tj = tid[j];
                            double fs = lj_scalar(r2, sig2[ti * T + tj], eps24[ti * T + tj]);
                            count += 1;
                            fxi += fs * dx;
                            fyi += fs * dy;
                            fzi += fs * dz;
                        }
                    }
                    for (i64 k = 0; k < nd; ++k) {
                        i64 c2x = bx + deltas[3 * k], c2y = by + deltas[3 * k + 1], c2z = bz + deltas[3 * k + 2];
                        if (!IN_GRID(c2x, c2y, c2z)) continue;
                        i64 c2 = FLAT(c2x, c2y, c2z);
                        for (i64 j = start[c2]; j < end[c2]; ++j) {
                            double dx = xi - PX(pos, j), dy = yi - PY(pos, j), dz = zi - PZ(pos, j);
                            double r2 = dx * dx + dy * dy + dz * dz;
                            if (r2 < rc2) {
                                i64 tj = tid[j];
                                double fs = lj_scalar(r2, sig2[ti * T + tj], eps24[ti * T + tj]);
                                count += 1;
                                fxi += fs * dx;
                                fyi += fs * dy;
                                fzi += fs * dz;
                            }
                        }
                    }
                    PX(f, i) += fxi;
                    PY(f, i) += fyi;
                    PZ(f, i) += fzi;
                }
            }
    return count;
}

/* Verlet-list forces with minimum image: kernels.py:730-818. */
i64 ljp_vl_force(const double* pos, double* f, i64 si, i64 sk, const i64* tid,
                 const i64* nbr, const i64* noff, i64 i_begin, i64 i_end,
                 const double* sig2, const double* eps24, i64 T, double rc2,
                 double lx, double ly, double lz, double mx, double my, double mz) {
    i64 count = 0;
    double inv_lx = 1.0 / lx, inv_ly = 1.0 / ly, inv_lz = 1.0 / lz;
    for (i64 i = i_begin; i < i_end; ++i) {
        double xi = PX(pos, i), yi = PY(pos, i), zi = PZ(pos, i);
        i64 ti = tid[i];
        double fxi = 0.0, fyi = 0.0, fzi = 0.0;
        for (i64 k = noff[i]; k < noff[i + 1]; ++k) {
            i64 j = nbr[k];
            double dx = xi - PX(pos, j), dy = yi - PY(pos, j), dz = zi - PZ(pos, j);
            dx -= mx * lx * rint(dx * inv_lx);
            dy -= my * ly * rint(dy * inv_ly);
            dz -= mz * lz * rint(dz * inv_lz);
            double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 < rc2) {
                i64 tj = tid[j];
                double fs = lj_scalar(r2, sig2[ti * T + tj], eps24[ti * T + tj]);
                count += 1;
                fxi += fs * dx;
                fyi += fs * dy;
                fzi += fs * dz;
            }
        }
        PX(f, i) += fxi;
        PY(f, i) += fyi;
        PZ(f, i) += fzi;
    }
    return count;
}

/* Verlet-list CSR passes over the CSF-1 grid (AoS scratch positions):
 * count kernels.py:823-864, fill :867-910.  fill==0 -> count pass. */
static void vl_pass(const double* pos, const i64* owner, const i64* start,
                    const i64* end, double ell2, i64 nx, i64 ny, i64 nz,
                    const i64* deltas, i64 nd, i64 olx, i64 oly, i64 olz,
                    i64 ohx, i64 ohy, i64 ohz, i64* counts_or_cursor,
                    i64* nbr, int fill) {
    const i64 si = 3, sk = 1;
    for (i64 bx = olx; bx < ohx; ++bx)
        for (i64 by = oly; by < ohy; ++by)
            for (i64 bz = olz; bz < ohz; ++bz) {
                i64 c1 = FLAT(bx, by, bz);
                i64 s1 = start[c1], e1 = end[c1];
                if (e1 <= s1) continue;
                for (i64 i = s1; i < e1; ++i) {
                    double xi = PX(pos, i), yi = PY(pos, i), zi = PZ(pos, i);
                    i64 oi = owner[i];
                    i64 c = fill ? counts_or_cursor[oi] : 0;
                    for (i64 j = s1; j < e1; ++j) {
                        if (j == i) continue;
                        double dx = xi - PX(pos, j), dy = yi - PY(pos, j), dz = zi - PZ(pos, j);
                        if (dx * dx + dy * dy + dz * dz <= ell2) {
                            if (fill) nbr[c] = owner[j];
                            c += 1;
                        }
                    }
                    for (i64 k = 0; k < nd; ++k) {
                        i64 c2x = bx + deltas[3 * k], c2y = by + deltas[3 * k + 1], c2z = bz + deltas[3 * k + 2];
                        if (!IN_GRID(c2x, c2y, c2z)) continue;
                        i64 c2 = FLAT(c2x, c2y, c2z);
                        for (i64 j = start[c2]; j < end[c2]; ++j) {
                            double dx = xi - PX(pos, j), dy = yi - PY(pos, j), dz = zi - PZ(pos, j);
                            if (dx * dx + dy * dy + dz * dz <= ell2) {
                                if (fill) nbr[c] = owner[j];
                                c += 1;
                            }
                        }
                    }
                    if (fill) counts_or_cursor[oi] = c;
                    else counts_or_cursor[oi] += c;
                }
            }
}

void ljp_vl_count_pairs(const double* pos, const i64* owner, const i64* start,
                        const i64* end, double ell2, i64 nx, i64 ny, i64 nz,
                        const i64* deltas, i64 nd, i64 olx, i64 oly, i64 olz,
                        i64 ohx, i64 ohy, i64 ohz, i64* counts) {
    vl_pass(pos, owner, start, end, ell2, nx, ny, nz, deltas, nd, olx, oly, olz,
            ohx, ohy, ohz, counts, 0, 0);
}

void ljp_vl_fill_pairs(const double* pos, const i64* owner, const i64* start,
                       const i64* end, double ell2, i64 nx, i64 ny, i64 nz,
                       const i64* deltas, i64 nd, i64 olx, i64 oly, i64 olz,
                       i64 ohx, i64 ohy, i64 ohz, i64* cursor, i64* nbr) {
    vl_pass(pos, owner, start, end, ell2, nx, ny, nz, deltas, nd, olx, oly, olz,
            ohx, ohy, ohz, cursor, nbr, 1);
}

/*
 * Brute-force check of selected rows (the reference's O(N^2) test oracle,
 * tests/conftest.py:22-44 / port.brute_forces), accelerated only by a cell
 * list of side >= rc so BASELINE-size systems (up to 67 M particles) can be
 * checked on sampled rows.  ljp_cell_list links every particle into its cell
 * (head: ncell entries, next: n entries; pos AoS).  ljp_sampled_forces: for
 * rows[q], q in [q0, q1), the sum over every j != i with minimum-image
 * (d -= L rint(d/L) on periodic axes, kernels.py:739-757) r2 < rc2 (strict,
 * kernels.py:40) of the LJ force (kernels.py:41-45, mixing forces.py:12-22),
 * and the number of such j.  Periodic axes with fewer than 3 cells visit
 * each cell once.  GIL-free: port.sampled_forces runs row ranges on threads.
 */
static void cell_dims(const double* L, double rc, i64* nc, double* cl) {
    for (int k = 0; k < 3; ++k) {
        nc[k] = (i64)floor(L[k] / rc);
        if (nc[k] < 1) nc[k] = 1;
        cl[k] = L[k] / (double)nc[k];
    }
}

static void cell_of(const double* p, const i64* nc, const double* cl, i64* c) {
    for (int k = 0; k < 3; ++k) {
        c[k] = (i64)floor(p[k] / cl[k]);
        if (c[k] < 0) c[k] = 0;
        if (c[k] >= nc[k]) c[k] = nc[k] - 1;
    }
}

void ljp_cell_list(const double* pos, i64 n, const double* L, double rc, i64* head, i64* next) {
    i64 nc[3];
    double cl[3];
    cell_dims(L, rc, nc, cl);
    for (i64 c = 0; c < nc[0] * nc[1] * nc[2]; ++c) head[c] = -1;
    for (i64 i = n - 1; i >= 0; --i) {
        i64 c[3];
        cell_of(pos + 3 * i, nc, cl, c);
        i64 f = (c[0] * nc[1] + c[1]) * nc[2] + c[2];
        next[i] = head[f];
        head[f] = i;
    }
}

void ljp_sampled_forces(const double* pos, const i64* tid, const double* sig2,
                        const double* eps24, i64 T, const double* L, const i64* per,
                        double rc, const i64* head, const i64* next, const i64* rows,
                        i64 q0, i64 q1, double* fout, i64* cout) {
    i64 nc[3];
    double cl[3];
    cell_dims(L, rc, nc, cl);
    const double rc2 = rc * rc;
    for (i64 q = q0; q < q1; ++q) {
        i64 i = rows[q];
        double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        i64 ci[3], lo[3], hi[3];
        cell_of(pos + 3 * i, nc, cl, ci);
        for (int k = 0; k < 3; ++k) {
            if (per[k] && nc[k] < 3) { lo[k] = 0; hi[k] = nc[k] - 1; }
            else { lo[k] = ci[k] - 1; hi[k] = ci[k] + 1; }
        }
        double fx = 0.0, fy = 0.0, fz = 0.0;
        i64 cnt = 0;
        for (i64 a = lo[0]; a <= hi[0]; ++a)
            for (i64 b = lo[1]; b <= hi[1]; ++b)
                for (i64 e = lo[2]; e <= hi[2]; ++e) {
                    i64 cc[3] = {a, b, e};
                    int skip = 0;
                    for (int k = 0; k < 3; ++k) {
                        if (cc[k] < 0 || cc[k] >= nc[k]) {
                            if (!per[k]) { skip = 1; break; }
                            cc[k] = (cc[k] + nc[k]) % nc[k];
                        }
                    }
                    if (skip) continue;
                    for (i64 j = head[(cc[0] * nc[1] + cc[1]) * nc[2] + cc[2]]; j >= 0; j = next[j]) {
                        if (j == i) continue;
                        double d[3] = {xi - pos[3 * j], yi - pos[3 * j + 1], zi - pos[3 * j + 2]};
                        for (int k = 0; k < 3; ++k)
                            if (per[k]) d[k] -= L[k] * rint(d[k] / L[k]);
                        double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
                        if (r2 < rc2) {
                            i64 tt = tid ? tid[i] * T + tid[j] : 0;
                            double fs = lj_scalar(r2, sig2[tt], eps24[tt]);
                            fx += fs * d[0];
                            fy += fs * d[1];
                            fz += fs * d[2];
                            ++cnt;
                        }
                    }
                }
        fout[3 * q] = fx;
        fout[3 * q + 1] = fy;
        fout[3 * q + 2] = fz;
        cout[q] = cnt;
    }
}
