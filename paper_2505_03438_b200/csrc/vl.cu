// Verlet lists: CSR build over the CSF-1 grid and the per-particle list walk.
//
// Reference: VerletListState (containers.py:343-375), vl_count_pairs /
// vl_fill_pairs (kernels.py:823-910), vl_force_aos/_soa (kernels.py:730-818).
// The list content and order are the reference's: for each owner particle,
// partners with r^2 <= (rc+skin)^2 (non-strict) from its own cell (j != i)
// then the pruned stencil cells in stencil order, stored as owner indices.
// Entries are int32 (owner indices), offsets int64.
#include "device.cuh"

namespace mdg {

// One thread per owned row of the build grid; FILL=false counts, FILL=true
// writes at noff[owner].
template <bool FILL>
__global__ void __launch_bounds__(128) vl_build_kernel(GridView gv, const double4* __restrict__ bpos,
                                                       const int* __restrict__ row_src, Stencil st,
                                                       double ell2, int* __restrict__ counts,
                                                       const long long* __restrict__ noff,
                                                       int* __restrict__ nbr) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= gv.m) return;
    int cell = gv.row_cell[r], cx, cy, cz;
    gv.decode(cell, cx, cy, cz);
    if (!gv.owned(cx, cy, cz)) return;
    double4 pi = bpos[r];
    int oi = row_src[r];
    long long out = FILL ? noff[oi] : 0;
    int c = 0;
    auto visit = [&](int j) {
        double4 pj = bpos[j];
        double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
        if (dx * dx + dy * dy + dz * dz <= ell2) {
            if (FILL) nbr[out + c] = row_src[j];
            ++c;
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
    if (!FILL) counts[oi] = c;
}

int vl_rebuild(Context& c) {
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    if (grid_rebuild(c, gr, c.pos, c.layout)) return -1;
    // build-time sorted positions (containers.py:356-358): AoS records
    grid_bind_scratch(c, gr, AOS);
    grid_refresh(c, gr, AOS);
    int64_t n = c.n;
    v.counts.ensure(n + 1);
    v.noff.ensure(n + 1);
    GridView gv = make_view(gr);
    double ell2 = gr.g.ell * gr.g.ell;
    int m = (int)gr.m;
    if (m > 0)
        vl_build_kernel<false><<<blocks_for(m, 128), 128, 0, c.stream>>>(
            gv, gr.spos4.p, gr.row_src.p, gr.pruned, ell2, v.counts.p, nullptr, nullptr), note_launch();
    MDG_CUDA(cudaMemsetAsync(v.counts.p + n, 0, sizeof(int), c.stream));
    exclusive_scan_i32_to_i64(v.counts.p, v.noff.p, n + 1, c.scal.p + 1, c.scan_tmp, c.stream);
    MDG_CUDA(cudaMemcpyAsync(c.h_scal + 1, c.scal.p + 1, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, c.stream));
    MDG_CUDA(cudaStreamSynchronize(c.stream));
    v.entries = (int64_t)c.h_scal[1];
    v.nbr.ensure(v.entries + 1);
    if (m > 0)
        vl_build_kernel<true><<<blocks_for(m, 128), 128, 0, c.stream>>>(
            gv, gr.spos4.p, gr.row_src.p, gr.pruned, ell2, nullptr, v.noff.p, v.nbr.p), note_launch();
    MDG_CUDA(cudaGetLastError());
    v.built = true;
    return 0;
}

struct MinImage {
    double L[3], invL[3];
    int per[3];
};

// vl_force (kernels.py:730-818): per particle, list walk on the particle
// arrays, minimum image on periodic axes, strict cutoff, writes only f_i.
template <int LAYOUT, bool MT>
__global__ void __launch_bounds__(128) vl_force_kernel(int64_t n, const double* __restrict__ pos,
                                                       double* __restrict__ force,
                                                       const int* __restrict__ tid,
                                                       const long long* __restrict__ noff,
                                                       const int* __restrict__ nbr, LJTab tab,
                                                       MinImage mi,
                                                       unsigned long long* counter) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned cnt = 0;
    if (i < n) {
        double xi = pos[pidx<LAYOUT>(i, 0, n)], yi = pos[pidx<LAYOUT>(i, 1, n)],
               zi = pos[pidx<LAYOUT>(i, 2, n)];
        int ti = MT ? tid[i] : 0;
        double fx = 0.0, fy = 0.0, fz = 0.0;
        long long k1 = noff[i + 1];
        for (long long k = noff[i]; k < k1; ++k) {
            int j = nbr[k];
            double dx = xi - pos[pidx<LAYOUT>(j, 0, n)];
            double dy = yi - pos[pidx<LAYOUT>(j, 1, n)];
            double dz = zi - pos[pidx<LAYOUT>(j, 2, n)];
            if (mi.per[0]) dx -= mi.L[0] * rint(dx * mi.invL[0]);
            if (mi.per[1]) dy -= mi.L[1] * rint(dy * mi.invL[1]);
            if (mi.per[2]) dz -= mi.L[2] * rint(dz * mi.invL[2]);
            double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 < tab.rc2) {
                double s2, e24;
                lj_params<MT>(tab, ti, MT ? tid[j] : 0, s2, e24);
                double fs = lj_fs(r2, s2, e24);
                ++cnt;
                fx += fs * dx;
                fy += fs * dy;
                fz += fs * dz;
            }
        }
        force[pidx<LAYOUT>(i, 0, n)] = fx;
        force[pidx<LAYOUT>(i, 1, n)] = fy;
        force[pidx<LAYOUT>(i, 2, n)] = fz;
    }
    warp_count(counter, cnt);
}

void vl_compute(Context& c) {
    if (c.n == 0) return;
    MinImage mi;
    for (int k = 0; k < 3; ++k) {
        mi.L[k] = c.L[k];
        mi.invL[k] = 1.0 / c.L[k];
        mi.per[k] = c.periodic[k];
    }
    bool mt = c.tab.T > 1;
    dim3 b(blocks_for(c.n, 128)), t(128);
    auto* v = &c.vl;
    c.prof_mark();
    if (c.layout == AOS) {
        if (mt) vl_force_kernel<AOS, true><<<b, t, 0, c.stream>>>(c.n, c.pos, c.force, c.tid, v->noff.p, v->nbr.p, c.tab, mi, c.scal.p), note_launch();
        else vl_force_kernel<AOS, false><<<b, t, 0, c.stream>>>(c.n, c.pos, c.force, c.tid, v->noff.p, v->nbr.p, c.tab, mi, c.scal.p), note_launch();
    } else {
        if (mt) vl_force_kernel<SOA, true><<<b, t, 0, c.stream>>>(c.n, c.pos, c.force, c.tid, v->noff.p, v->nbr.p, c.tab, mi, c.scal.p), note_launch();
        else vl_force_kernel<SOA, false><<<b, t, 0, c.stream>>>(c.n, c.pos, c.force, c.tid, v->noff.p, v->nbr.p, c.tab, mi, c.scal.p), note_launch();
    }
    c.prof_mark();
}

}  // namespace mdg
