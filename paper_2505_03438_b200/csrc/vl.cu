// Verlet lists (VL-List_Iter-NoN3L-{AoS,SoA}) realised for the GPU.
//
// Reference: VerletListState (containers.py:343-375), vl_count_pairs /
// vl_fill_pairs (kernels.py:823-910), vl_force_aos/_soa (kernels.py:730-818).
//
// Same pair sets, same per-owner order, same counts as the reference; the
// storage is GPU-shaped:
//  * lists live in the cell-sorted row space of the CSF-1 grid (owned rows +
//    periodic-image rows, containers.py:78-118), one row per list, entries are
//    int32 row indices, stored warp-blocked column-major with a fixed width
//    (entry k of row r at [(r/32)*32*cap + k*32 + r%32]) so a warp's k-th
//    loads are one 128-byte line;
//  * the build is a single pass (count + fill) with r^2 <= (rc+skin)^2 in fp64
//    on the build-time positions pos[src] + shift; the width is retried upward
//    if any row overflows;
//  * every compute first refreshes an "unwrapped" sorted copy of the positions:
//    each row takes the periodic image of pos[src] (+ build shift) nearest to
//    its previous value, so d = x_i - x_j is the minimum-image displacement of
//    the reference (kernels.py:755-757) without per-pair rint() work;
//  * the force walk is one thread per row (halo rows have empty lists), writes
//    only f_i (NoN3L), counts each within-cutoff direction.
#include <algorithm>
#include <vector>

#include "device.cuh"

namespace mdg {

// ---------------------------------------------------------------- build

// The build positions of every row in one pass: pos[src] + shift (the
// arithmetic of grid.cu's refresh_kernel, containers.py:356-358) into the grid
// scratch (fp64 membership tests) and the unwrapped force-time copy s4, and
// their fp32 copy + max |coordinate| (the fp32 filter's margin; a block
// maximum, then one atomic per block: x >= 0 orders like its bit pattern).
template <int PLAYOUT>
__global__ void vl_build_pos_kernel(const double* __restrict__ pos, int64_t n, int m,
                                    const int* __restrict__ row_src, const uint8_t* __restrict__ row_code,
                                    const int* __restrict__ row_tid, double L0, double L1, double L2,
                                    double4* __restrict__ spos4, double4* __restrict__ s4,
                                    float4* __restrict__ b32, unsigned* __restrict__ maxabs_bits,
                                    float* __restrict__ disp) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    float mx = 0.f;
    if (disp && r <= m) disp[r] = 0.f;   // dynamic pruning: path lengths since the (first) prune
    if (r < m) {
        int src = row_src[r], code = row_code[r];
        double x = pos[pidx<PLAYOUT>(src, 0, n)] + (double)(code / 9 - 1) * L0;
        double y = pos[pidx<PLAYOUT>(src, 1, n)] + (double)((code / 3) % 3 - 1) * L1;
        double z = pos[pidx<PLAYOUT>(src, 2, n)] + (double)(code % 3 - 1) * L2;
        double4 p = make_double4(x, y, z, (double)row_tid[r]);
        spos4[r] = p;
        s4[r] = p;
        float4 q = make_float4((float)x, (float)y, (float)z, 0.f);
        b32[r] = q;
        mx = fmaxf(fabsf(q.x), fmaxf(fabsf(q.y), fabsf(q.z)));
    }
    __shared__ float wmax[32];
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, wmax[w]);
        atomicMax(maxabs_bits, __float_as_uint(mx));
    }
}

// Membership r^2 <= ell^2 (non-strict, kernels.py:848), decided in fp32 where
// provably safe and in fp64 otherwise, so the pair set is exactly the
// reference's.  Rounding bound for coordinates |x| <= X, |d| ~ ell, u = 2^-24:
// eta = 2uX + 2u ell bounds |d32 - d| per component, and
// |r2_32 - r2| <= 2 sqrt(3) eta ell + 3 eta^2 + 3u ell^2 =: B.  Candidates with
// r2_32 <= ell^2 - 2B are in, r2_32 > ell^2 + 2B are out, the rest are tested
// on the fp64 positions.
constexpr int kBuildThreads = 128;

__global__ void __launch_bounds__(kBuildThreads) vl_build_kernel(
    GridView gv, const double4* __restrict__ bpos, const float4* __restrict__ b32,
    const unsigned* __restrict__ maxabs_bits, const uint8_t* __restrict__ row_code, Stencil st,
    double ell2, int cap, int* __restrict__ cnt, int* __restrict__ nbr, int* __restrict__ maxcnt,
    const uint8_t* __restrict__ only) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    // periodic-image rows own no list; `only` restricts the build to flagged rows
    bool active = r < gv.m && row_code[r] == kNoShift && (!only || only[r]);
    int c = 0;
    if (active) {
    int cell = gv.row_cell[r], cx, cy, cz;
    gv.decode(cell, cx, cy, cz);
    double4 pi = bpos[r];
    float4 qi = b32[r];
    const double u = 5.9604644775390625e-08;   // 2^-24
    double X = (double)__uint_as_float(*maxabs_bits) * (1.0 + 4.0 * u);
    double ell = sqrt(ell2);
    double eta = 2.0 * u * X + 2.0 * u * ell;
    double B = 3.4641016151377544 * eta * ell + 3.0 * eta * eta + 3.0 * u * ell2;
    float lo = __double2float_rd(ell2 - 2.0 * B), hi = __double2float_ru(ell2 + 2.0 * B);
    int* out = nbr + (size_t)(r >> 5) * 32 * cap + (r & 31);
    // Tight scan: the next candidate's load is issued before the current one
    // is tested, the store is predicated and the count advances by the test
    // result, so the loop has no data-dependent branch except the rare
    // borderline fp64 re-test.
    auto visit_range = [&](int s2, int e2, int skip) {
        // chunks of four: four independent loads, then predicated tests; the
        // borderline fp64 re-test is one (rarely taken) branch per chunk
        for (int j0 = s2; j0 < e2; j0 += 4) {
            float4 q[4];
            float r2f[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = b32[min(j0 + u, e2 - 1)];
            bool border = false;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float fx = qi.x - q[u].x, fy = qi.y - q[u].y, fz = qi.z - q[u].z;
                r2f[u] = fx * fx + fy * fy + fz * fz;
                border |= (r2f[u] > lo) & (r2f[u] <= hi) & (j0 + u < e2);
            }
            bool in[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) in[u] = r2f[u] <= lo;
            if (border) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (r2f[u] > lo && r2f[u] <= hi && j0 + u < e2) {
                        double4 pj = ldg256(bpos + j0 + u);
                        double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
                        in[u] = dx * dx + dy * dy + dz * dz <= ell2;
                    }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                int j = j0 + u;
                bool ok = in[u] & (j < e2) & (j != skip);
                if (ok && c < cap) out[(size_t)c * 32] = j;
                c += ok;
            }
        }
    };
    if (st.n == 26) {
        // CSF-1 grid: the stencil is the full 3x3x3 block, i.e. nine z-runs of
        // up to three cells that are contiguous in row order; scanning them in
        // (dx, dy) order visits rows in ascending order, exactly like the
        // cell-by-cell walk below.
        int za = max(cz - 1, 0), zb = min(cz + 1, gv.D2 - 1);
        for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy) {
                int x2 = cx + dx, y2 = cy + dy;
                if (x2 < 0 || x2 >= gv.D0 || y2 < 0 || y2 >= gv.D1) continue;
                visit_range(gv.start[gv.flat(x2, y2, za)], gv.start[gv.flat(x2, y2, zb) + 1],
                            (dx == 0 && dy == 0) ? r : -1);
            }
    } else {
        auto visit_cell = [&](int k) {
            int x2 = cx + st.d[k][0], y2 = cy + st.d[k][1], z2 = cz + st.d[k][2];
            if (!gv.in_grid(x2, y2, z2)) return;
            int c2 = gv.flat(x2, y2, z2);
            visit_range(gv.start[c2], gv.start[c2 + 1], -1);
        };
        int half = st.n / 2;
        for (int k = 0; k < half; ++k) visit_cell(k);
        visit_range(gv.start[cell], gv.start[cell + 1], r);
        for (int k = half; k < st.n; ++k) visit_cell(k);
    }
    }
    if (r < gv.m) cnt[r] = c;
    if (c > cap) atomicMax(maxcnt, c);
}

// Row-space lists for every row (only == nullptr) or for the flagged rows;
// the width is retried upward if a row overflows.
int vl_build_rows(Context& c, const uint8_t* only) {
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    int m = (int)gr.m;
    size_t mpad = ((size_t)m + 31) / 32 * 32;
    GridView gv = make_view(gr);
    double ell2 = gr.g.ell * gr.g.ell;
    int* maxcnt = (int*)(c.scal.p + 3);
    const unsigned* maxabs = (const unsigned*)(c.scal.p + 5);
    for (int attempt = 0; attempt < 3 && m > 0; ++attempt) {
        v.nbr.ensure(mpad * (size_t)v.cap);
        if (!v.nbr.p) { set_error("out of device memory (Verlet lists)"); return -1; }
        MDG_CUDA(cudaMemsetAsync(maxcnt, 0, sizeof(int), c.stream));
        vl_build_kernel<<<blocks_for(m, kBuildThreads), kBuildThreads, 0, c.stream>>>(
            gv, gr.spos4.p, v.b32.p, maxabs, gr.row_code.p, gr.pruned, ell2, v.cap, v.cnt.p, v.nbr.p,
            maxcnt, only), note_launch();
        int hmax = 0;
        MDG_CUDA(cudaMemcpyAsync(&hmax, maxcnt, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        MDG_CUDA(cudaStreamSynchronize(c.stream));
        if (hmax <= v.cap) break;
        v.cap = (hmax + hmax / 8 + 7) / 8 * 8;
    }
    if (!only) v.rows_valid = true;
    return 0;
}

// The row-space lists are what the energy, the exports, the fp32 variant and
// the untiled walk read; with tiles they are built on first use after a rebuild.
int vl_ensure_rows(Context& c) {
    if (c.vl.rows_valid || !c.vl.built) return 0;
    return vl_build_rows(c, nullptr);
}

int vl_rebuild(Context& c) {
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    v.built = false;
    v.rows_valid = false;
    if (grid_rebuild(c, gr, c.pos, c.layout)) return -1;
    grid_bind_scratch(c, gr, AOS);
    int m = (int)gr.m;
    size_t mpad = ((size_t)m + 31) / 32 * 32;
    v.cnt.ensure(mpad + 1);
    if (v.cap == 0) {
        // first guess from the mean density: rho * 4/3 pi ell^3, plus headroom
        // (MDG_VL_CAP0: a forced first guess, to exercise the capacity retry)
        double vol = c.L[0] * c.L[1] * c.L[2];
        double ell = gr.g.ell;
        double expect = (double)c.n / vol * 4.18879020479 * ell * ell * ell;
        v.cap = ((int)(1.5 * expect) + 16 + 7) / 8 * 8;
        if (const char* e = getenv("MDG_VL_CAP0")) v.cap = std::max(8, atoi(e));
    }
    unsigned* maxabs = (unsigned*)(c.scal.p + 5);   // zeroed by grid_rebuild's binning
    v.b32.ensure(mpad + 1);
    // the unwrapped force-time copy s4 starts from the build positions
    v.s4.ensure(mpad + 1);
    float* disp = vlt_prune_prepare(c);
    if (m > 0) {
        // build-time positions pos[src] + shift (containers.py:356-358), s4, fp32 copy
        if (c.layout == AOS)
            vl_build_pos_kernel<AOS><<<blocks_for(m + 1, 256), 256, 0, c.stream>>>(
                c.pos, c.n, m, gr.row_src.p, gr.row_code.p, gr.row_tid.p, c.L[0], c.L[1], c.L[2], gr.spos4.p,
                v.s4.p, v.b32.p, maxabs, disp), note_launch();
        else
            vl_build_pos_kernel<SOA><<<blocks_for(m + 1, 256), 256, 0, c.stream>>>(
                c.pos, c.n, m, gr.row_src.p, gr.row_code.p, gr.row_tid.p, c.L[0], c.L[1], c.L[2], gr.spos4.p,
                v.s4.p, v.b32.p, maxabs, disp), note_launch();
    }
    int e = vlt_build(c);               // tile lists (vltile.cu); 1 = not applicable
    if (e < 0) return -1;
    if (e == 1 && vl_build_rows(c, nullptr)) return -1;
    v.s3_valid = false;
    MDG_CUDA(cudaGetLastError());
    v.built = true;
    return 0;
}

// ---------------------------------------------------------------- refresh

struct Wrap {
    double L[3];
    double invL[3];
    int per[3];
};

// Nearest periodic image of pos[src] + shift to the previous row value.
//
// With `disp` (dynamic pruning of the tile lists, vltile.cu) every owned row
// also adds the length of its move, rounded up, to disp[r]; a row past `thr`
// raises pst[0], which makes the walk that follows prune again.
template <int PLAYOUT, int SLAYOUT>
__global__ void vl_refresh_kernel(const double* __restrict__ pos, int64_t n, int m, int ms,
                                  const int* __restrict__ row_src,
                                  const uint8_t* __restrict__ row_code, Wrap w,
                                  double4* __restrict__ s4, double* __restrict__ s3,
                                  bool from_s4, int* zero_me, float* __restrict__ disp, int* pst,
                                  float thr, unsigned long long* zero_cnt = nullptr) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r == 0 && zero_me) *zero_me = 0;   // work counter of the tiled walk
    if (r == 0 && zero_cnt) *zero_cnt = 0;   // the eval count the walk accumulates (no memset launch)
    bool over = false;
    if (r < m) {
        int src = row_src[r], code = row_code[r];
        double q[3] = {pos[pidx<PLAYOUT>(src, 0, n)], pos[pidx<PLAYOUT>(src, 1, n)],
                       pos[pidx<PLAYOUT>(src, 2, n)]};
        int sh[3] = {code / 9 - 1, (code / 3) % 3 - 1, code % 3 - 1};
        double prev[3];
        // the SoA copy's previous values come from s3 itself: no 32-byte s4
        // read per row on the steady path
        double4 old = make_double4(0.0, 0.0, 0.0, 0.0);
        if (SLAYOUT == AOS || from_s4) {
            old = s4[r];
            prev[0] = old.x; prev[1] = old.y; prev[2] = old.z;
        } else {
            prev[0] = s3[r]; prev[1] = s3[(size_t)ms + r]; prev[2] = s3[2 * (size_t)ms + r];
        }
        for (int k = 0; k < 3; ++k) {
            double x = q[k] + (double)sh[k] * w.L[k];
            if (w.per[k]) x += w.L[k] * rint((prev[k] - x) * w.invL[k]);
            q[k] = x;
        }
        if (disp && code == kNoShift) {
            double ex = q[0] - prev[0], ey = q[1] - prev[1], ez = q[2] - prev[2];
            float a = __fadd_ru(disp[r], __double2float_ru(sqrt(ex * ex + ey * ey + ez * ez)));
            disp[r] = a;
            over = !(a <= thr);   // NaN counts as a violation
        }
        if (SLAYOUT == AOS) {
            s4[r] = make_double4(q[0], q[1], q[2], old.w);
        } else {
            s3[r] = q[0];
            s3[(size_t)ms + r] = q[1];
            s3[2 * (size_t)ms + r] = q[2];
        }
    }
    if (over) *pst = 1;   // rare; every writer stores the same value
}

// ---------------------------------------------------------------- force

// The list is streamed once per step (~4 B per entry, hundreds of MB): it is
// read with evict-first (__ldcs) so it does not push the positions -- the
// data every gather reuses -- out of L2.
//
// G entries per round (a multiple of 4: every four share one reciprocal,
// y = 1/(q0 q1 q2 q3), 1/q0 = y q1 q2 q3 etc., so the XU pipe sees one
// MUFU.RCP64H per four pairs).  PF: the next round's list indices are loaded
// before this round's gathers, so the HBM latency of the list stream overlaps
// the gather + arithmetic of the current round.
template <int SLAYOUT, int PLAYOUT, bool MT, int G, bool PF, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) vl_force_kernel(int m, int ms, int64_t n, int cap,
                                                      const double4* __restrict__ s4,
                                                      const double* __restrict__ s3,
                                                      const int* __restrict__ row_tid,
                                                      const int* __restrict__ cnt,
                                                      const int* __restrict__ nbr,
                                                      const int* __restrict__ row_src,
                                                      const uint8_t* __restrict__ row_code,
                                                      double* __restrict__ force, LJTab tab,
                                                      unsigned long long* counter,
                                                      const uint8_t* __restrict__ only) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned hits = 0;
    if (r < m && row_code[r] == kNoShift && (!only || only[r])) {
        double xi, yi, zi;
        int ti = 0;
        if (SLAYOUT == AOS) {
            double4 p = s4[r];
            xi = p.x; yi = p.y; zi = p.z;
            if (MT) ti = (int)p.w;
        } else {
            xi = s3[r]; yi = s3[(size_t)ms + r]; zi = s3[2 * (size_t)ms + r];
            if (MT) ti = row_tid[r];
        }
        double fx = 0.0, fy = 0.0, fz = 0.0;
        const int* lp = nbr + (size_t)(r >> 5) * 32 * cap + (r & 31);
        int c = cnt[r];
        int jn[G];
#pragma unroll
        for (int u = 0; u < G; ++u) jn[u] = u < c ? __ldcs(lp + (size_t)u * 32) : r;
        for (int k0 = 0; k0 < c; k0 += G) {
            double dx[G], dy[G], dz[G], q[G];
            int tj[G], jc[G];
            bool ok[G];
#pragma unroll
            for (int u = 0; u < G; ++u) jc[u] = jn[u];
            if (PF) {
#pragma unroll
                for (int u = 0; u < G; ++u)
                    jn[u] = k0 + G + u < c ? __ldcs(lp + (size_t)(k0 + G + u) * 32) : r;
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
                bool has = k0 + u < c;
                int j = jc[u];
                double xj, yj, zj;
                tj[u] = 0;
                if (SLAYOUT == AOS) {
                    // one 256-bit load per record (measured faster than a
                    // 128+64-bit split even though it moves 8 more bytes)
                    double4 p = ldg256(s4 + j);
                    xj = p.x; yj = p.y; zj = p.z;
                    if (MT) tj[u] = (int)p.w;
                } else {
                    xj = s3[j]; yj = s3[(size_t)ms + j]; zj = s3[2 * (size_t)ms + j];
                    if (MT) tj[u] = row_tid[j];
                }
                dx[u] = xi - xj; dy[u] = yi - yj; dz[u] = zi - zj;
                double r2 = dx[u] * dx[u] + dy[u] * dy[u] + dz[u] * dz[u];
                ok[u] = has && r2 < tab.rc2;
                q[u] = ok[u] ? r2 : 1.0;
            }
            double inv[G];
#pragma unroll
            for (int b = 0; b < G; b += 4) {
                double p01 = q[b] * q[b + 1], p23 = q[b + 2] * q[b + 3];
                double y = fast_rcp(p01 * p23);
                double y01 = y * p23, y23 = y * p01;
                inv[b] = y01 * q[b + 1];
                inv[b + 1] = y01 * q[b];
                inv[b + 2] = y23 * q[b + 3];
                inv[b + 3] = y23 * q[b + 2];
            }
            if (!PF) {
#pragma unroll
                for (int u = 0; u < G; ++u)
                    jn[u] = k0 + G + u < c ? __ldcs(lp + (size_t)(k0 + G + u) * 32) : r;
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
                if (ok[u]) {
                    double s2, e24;
                    lj_params<MT>(tab, ti, tj[u], s2, e24);
                    double a = s2 * inv[u];
                    double a6 = a * a * a;
                    double fs = (e24 * inv[u]) * (a6 * fma(2.0, a6, -1.0));
                    ++hits;
                    fx = fma(fs, dx[u], fx);
                    fy = fma(fs, dy[u], fy);
                    fz = fma(fs, dz[u], fz);
                }
            }
        }
        int i = row_src[r];
        force[pidx<PLAYOUT>(i, 0, n)] = fx;
        force[pidx<PLAYOUT>(i, 1, n)] = fy;
        force[pidx<PLAYOUT>(i, 2, n)] = fz;
    }
    warp_count(counter, hits);
}

// Force-walk variant (tuning experiments): MDG_VL_VARIANT=0..5, read once.
static int vl_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VL_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <int SLAYOUT, int PLAYOUT>
static void vl_launch(Context& c, bool mt) {
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    int m = (int)gr.m;
    Wrap w;
    for (int k = 0; k < 3; ++k) {
        w.L[k] = c.L[k];
        w.invL[k] = 1.0 / c.L[k];
        w.per[k] = c.periodic[k];
    }
    dim3 b(blocks_for(m, 256)), t(256);
    bool from_s4 = SLAYOUT == SOA && !v.s3_valid;
    vl_refresh_kernel<PLAYOUT, SLAYOUT><<<b, t, 0, c.stream>>>(c.pos, c.n, m, s3_stride(m), gr.row_src.p, gr.row_code.p, w, v.s4.p, v.s3.p, from_s4, nullptr, nullptr, nullptr, 0.f), note_launch();
    vl_prune_invalidate(c);
    if (SLAYOUT == SOA) v.s3_valid = true;
    c.prof_mark();
#define MDG_VLF(G, PF, NT, MB)                                                                     \
    do {                                                                                         \
        if (mt)                                                                                  \
            vl_force_kernel<SLAYOUT, PLAYOUT, true, G, PF, NT, MB><<<blocks_for(m, NT), NT, 0, c.stream>>>( \
                m, s3_stride(m), c.n, v.cap, v.s4.p, v.s3.p, gr.row_tid.p, v.cnt.p, v.nbr.p, gr.row_src.p,      \
                gr.row_code.p, c.force, c.tab, c.scal.p, nullptr), note_launch();                 \
        else                                                                                     \
            vl_force_kernel<SLAYOUT, PLAYOUT, false, G, PF, NT, MB><<<blocks_for(m, NT), NT, 0, c.stream>>>( \
                m, s3_stride(m), c.n, v.cap, v.s4.p, v.s3.p, gr.row_tid.p, v.cnt.p, v.nbr.p, gr.row_src.p,      \
                gr.row_code.p, c.force, c.tab, c.scal.p, nullptr), note_launch();                 \
    } while (0)
    // measured on B200, config 2 (profiles/round1_vl_variants.txt): all within
    // 6%; index prefetch with 4-entry rounds and 128-thread CTAs is fastest
    switch (vl_variant()) {
        case 10: MDG_VLF(4, false, 128, 1); break;
        case 2: MDG_VLF(8, false, 128, 1); break;
        case 3: MDG_VLF(8, true, 128, 1); break;
        case 4: MDG_VLF(4, true, 256, 1); break;
        case 5: MDG_VLF(4, true, 64, 1); break;
        case 6: MDG_VLF(4, true, 128, 8); break;
        case 7: MDG_VLF(4, true, 128, 10); break;
        case 8: MDG_VLF(4, true, 128, 12); break;
        case 9: MDG_VLF(4, false, 128, 12); break;
        default: MDG_VLF(4, true, 128, 1); break;
    }
#undef MDG_VLF
    c.prof_mark();
}

static Wrap make_wrap(const Context& c) {
    Wrap w;
    for (int k = 0; k < 3; ++k) {
        w.L[k] = c.L[k];
        w.invL[k] = 1.0 / c.L[k];
        w.per[k] = c.periodic[k];
    }
    return w;
}

template <int PLAYOUT, int SLAYOUT>
void vl_refresh_launch(Context& c, int* zero_me, unsigned long long* zero_cnt) {
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    int m = (int)gr.m;
    bool from_s4 = SLAYOUT == SOA && !v.s3_valid;
    vl_refresh_kernel<PLAYOUT, SLAYOUT><<<blocks_for(m, 256), 256, 0, c.stream>>>(
        c.pos, c.n, m, s3_stride(m), gr.row_src.p, gr.row_code.p, make_wrap(c), v.s4.p, v.s3.p, from_s4, zero_me,
        v.prune ? v.disp.p : nullptr, v.pst.p, v.prune_thr, zero_cnt), note_launch();
    if (SLAYOUT == SOA) v.s3_valid = true;
}
template void vl_refresh_launch<AOS, SOA>(Context&, int*, unsigned long long*);

// the same unwrapped refresh for another container's rows (VCL, vcl.cu)
void vl_refresh_into(Context& c, Grid& gr, double4* s4, double* s3, bool& s3_valid) {
    int m = (int)gr.m;
    if (m == 0) return;
    if (c.layout == AOS)
        vl_refresh_kernel<AOS, SOA><<<blocks_for(m, 256), 256, 0, c.stream>>>(
            c.pos, c.n, m, s3_stride(m), gr.row_src.p, gr.row_code.p, make_wrap(c), s4, s3, !s3_valid,
            nullptr, nullptr, nullptr, 0.f), note_launch();
    else
        vl_refresh_kernel<SOA, SOA><<<blocks_for(m, 256), 256, 0, c.stream>>>(
            c.pos, c.n, m, s3_stride(m), gr.row_src.p, gr.row_code.p, make_wrap(c), s4, s3, !s3_valid,
            nullptr, nullptr, nullptr, 0.f), note_launch();
    s3_valid = true;
}
template void vl_refresh_launch<SOA, SOA>(Context&, int*, unsigned long long*);

// global-gather walk over the rows flagged in `only` (SoA source)
template <int PLAYOUT>
void vl_force_rows_launch(Context& c, const uint8_t* only) {
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    int m = (int)gr.m;
    if (c.tab.T > 1)
        vl_force_kernel<SOA, PLAYOUT, true, 4, true, 128, 1><<<blocks_for(m, 128), 128, 0, c.stream>>>(
            m, s3_stride(m), c.n, v.cap, v.s4.p, v.s3.p, gr.row_tid.p, v.cnt.p, v.nbr.p, gr.row_src.p,
            gr.row_code.p, c.force, c.tab, c.scal.p, only), note_launch();
    else
        vl_force_kernel<SOA, PLAYOUT, false, 4, true, 128, 1><<<blocks_for(m, 128), 128, 0, c.stream>>>(
            m, s3_stride(m), c.n, v.cap, v.s4.p, v.s3.p, gr.row_tid.p, v.cnt.p, v.nbr.p, gr.row_src.p,
            gr.row_code.p, c.force, c.tab, c.scal.p, only), note_launch();
}
template void vl_force_rows_launch<AOS>(Context&, const uint8_t*);
template void vl_force_rows_launch<SOA>(Context&, const uint8_t*);

// the deferred tile-build check; if it fails the row-space lists take over
static void vl_finish_build(Context& c) {
    if (vlt_finish(c)) {
        c.vl.tiled = false;
        c.vl.prune = false;
        vl_ensure_rows(c);
    }
}

void vl_compute(Context& c, int layout) {
    if (c.n == 0) return;
    Verlet& v = c.vl;
    bool mt = c.tab.T > 1;
    if (vlt_speculate(c)) {
        // the first walk after a build, queued before the build's host check
        // (vlt_finish): the host then waits on the build while the GPU walks,
        // instead of the GPU idling through the wake-up and the launches.  A
        // failed check is repaired after the fact: lists rebuilt with a larger
        // capacity are walked again (forces and count overwritten), overflow
        // tiles' rows go through the row-space walk, a failed build falls back
        // to the row-space lists below.
        v.s3.ensure(3 * (size_t)s3_stride((int)v.grid.m) + 8);
        const int cap0 = v.cap;
        vlt_compute(c);
        if (vlt_finish(c) == 0 && v.tiled) {
            if (v.cap != cap0) vlt_compute(c);   // (walks the overflow tiles' rows too)
            else vlt_big_rows(c);
            return;
        }
        v.tiled = false;
        v.prune = false;
        vl_ensure_rows(c);
    } else {
        vl_finish_build(c);
    }
    if (v.tiled) {
        v.s3.ensure(3 * (size_t)s3_stride((int)v.grid.m) + 8);
        if (vlt_compute(c)) return;   // its refresh zeroes the eval count
    }
    cudaMemsetAsync(c.scal.p, 0, sizeof(unsigned long long), c.stream);
    if (layout == SOA) v.s3.ensure(3 * (size_t)s3_stride((int)v.grid.m) + 8);
    if (c.layout == AOS) {
        if (layout == AOS) vl_launch<AOS, AOS>(c, mt);
        else vl_launch<SOA, AOS>(c, mt);
    } else {
        if (layout == AOS) vl_launch<AOS, SOA>(c, mt);
        else vl_launch<SOA, SOA>(c, mt);
    }
}

// ---------------------------------------------------------------- fp32 variant

// fp32-compute / fp64-accumulate walk (north_star: "fp64 accumulation with an
// fp32-compute variant", tolerance 1e-4).  Each row carries its position
// relative to the origin of its build-time cell in fp32 plus that cell's
// integer coordinates (10 bits each) in the fourth word, so a displacement is
// (r_i - r_j) + (c_i - c_j) * cell_len with the integer part exact: the fp32
// error is that of coordinates inside one cell, not of the box.  Gathers are
// 16 bytes (one LDG.128) instead of 32.
__device__ __forceinline__ int pack_cell(int x, int y, int z) { return (x << 20) | (y << 10) | z; }

template <int PLAYOUT>
__global__ void vl_refresh32_kernel(const double* __restrict__ pos, int64_t n, int m,
                                    const int* __restrict__ row_src,
                                    const uint8_t* __restrict__ row_code,
                                    const int* __restrict__ row_cell, GridView gv, Wrap w, Cells32 cc,
                                    double4* __restrict__ s4, float4* __restrict__ q32, int* zero_me,
                                    float* __restrict__ disp, int* pst, float thr) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r == 0 && zero_me) *zero_me = 0;   // work counter of the tiled walk
    if (r >= m) return;
    int src = row_src[r], code = row_code[r];
    double q[3] = {pos[pidx<PLAYOUT>(src, 0, n)], pos[pidx<PLAYOUT>(src, 1, n)],
                   pos[pidx<PLAYOUT>(src, 2, n)]};
    int sh[3] = {code / 9 - 1, (code / 3) % 3 - 1, code % 3 - 1};
    double4 old = s4[r];
    double prev[3] = {old.x, old.y, old.z};
    for (int k = 0; k < 3; ++k) {
        double x = q[k] + (double)sh[k] * w.L[k];
        if (w.per[k]) x += w.L[k] * rint((prev[k] - x) * w.invL[k]);
        q[k] = x;
    }
    s4[r] = make_double4(q[0], q[1], q[2], old.w);
    if (disp && code == kNoShift) {   // dynamic pruning's path length, as in vl_refresh_kernel
        double ex = q[0] - prev[0], ey = q[1] - prev[1], ez = q[2] - prev[2];
        float a = __fadd_ru(disp[r], __double2float_ru(sqrt(ex * ex + ey * ey + ez * ez)));
        disp[r] = a;
        if (!(a <= thr)) *pst = 1;
    }
    int cx, cy, cz;
    gv.decode(row_cell[r], cx, cy, cz);
    // padded-grid cell (cx, cy, cz) spans [(c - H) * cl, (c - H + 1) * cl)
    float4 o;
    o.x = (float)(q[0] - (double)(cx - gv.H0) * cc.cld[0]);
    o.y = (float)(q[1] - (double)(cy - gv.H1) * cc.cld[1]);
    o.z = (float)(q[2] - (double)(cz - gv.H2) * cc.cld[2]);
    o.w = __int_as_float(pack_cell(cx, cy, cz));
    q32[r] = o;
}

template <int PLAYOUT, bool MT>
__global__ void __launch_bounds__(128) vl_force32_kernel(int m, int64_t n, int cap,
                                                         const float4* __restrict__ q32,
                                                         const int* __restrict__ row_tid,
                                                         const int* __restrict__ cnt,
                                                         const int* __restrict__ nbr,
                                                         const int* __restrict__ row_src,
                                                         const uint8_t* __restrict__ row_code,
                                                         double* __restrict__ force, LJTab tab,
                                                         Cells32 cc, unsigned long long* counter,
                                                         const uint8_t* __restrict__ only) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned hits = 0;
    if (r < m && row_code[r] == kNoShift && (!only || only[r])) {
        float4 qi = q32[r];
        int ci = __float_as_int(qi.w);
        int ti = MT ? row_tid[r] : 0;
        float rc2 = (float)tab.rc2;
        double fx = 0.0, fy = 0.0, fz = 0.0;
        const int* lp = nbr + (size_t)(r >> 5) * 32 * cap + (r & 31);
        int c = cnt[r];
        // fp32 partial sums over rounds of 8 pairs, folded into the fp64
        // accumulators once per round (3 conversions per 8 pairs, not per pair)
        for (int k0 = 0; k0 < c; k0 += 8) {
            float px = 0.f, py = 0.f, pz = 0.f;
            int kend = min(c, k0 + 8);
            for (int k = k0; k < kend; ++k) {
                int j = __ldcs(lp + (size_t)k * 32);
                float4 qj = __ldg(q32 + j);
                int cj = __float_as_int(qj.w);
                float dx = (qi.x - qj.x) + (float)((ci >> 20) - (cj >> 20)) * cc.cl[0];
                float dy = (qi.y - qj.y) + (float)(((ci >> 10) & 1023) - ((cj >> 10) & 1023)) * cc.cl[1];
                float dz = (qi.z - qj.z) + (float)((ci & 1023) - (cj & 1023)) * cc.cl[2];
                float r2 = dx * dx + dy * dy + dz * dz;
                if (r2 < rc2) {
                    double s2d, e24d;
                    lj_params<MT>(tab, ti, MT ? row_tid[j] : 0, s2d, e24d);
                    float inv = __frcp_rn(r2);
                    float a = (float)s2d * inv;
                    float a6 = a * a * a;
                    float fs = ((float)e24d * inv) * (a6 * fmaf(2.0f, a6, -1.0f));
                    ++hits;
                    px = fmaf(fs, dx, px);
                    py = fmaf(fs, dy, py);
                    pz = fmaf(fs, dz, pz);
                }
            }
            fx += (double)px;
            fy += (double)py;
            fz += (double)pz;
        }
        int i = row_src[r];
        force[pidx<PLAYOUT>(i, 0, n)] = fx;
        force[pidx<PLAYOUT>(i, 1, n)] = fy;
        force[pidx<PLAYOUT>(i, 2, n)] = fz;
    }
    warp_count(counter, hits);
}

void vl_compute32(Context& c) {
    if (c.n == 0) return;
    vl_finish_build(c);
    Verlet& v = c.vl;
    bool tiled = v.tiled;
    if (!tiled && vl_ensure_rows(c)) return;
    Grid& gr = v.grid;
    int m = (int)gr.m;
    v.q32.ensure((size_t)m + 32);
    Wrap w;
    Cells32 cc;
    for (int k = 0; k < 3; ++k) {
        w.L[k] = c.L[k];
        w.invL[k] = 1.0 / c.L[k];
        w.per[k] = c.periodic[k];
        cc.cld[k] = gr.g.cl[k];
        cc.cl[k] = (float)gr.g.cl[k];
    }
    GridView gv = make_view(gr);
    bool mt = c.tab.T > 1;
    int* next = tiled ? (int*)(c.scal.p + 6) : nullptr;   // zeroed for the tiled walk
    if (c.layout == AOS)
        vl_refresh32_kernel<AOS><<<blocks_for(m, 256), 256, 0, c.stream>>>(c.pos, c.n, m, gr.row_src.p, gr.row_code.p, gr.row_cell.p, gv, w, cc, v.s4.p, v.q32.p, next, tiled && v.prune ? v.disp.p : nullptr, v.pst.p, v.prune_thr), note_launch();
    else
        vl_refresh32_kernel<SOA><<<blocks_for(m, 256), 256, 0, c.stream>>>(c.pos, c.n, m, gr.row_src.p, gr.row_code.p, gr.row_cell.p, gv, w, cc, v.s4.p, v.q32.p, next, tiled && v.prune ? v.disp.p : nullptr, v.pst.p, v.prune_thr), note_launch();
    c.prof_mark();
    if (tiled) vlt_compute32(c, cc);   // tiles; overflow tiles below
    if (!tiled || v.nbig) {
        const uint8_t* only = tiled ? v.big_row.p : nullptr;
        dim3 b(blocks_for(m, 128)), t(128);
#define MDG_VL32(P, M) vl_force32_kernel<P, M><<<b, t, 0, c.stream>>>(m, c.n, v.cap, v.q32.p, gr.row_tid.p, v.cnt.p, v.nbr.p, gr.row_src.p, gr.row_code.p, c.force, c.tab, cc, c.scal.p, only), note_launch()
        if (c.layout == AOS) {
            if (mt) MDG_VL32(AOS, true); else MDG_VL32(AOS, false);
        } else {
            if (mt) MDG_VL32(SOA, true); else MDG_VL32(SOA, false);
        }
#undef MDG_VL32
    }
    c.prof_mark();
}

// ---------------------------------------------------------------- energy

// Shifted LJ potential energy, U = 1/2 sum_i sum_{j in list(i), r<rc}
// 4 eps [(s/r)^12 - (s/r)^6 - (s/rc)^12 + (s/rc)^6] (the energy the truncated
// force conserves; reference helper tests/test_integrator.py:227-247).  No
// reference ForceCalculator counterpart (north_star: PE output).
template <bool MT>
__global__ void __launch_bounds__(256) vl_energy_kernel(int m, int cap, const double4* __restrict__ s4,
                                                        const int* __restrict__ cnt,
                                                        const int* __restrict__ nbr,
                                                        const uint8_t* __restrict__ row_code, LJTab tab,
                                                        double* __restrict__ out) {
    __shared__ double ws[8];
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    double e = 0.0;
    if (r < m && row_code[r] == kNoShift) {
        double4 pi = s4[r];
        int ti = MT ? (int)pi.w : 0;
        const int* lp = nbr + (size_t)(r >> 5) * 32 * cap + (r & 31);
        int c = cnt[r];
        for (int k = 0; k < c; ++k) {
            double4 pj = ldg256(s4 + lp[(size_t)k * 32]);
            double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
            double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 < tab.rc2) {
                double s2, e24;
                lj_params<MT>(tab, ti, MT ? (int)pj.w : 0, s2, e24);
                double a = s2 / r2, a6 = a * a * a;
                double ac = s2 / tab.rc2, ac6 = ac * ac * ac;
                e += (e24 / 6.0) * ((a6 * a6 - a6) - (ac6 * ac6 - ac6));
            }
        }
    }
    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) atomicAdd(out, 0.5 * v);
    }
}

int vl_energy(Context& c, double* pe) {
    if (vl_ensure_rows(c)) return -1;
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    int m = (int)gr.m;
    *pe = 0.0;
    if (!m) return 0;
    Wrap w;
    for (int k = 0; k < 3; ++k) {
        w.L[k] = c.L[k];
        w.invL[k] = 1.0 / c.L[k];
        w.per[k] = c.periodic[k];
    }
    if (c.layout == AOS)
        vl_refresh_kernel<AOS, AOS><<<blocks_for(m, 256), 256, 0, c.stream>>>(c.pos, c.n, m, s3_stride(m), gr.row_src.p, gr.row_code.p, w, v.s4.p, v.s3.p, false, nullptr, nullptr, nullptr, 0.f), note_launch();
    else
        vl_refresh_kernel<SOA, AOS><<<blocks_for(m, 256), 256, 0, c.stream>>>(c.pos, c.n, m, s3_stride(m), gr.row_src.p, gr.row_code.p, w, v.s4.p, v.s3.p, false, nullptr, nullptr, nullptr, 0.f), note_launch();
    vl_prune_invalidate(c);
    double* dpe = (double*)(c.scal.p + 6);
    MDG_CUDA(cudaMemsetAsync(dpe, 0, sizeof(double), c.stream));
    if (c.tab.T > 1)
        vl_energy_kernel<true><<<blocks_for(m, 256), 256, 0, c.stream>>>(m, v.cap, v.s4.p, v.cnt.p, v.nbr.p, gr.row_code.p, c.tab, dpe), note_launch();
    else
        vl_energy_kernel<false><<<blocks_for(m, 256), 256, 0, c.stream>>>(m, v.cap, v.s4.p, v.cnt.p, v.nbr.p, gr.row_code.p, c.tab, dpe), note_launch();
    MDG_CUDA(cudaMemcpyAsync(pe, dpe, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    MDG_CUDA(cudaStreamSynchronize(c.stream));
    return 0;
}

// Reference-format export: CSR by owner index with owner indices.
int vl_export(Context& c, int64_t* entries, int64_t* noff, int32_t* nbr) {
    if (vl_ensure_rows(c)) return -1;
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    int m = (int)gr.m;
    size_t mpad = ((size_t)m + 31) / 32 * 32;
    std::vector<int> cnt(m), src(m), cellof(m), ent(m), ell(mpad * (size_t)v.cap);
    std::vector<uint8_t> code(m);
    MDG_CUDA(cudaStreamSynchronize(c.stream));
    if (m) {
        MDG_CUDA(cudaMemcpy(cnt.data(), v.cnt.p, m * sizeof(int), cudaMemcpyDeviceToHost));
        MDG_CUDA(cudaMemcpy(src.data(), gr.row_src.p, m * sizeof(int), cudaMemcpyDeviceToHost));
        MDG_CUDA(cudaMemcpy(cellof.data(), gr.row_cell.p, m * sizeof(int), cudaMemcpyDeviceToHost));
        MDG_CUDA(cudaMemcpy(ent.data(), gr.row_ent.p, m * sizeof(int), cudaMemcpyDeviceToHost));
        MDG_CUDA(cudaMemcpy(code.data(), gr.row_code.p, m, cudaMemcpyDeviceToHost));
        MDG_CUDA(cudaMemcpy(ell.data(), v.nbr.p, ell.size() * sizeof(int), cudaMemcpyDeviceToHost));
    }
    int64_t n = c.n;
    std::vector<int64_t> per(n + 1, 0);
    std::vector<int> row_of(n, -1);
    for (int r = 0; r < m; ++r)
        if (code[r] == kNoShift) {
            per[src[r] + 1] = cnt[r];
            row_of[src[r]] = r;
        }
    for (int64_t i = 0; i < n; ++i) per[i + 1] += per[i];
    *entries = per[n];
    if (noff) std::copy(per.begin(), per.end(), noff);
    if (nbr) {
        // the reference order (kernels.py:886-906): own cell first, then the
        // stencil cells in order (ascending cell index on the CSF-1 grid), and
        // within a cell the stable entry order (the device grid orders a
        // cell's rows by z, so sort by entry id here)
        std::vector<int> rows;
        for (int64_t i = 0; i < n; ++i) {
            int r = row_of[i];
            const int* lp = ell.data() + (size_t)(r >> 5) * 32 * v.cap + (r & 31);
            rows.assign(cnt[r], 0);
            for (int k = 0; k < cnt[r]; ++k) rows[k] = lp[(size_t)k * 32];
            int own = cellof[r];
            std::sort(rows.begin(), rows.end(), [&](int a, int b) {
                int ca = cellof[a] == own ? -1 : cellof[a], cb = cellof[b] == own ? -1 : cellof[b];
                return ca != cb ? ca < cb : ent[a] < ent[b];
            });
            int64_t o = per[i];
            for (int j : rows) nbr[o++] = src[j];
        }
    }
    return 0;
}

}  // namespace mdg
