// Cell geometry, the stable counting sort (binning) and the scratch
// gather / force fold-back of the linked-cells container.
//
// Reference: cells.py:48-156 (geometry, stencils, cell coordinates, periodic
// images), containers.py:78-171 (GridState.rebuild, LayoutBuffers).
#include <math.h>

#include <algorithm>
#include <chrono>
#include <cstring>

#include "device.cuh"

namespace mdg {

// ---------------------------------------------------------------- geometry

Geom make_geometry(const double L[3], const int periodic[3], double ell, double csf) {
    Geom g;
    double target = csf * ell;
    g.ell = ell;
    g.csf = csf;
    for (int k = 0; k < 3; ++k) {
        g.L[k] = L[k];
        g.periodic[k] = periodic[k] ? 1 : 0;
        double q = floor(L[k] / target);
        int s = q < 1.0 ? 1 : (int)q;
        g.S[k] = s;
        g.cl[k] = L[k] / (double)s;
        int o = (int)floor(ell / g.cl[k]);
        while ((double)o * g.cl[k] < ell) ++o;
        g.overlap[k] = o < 1 ? 1 : o;
        g.H[k] = g.periodic[k] ? g.overlap[k] : 0;
        g.D[k] = s + 2 * g.H[k];
    }
    g.ncells = (int64_t)g.D[0] * g.D[1] * g.D[2];
    return g;
}

static double box_min_dist2(const int d[3], const double cl[3]) {
    double s = 0.0;
    for (int k = 0; k < 3; ++k) {
        double gap = (double)(abs(d[k]) - 1) * cl[k];
        if (gap > 0.0) s += gap * gap;
    }
    return s;
}

// cells.py:80-95: product order over (-o..o)^3, (0,0,0) skipped.
Stencil pruned_stencil(const Geom& g) {
    Stencil st;
    st.n = 0;
    double ell2 = g.ell * g.ell;
    for (int x = -g.overlap[0]; x <= g.overlap[0]; ++x)
        for (int y = -g.overlap[1]; y <= g.overlap[1]; ++y)
            for (int z = -g.overlap[2]; z <= g.overlap[2]; ++z) {
                if (!x && !y && !z) continue;
                int d[3] = {x, y, z};
                if (box_min_dist2(d, g.cl) <= ell2 && st.n < kMaxStencil) {
                    st.d[st.n][0] = x; st.d[st.n][1] = y; st.d[st.n][2] = z;
                    ++st.n;
                }
            }
    return st;
}

// cells.py:98-111: keep offsets that are lexicographically positive with the
// major axis first.
Stencil forward_stencil(const Geom& g, int major) {
    Stencil all = pruned_stencil(g), st;
    st.n = 0;
    int order[3] = {major, major == 0 ? 1 : 0, major == 2 ? 1 : 2};
    for (int i = 0; i < all.n; ++i) {
        int a = all.d[i][order[0]], b = all.d[i][order[1]], c = all.d[i][order[2]];
        bool pos = a > 0 || (a == 0 && (b > 0 || (b == 0 && c > 0)));
        if (pos) {
            std::memcpy(st.d[st.n], all.d[i], sizeof(all.d[i]));
            ++st.n;
        }
    }
    return st;
}

// ---------------------------------------------------------------- buffers

template <class T>
void DBuf<T>::ensure(size_t n) {
    if (n <= cap && p) return;
    size_t want = std::max<size_t>(n + n / 8, 64);
    // MDG_ALLOC_TRACE=1: every (re)allocation on stderr (a cudaFree + cudaMalloc
    // inside a timed loop is a host stall of milliseconds)
    static const bool trace = getenv("MDG_ALLOC_TRACE") != nullptr;
    if (trace)
        fprintf(stderr, "mdg alloc: %zu -> %zu bytes (%s)\n", cap * sizeof(T), want * sizeof(T),
                p ? "grow: cudaFree + cudaMalloc" : "new");
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, want * sizeof(T)) == cudaSuccess) cap = want;
    else p = nullptr;
}

template <class T>
void DBuf<T>::release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

template struct DBuf<int>;
template struct DBuf<uint8_t>;
template struct DBuf<double>;
template struct DBuf<double4>;
template struct DBuf<long long>;
template struct DBuf<unsigned long long>;
template struct DBuf<uint16_t>;
template struct DBuf<int4>;
template struct DBuf<int2>;
template struct DBuf<float4>;
template struct DBuf<float>;
template struct DBuf<PwLeaf>;

void Grid::release() {
    cell_count.release(); cell_start.release();
    counts_clear = 0;
    img_cnt.release(); img_off.release(); img_src.release(); img_code.release();
    tmp_ent.release(); row_ent.release(); row_src.release(); row_cell.release();
    row_tid.release(); inv.release(); row_code.release();
    spos4.release(); spos3.release(); sforce.release(); cpart.release();
    cpart_zero = 0;
    c08l_tot.release(); c08l_j.release(); c08l_f.release();
    c08l_for = -1;
    built = false;
}

void Vcl::release() {
    grid.release(); bb_lo.release(); bb_hi.release(); ccnt.release(); clist.release();
    s4.release(); s3.release();
    ncl = capc = 0;
    built = s3_valid = false;
}

void Verlet::release() {
    grid.release(); cnt.release(); nbr.release(); s4.release(); s3.release(); b32.release();
    q32.release();
    tdesc.release(); tsize.release(); tbase.release(); tl.release(); tcnt.release();
    big_row.release();
    tl_in.release(); tcnt_in.release(); disp.release(); pst.release(); bmax.release();
    nblk = 0;
    if (h_build) cudaFreeHost(h_build);
    if (ev_build) cudaEventDestroy(ev_build);
    h_build = nullptr;
    d_h_build = nullptr;
    ev_build = nullptr;
    build_pending = false;
    prune = false;
    tiled = false;
    ntiles = nbig = 0;
    cap = 0;
    built = false;
}

// ---------------------------------------------------------------- scans

// Exclusive scan in ONE launch (decoupled look-back): a CTA takes a tile of
// kSpTile elements by ticket, publishes its aggregate, and warp 0 looks back
// over the predecessors' published words, 32 at a time, until it meets an
// inclusive prefix.  Status words carry the call's epoch (16 bits), a flag
// (1 aggregate, 2 inclusive prefix) and the value (46 bits), so the array is
// never cleared between calls.  Replaces three launches per scan (tile sums,
// a one-CTA scan, tile scans): a rebuild runs three scans.  `sumsq`
// (optional) receives the sum of squared inputs (the tile plan's occupancy).
constexpr int kSpThreads = 256;
constexpr int kSpPer = 16;
constexpr int kSpTile = kSpThreads * kSpPer;
constexpr unsigned long long kSpValMask = (1ull << 46) - 1ull;

__device__ __forceinline__ unsigned long long sp_word(unsigned epoch, unsigned flag, unsigned long long v) {
    return ((unsigned long long)epoch << 48) | ((unsigned long long)flag << 46) | (v & kSpValMask);
}

template <class TI, class TO>
__global__ void __launch_bounds__(kSpThreads) scan_onepass_kernel(
    const TI* __restrict__ in, TO* __restrict__ out, int64_t n, int64_t ntiles,
    unsigned long long* __restrict__ st, unsigned epoch, unsigned long long* total,
    unsigned long long* sumsq) {
    __shared__ unsigned long long ws[kSpThreads / 32];
    __shared__ unsigned long long s_excl;
    __shared__ int64_t s_tile;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned* ticket = reinterpret_cast<unsigned*>(st);   // st[0]: the ticket counter
    volatile unsigned long long* flags = st + 1;
    if (threadIdx.x == 0) {
        int64_t t = atomicAdd(ticket, 1u);
        if (t == ntiles - 1) *ticket = 0u;   // every ticket of this launch is taken
        s_tile = t;
    }
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t i0 = tile * kSpTile + (int64_t)threadIdx.x * kSpPer;
    unsigned long long v[kSpPer], loc = 0, sq = 0;
    if (sizeof(TI) == 4 && i0 + kSpPer <= n && ((uintptr_t)in & 15) == 0) {   // a full run: four 16-byte loads
        const int4* p4 = reinterpret_cast<const int4*>(in + i0);
#pragma unroll
        for (int k = 0; k < kSpPer / 4; ++k) {
            const int4 q = p4[k];
            v[4 * k] = (unsigned)q.x;
            v[4 * k + 1] = (unsigned)q.y;
            v[4 * k + 2] = (unsigned)q.z;
            v[4 * k + 3] = (unsigned)q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kSpPer; ++k) v[k] = i0 + k < n ? (unsigned long long)in[i0 + k] : 0ull;
    }
#pragma unroll
    for (int k = 0; k < kSpPer; ++k) {
        loc += v[k];
        sq += v[k] * v[k];
    }
    if (sumsq) {
        for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0 && sq) atomicAdd(sumsq, sq);
    }
    // block exclusive scan of the per-thread sums
    unsigned long long inc = loc;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
        unsigned long long x = lane < kSpThreads / 32 ? ws[lane] : 0ull, xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        const unsigned long long agg = __shfl_sync(0xffffffffu, xi, kSpThreads / 32 - 1);
        if (lane < kSpThreads / 32) ws[lane] = xi - x;
        // publish, then look back
        unsigned long long excl = 0;
        if (tile == 0) {
            if (lane == 0) flags[0] = sp_word(epoch, 2, agg);
        } else {
            if (lane == 0) flags[tile] = sp_word(epoch, 1, agg);
            int64_t p = tile - 1;
            for (;;) {
                const int64_t q = p - lane;
                unsigned long long wv = 0;
                unsigned fl = 2;   // before tile 0: nothing to add, stop
                if (q >= 0) {
                    do {
                        wv = flags[q];
                    } while ((unsigned)(wv >> 48) != epoch || ((wv >> 46) & 3ull) == 0ull);
                    fl = (unsigned)((wv >> 46) & 3ull);
                }
                const unsigned pm = __ballot_sync(0xffffffffu, fl == 2);
                const int stop = pm ? __ffs(pm) - 1 : 31;   // the nearest inclusive prefix
                unsigned long long add = (lane <= stop && q >= 0) ? (wv & kSpValMask) : 0ull;
                for (int o = 16; o; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
                excl += add;
                if (pm) break;
                p -= 32;
            }
            if (lane == 0) flags[tile] = sp_word(epoch, 2, excl + agg);
        }
        if (lane == 0) {
            s_excl = excl;
            if (tile == ntiles - 1 && total) *total = excl + agg;
        }
    }
    __syncthreads();
    unsigned long long e = s_excl + ws[w] + (inc - loc);
    if (sizeof(TO) == 4 && i0 + kSpPer <= n && ((uintptr_t)out & 15) == 0) {   // four 16-byte stores
        int4* o4 = reinterpret_cast<int4*>(out + i0);
#pragma unroll
        for (int k = 0; k < kSpPer / 4; ++k) {
            int4 q;
            q.x = (int)e; e += v[4 * k];
            q.y = (int)e; e += v[4 * k + 1];
            q.z = (int)e; e += v[4 * k + 2];
            q.w = (int)e; e += v[4 * k + 3];
            o4[k] = q;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kSpPer; ++k) {
            if (i0 + k < n) out[i0 + k] = (TO)e;
            e += v[k];
        }
    }
}

template <class TI, class TO>
static void scan_impl(Context& c, const TI* in, TO* out, int64_t n, unsigned long long* total,
                      unsigned long long* sumsq) {
    int64_t nt = (n + kSpTile - 1) / kSpTile;
    if (nt < 1) nt = 1;
    DBuf<unsigned long long>& st = c.scan_tmp;
    const unsigned long long* before = st.p;
    st.ensure((size_t)nt + 2);
    if (st.p != before || ++c.scan_epoch >= 65536u) {   // fresh memory or the epoch wrapped
        cudaMemsetAsync(st.p, 0, st.cap * sizeof(unsigned long long), c.stream);
        c.scan_epoch = 1;
    }
    scan_onepass_kernel<TI, TO><<<(unsigned)nt, kSpThreads, 0, c.stream>>>(in, out, n, nt, st.p, c.scan_epoch,
                                                                           total, sumsq), note_launch();
}

void exclusive_scan_i32(Context& c, const int* in, int* out, int64_t n, unsigned long long* total,
                        unsigned long long* sumsq) {
    scan_impl<int, int>(c, in, out, n, total, sumsq);
}

void exclusive_scan_i32_to_i64(Context& c, const int* in, long long* out, int64_t n,
                               unsigned long long* total) {
    scan_impl<int, long long>(c, in, out, n, total, nullptr);
}

// ---------------------------------------------------------------- scalars to host

__global__ void scal_to_host_kernel(const unsigned long long* __restrict__ src, int count,
                                    unsigned long long* __restrict__ dst) {
    if (threadIdx.x < count) dst[threadIdx.x] = src[threadIdx.x];
}

void scal_to_host(Context& c, const unsigned long long* src, int count, unsigned long long* dst_mapped) {
    scal_to_host_kernel<<<1, 32, 0, c.stream>>>(src, count, dst_mapped), note_launch();
}

// ---------------------------------------------------------------- binning

struct BinParams {
    double cl[3];
    int S[3], H[3], D[3], periodic[3];
    int64_t n;
};

// bin_cell_coords (cells.py:114-119): floor(x / cell_len) with IEEE division,
// clipped to the owned range; NaN/inf land in cell 0 like numpy's cast+clip.
__device__ __forceinline__ int cell_coord(double x, double cl, int S) {
    double f = floor(x / cl);
    if (!(f >= 0.0)) return 0;            // negative, NaN, -inf
    if (f > (double)(S - 1)) return S - 1;  // includes +inf
    return (int)f;
}

template <int LAYOUT>
__device__ __forceinline__ void load_pos(const double* pos, int64_t i, int64_t n, double& x,
                                         double& y, double& z) {
    x = pos[pidx<LAYOUT>(i, 0, n)];
    y = pos[pidx<LAYOUT>(i, 1, n)];
    z = pos[pidx<LAYOUT>(i, 2, n)];
}

// Image combos in the reference's product order (cells.py:134-150): axis
// options (-1, 0, 1) on periodic axes, the combo (0,0,0) skipped; an image
// exists when every nonzero shift is allowed (s>0: c<H, s<0: c>=S-H).
// `fn(code, cell)` is called per image in that order; returns the count.
template <class F>
__device__ __forceinline__ int for_each_image(const BinParams& p, const int c[3], F fn) {
    int cnt = 0;
    int lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
        lo[k] = p.periodic[k] ? -1 : 0;
        hi[k] = p.periodic[k] ? 1 : 0;
    }
    for (int sx = lo[0]; sx <= hi[0]; ++sx) {
        if ((sx > 0 && !(c[0] < p.H[0])) || (sx < 0 && !(c[0] >= p.S[0] - p.H[0]))) continue;
        for (int sy = lo[1]; sy <= hi[1]; ++sy) {
            if ((sy > 0 && !(c[1] < p.H[1])) || (sy < 0 && !(c[1] >= p.S[1] - p.H[1]))) continue;
            for (int sz = lo[2]; sz <= hi[2]; ++sz) {
                if (!sx && !sy && !sz) continue;
                if ((sz > 0 && !(c[2] < p.H[2])) || (sz < 0 && !(c[2] >= p.S[2] - p.H[2]))) continue;
                int ix = c[0] + sx * p.S[0] + p.H[0];
                int iy = c[1] + sy * p.S[1] + p.H[1];
                int iz = c[2] + sz * p.S[2] + p.H[2];
                int code = (sx + 1) * 9 + (sy + 1) * 3 + (sz + 1);
                fn(code, (ix * p.D[1] + iy) * p.D[2] + iz);
                ++cnt;
            }
        }
    }
    return cnt;
}

template <int LAYOUT>
__global__ void bin_count_kernel(const double* __restrict__ pos, BinParams p,
                                 int* __restrict__ cell_count, int* __restrict__ img_cnt,
                                 unsigned long long* scal) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        // this rebuild's accumulators in the context scalars, zeroed here
        // instead of by memset launches: [9] sum of squared cell occupancies
        // (the cell-count scan), and the Verlet build's [3] longest list, [5]
        // max |coordinate|, [7] overflow tiles
        scal[3] = 0;
        scal[5] = 0;
        scal[7] = 0;
        scal[9] = 0;
    }
    if (i >= p.n) return;
    double x, y, z;
    load_pos<LAYOUT>(pos, i, p.n, x, y, z);
    int c[3] = {cell_coord(x, p.cl[0], p.S[0]), cell_coord(y, p.cl[1], p.S[1]),
                cell_coord(z, p.cl[2], p.S[2])};
    int own = ((c[0] + p.H[0]) * p.D[1] + c[1] + p.H[1]) * p.D[2] + c[2] + p.H[2];
    atomicAdd(cell_count + own, 1);
    int k = for_each_image(p, c, [&](int, int cell) { atomicAdd(cell_count + cell, 1); });
    img_cnt[i] = k;
}

template <int LAYOUT>
__global__ void bin_scatter_kernel(const double* __restrict__ pos, BinParams p,
                                   const int* __restrict__ cell_start, int* __restrict__ cell_count,
                                   const int* __restrict__ img_off, int* __restrict__ img_src,
                                   uint8_t* __restrict__ img_code, int* __restrict__ tmp_ent) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    double x, y, z;
    load_pos<LAYOUT>(pos, i, p.n, x, y, z);
    int c[3] = {cell_coord(x, p.cl[0], p.S[0]), cell_coord(y, p.cl[1], p.S[1]),
                cell_coord(z, p.cl[2], p.S[2])};
    int own = ((c[0] + p.H[0]) * p.D[1] + c[1] + p.H[1]) * p.D[2] + c[2] + p.H[2];
    {
        int slot = cell_start[own] + atomicSub(cell_count + own, 1) - 1;   // the in-cell order comes from cell_sort
        MDG_DCHECK(slot >= cell_start[own] && slot < cell_start[own + 1]);
        tmp_ent[slot] = (int)i;
    }
    int base = img_off[i];
    int q = 0;
    for_each_image(p, c, [&](int code, int cell) {
        int e = base + q;
        img_src[e] = (int)i;
        img_code[e] = (uint8_t)code;
        int slot = cell_start[cell] + atomicSub(cell_count + cell, 1) - 1;
        MDG_DCHECK(slot >= cell_start[cell] && slot < cell_start[cell + 1]);
        tmp_ent[slot] = (int)(p.n + e);
        ++q;
    });
}

// Per-cell ordering fix: entries of one cell sorted by entry id (== the
// reference's stable argsort order, containers.py:107).  One warp per cell;
// cells up to 32 entries rank through shuffles, larger ones by counting.
// Rank each cell's entries (one warp per cell).  KEYZ = 0: by entry id, the
// reference's stable order (containers.py:107).  KEYZ = 1: by the entry's z
// coordinate, ties by id -- the cluster-list grid only (vcl.cu), where 8
// consecutive rows then form a compact slab of the cell; every entry of a
// cell shares one shift, so the unshifted z orders them.
template <int KEYZ, int PLAYOUT>
__global__ void cell_sort_kernel(int64_t ncells, int64_t n, const int* __restrict__ cell_start,
                                 const int* __restrict__ tmp_ent, const int* __restrict__ img_src,
                                 const uint8_t* __restrict__ img_code, const int* __restrict__ tid,
                                 const double* __restrict__ pos,
                                 int* __restrict__ row_ent, int* __restrict__ row_src,
                                 uint8_t* __restrict__ row_code, int* __restrict__ row_cell,
                                 int* __restrict__ row_tid, int* __restrict__ inv) {
    int64_t cell = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (cell >= ncells) return;
    int s = cell_start[cell], e = cell_start[cell + 1], k = e - s;
    if (k == 0) return;
    auto src_of = [&](int ent) { return ent < n ? ent : img_src[ent - n]; };
    auto key_of = [&](int ent) { return KEYZ ? pos[pidx<PLAYOUT>(src_of(ent), 2, n)] : 0.0; };
    auto before = [&](double ko, int o, double kv, int v) {
        return KEYZ ? (ko < kv || (ko == kv && o < v)) : o < v;
    };
    auto emit = [&](int r, int ent) {
        row_ent[r] = ent;
        int src = src_of(ent);
        row_src[r] = src;
        row_code[r] = ent < n ? (uint8_t)kNoShift : img_code[ent - n];
        row_cell[r] = (int)cell;
        row_tid[r] = tid ? tid[src] : 0;
        inv[ent] = r;
    };
    if (k <= 32) {
        int v = lane < k ? tmp_ent[s + lane] : 0x7fffffff;
        double kv = lane < k ? key_of(v) : INFINITY;
        int rank = 0;
        for (int j = 0; j < k; ++j) {   // k is the same for the whole warp
            int o = __shfl_sync(0xffffffffu, v, j);
            double ko = KEYZ ? __shfl_sync(0xffffffffu, kv, j) : 0.0;
            rank += before(ko, o, kv, v);
        }
        MDG_DCHECK(lane >= k || rank < k);
        if (lane < k) emit(s + rank, v);
    } else {
        for (int a = lane; a < k; a += 32) {
            int v = tmp_ent[s + a], rank = 0;
            double kv = key_of(v);
            for (int b = 0; b < k; ++b) {
                int o = tmp_ent[s + b];
                rank += before(key_of(o), o, kv, v);
            }
            MDG_DCHECK(rank < k);
            emit(s + rank, v);
        }
    }
}

int grid_rebuild(Context& c, Grid& gr, const double* pos, int layout) {
    cudaStream_t st = c.stream;
    int64_t n = c.n;
    gr.n = n;
    BinParams p;
    for (int k = 0; k < 3; ++k) {
        p.cl[k] = gr.g.cl[k]; p.S[k] = gr.g.S[k]; p.H[k] = gr.g.H[k];
        p.D[k] = gr.g.D[k]; p.periodic[k] = gr.g.periodic[k];
    }
    p.n = n;
    int64_t nc = gr.g.ncells;
    // cell_count returns to zero by itself: bin_scatter claims slots by
    // counting it back down, so a completed rebuild leaves it clear for the
    // next one (no memset launches; cleared only after a fresh allocation,
    // a change of grid or an abandoned rebuild)
    const int* before = gr.cell_count.p;
    gr.cell_count.ensure(nc + 1);
    gr.cell_start.ensure(nc + 1);
    gr.img_cnt.ensure(n + 1);
    gr.img_off.ensure(n + 1);
    if (gr.cell_count.p != before || gr.counts_clear != nc + 1) {
        MDG_CUDA(cudaMemsetAsync(gr.cell_count.p, 0, (nc + 1) * sizeof(int), st));
    }
    gr.counts_clear = 0;   // until this rebuild's scatter has counted them down
    unsigned long long* occ2 = c.scal.p + 9;
    if (n == 0) MDG_CUDA(cudaMemsetAsync(occ2, 0, sizeof(unsigned long long), st));
    if (n > 0) {
        if (layout == AOS)
            bin_count_kernel<AOS><<<blocks_for(n, 256), 256, 0, st>>>(pos, p, gr.cell_count.p, gr.img_cnt.p, c.scal.p), note_launch();
        else
            bin_count_kernel<SOA><<<blocks_for(n, 256), 256, 0, st>>>(pos, p, gr.cell_count.p, gr.img_cnt.p, c.scal.p), note_launch();
    }
    // images total and cell offsets (+ the Verlet grid's squared occupancies);
    // one copy brings [1] the image count, [2] the status word (mdg_rebuild_checked)
    // and [9] the occupancy sum to the pinned mirror
    exclusive_scan_i32(c, gr.img_cnt.p, gr.img_off.p, n, c.scal.p + 1);
    exclusive_scan_i32(c, gr.cell_count.p, gr.cell_start.p, nc + 1, nullptr, gr.sort_by_z ? occ2 : nullptr);
    scal_to_host(c, c.scal.p + 1, 9, c.d_h_scal + 1);   // (mapped pinned: no copy-engine bubble)
    static const bool trace = getenv("MDG_STEP_TRACE") != nullptr;   // host ms of this wait, when long
    const auto t0 = std::chrono::steady_clock::now();
    MDG_CUDA(cudaStreamSynchronize(st));
    if (trace) {
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > 3.5) fprintf(stderr, "mdg grid_rebuild: waited %.3f ms for the stream\n", ms);
    }
    if (c.flags_probe) {   // status word copied before this rebuild's first kernel
        c.flags_probe = false;
        c.flags_seen = (unsigned)(c.h_scal[2] & 3ull);
        if (c.flags_seen) {
            gr.built = false;
            set_error("status flags raised");
            return -1;
        }
    }
    gr.nimg = (int64_t)c.h_scal[1];
    gr.m = n + gr.nimg;
    gr.occ2 = gr.sort_by_z && n > 0 ? (double)c.h_scal[9] : 0.0;
    int64_t m = gr.m;
    gr.img_src.ensure(gr.nimg + 1);
    gr.img_code.ensure(gr.nimg + 1);
    gr.tmp_ent.ensure(m + 1);
    gr.row_ent.ensure(m + 1);
    gr.row_src.ensure(m + 1);
    gr.row_code.ensure(m + 1);
    gr.row_cell.ensure(m + 1);
    gr.row_tid.ensure(m + 1);
    gr.inv.ensure(m + 1);
    if (n > 0) {
        if (layout == AOS)
            bin_scatter_kernel<AOS><<<blocks_for(n, 256), 256, 0, st>>>(
                pos, p, gr.cell_start.p, gr.cell_count.p, gr.img_off.p, gr.img_src.p, gr.img_code.p,
                gr.tmp_ent.p), note_launch();
        else
            bin_scatter_kernel<SOA><<<blocks_for(n, 256), 256, 0, st>>>(
                pos, p, gr.cell_start.p, gr.cell_count.p, gr.img_off.p, gr.img_src.p, gr.img_code.p,
                gr.tmp_ent.p), note_launch();
#define MDG_CSORT(KZ, PL)                                                                       \
    cell_sort_kernel<KZ, PL><<<blocks_for(nc * 32, 256), 256, 0, st>>>(                          \
        nc, n, gr.cell_start.p, gr.tmp_ent.p, gr.img_src.p, gr.img_code.p, c.tid, pos,            \
        gr.row_ent.p, gr.row_src.p, gr.row_code.p, gr.row_cell.p, gr.row_tid.p, gr.inv.p), note_launch()
        if (!gr.sort_by_z) MDG_CSORT(0, AOS);
        else if (layout == AOS) MDG_CSORT(1, AOS);
        else MDG_CSORT(1, SOA);
#undef MDG_CSORT
    }
    MDG_CUDA(cudaGetLastError());
    gr.built = true;
    gr.counts_clear = nc + 1;   // the scatter counted every cell back to zero
    ++gr.build_id;
    gr.scratch_layout = -1;
    return 0;
}

// ---------------------------------------------------------------- owned order

__global__ void owned_flag_kernel(int m, const uint8_t* __restrict__ row_code, int* __restrict__ flag) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m) flag[r] = row_code[r] == kNoShift;
}

__global__ void owned_order_kernel(int m, const uint8_t* __restrict__ row_code,
                                   const int* __restrict__ row_src, const int* __restrict__ rank,
                                   int* __restrict__ out) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m && row_code[r] == kNoShift) out[rank[r]] = row_src[r];
}

// The particles in the grid's row order (owned rows only): out[k] = the
// particle of the k-th owned row, a permutation of 0..n-1 (device buffer).
int grid_owned_order(Context& c, Grid& gr, int* out) {
    int m = (int)gr.m;
    if (m == 0) return 0;
    c.order_tmp.ensure(2 * (size_t)m + 2);
    if (!c.order_tmp.p) {
        set_error("out of device memory (owned order)");
        return -1;
    }
    int* flag = c.order_tmp.p;
    int* rank = c.order_tmp.p + m + 1;
    owned_flag_kernel<<<blocks_for(m, 256), 256, 0, c.stream>>>(m, gr.row_code.p, flag), note_launch();
    exclusive_scan_i32(c, flag, rank, m, nullptr);
    owned_order_kernel<<<blocks_for(m, 256), 256, 0, c.stream>>>(m, gr.row_code.p, gr.row_src.p, rank, out), note_launch();
    MDG_CUDA(cudaGetLastError());
    return 0;
}

// ---------------------------------------------------------------- scratch

void grid_bind_scratch(Context& c, Grid& gr, int layout) {
    int64_t m = gr.m;
    if (layout == AOS) gr.spos4.ensure(m + 1);
    else gr.spos3.ensure(3 * m + 3);
    gr.sforce.ensure(3 * m + 3);
    gr.scratch_layout = layout;
}

struct ShiftL {
    double L[3];
};

__device__ __forceinline__ void decode_shift(int code, const ShiftL& s, double& dx, double& dy,
                                             double& dz) {
    // shift = combo * L exactly (cells.py:146), combo in {-1,0,1}
    dx = (double)(code / 9 - 1) * s.L[0];
    dy = (double)((code / 3) % 3 - 1) * s.L[1];
    dz = (double)(code % 3 - 1) * s.L[2];
}

// LayoutBuffers.refresh (containers.py:147-154): pos[src] + shift per row.
template <int PLAYOUT, int SLAYOUT>
__global__ void refresh_kernel(const double* __restrict__ pos, int64_t n, int m,
                               const int* __restrict__ row_src, const uint8_t* __restrict__ row_code,
                               const int* __restrict__ row_tid, ShiftL sl, double4* __restrict__ s4,
                               double* __restrict__ s3) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    int src = row_src[r];
    double sx, sy, sz;
    decode_shift(row_code[r], sl, sx, sy, sz);
    double x = pos[pidx<PLAYOUT>(src, 0, n)] + sx;
    double y = pos[pidx<PLAYOUT>(src, 1, n)] + sy;
    double z = pos[pidx<PLAYOUT>(src, 2, n)] + sz;
    if (SLAYOUT == AOS) {
        s4[r] = make_double4(x, y, z, (double)row_tid[r]);
    } else {
        s3[r] = x;
        s3[(size_t)m + r] = y;
        s3[2 * (size_t)m + r] = z;
    }
}

void grid_refresh(Context& c, Grid& gr, int layout) {
    int m = (int)gr.m;
    if (m == 0) return;
    ShiftL sl{{c.L[0], c.L[1], c.L[2]}};
    dim3 b(blocks_for(m, 256)), t(256);
    // the scratch layout follows the configuration; the particle arrays follow
    // the ParticleSet (they agree after convert_layout, simulation.py:161-163)
    if (c.layout == AOS) {
        if (layout == AOS)
            refresh_kernel<AOS, AOS><<<b, t, 0, c.stream>>>(c.pos, c.n, m, gr.row_src.p, gr.row_code.p, gr.row_tid.p, sl, gr.spos4.p, gr.spos3.p), note_launch();
        else
            refresh_kernel<AOS, SOA><<<b, t, 0, c.stream>>>(c.pos, c.n, m, gr.row_src.p, gr.row_code.p, gr.row_tid.p, sl, gr.spos4.p, gr.spos3.p), note_launch();
    } else {
        if (layout == AOS)
            refresh_kernel<SOA, AOS><<<b, t, 0, c.stream>>>(c.pos, c.n, m, gr.row_src.p, gr.row_code.p, gr.row_tid.p, sl, gr.spos4.p, gr.spos3.p), note_launch();
        else
            refresh_kernel<SOA, SOA><<<b, t, 0, c.stream>>>(c.pos, c.n, m, gr.row_src.p, gr.row_code.p, gr.row_tid.p, sl, gr.spos4.p, gr.spos3.p), note_launch();
    }
}

// LayoutBuffers.scatter_forces (containers.py:156-171) as a gather: owned row
// assigned, image rows added (images of one particle in combo order).
// ncol > 0: the scratch forces are ncol colour partials (the one-launch
// small-system C08, lc.cu), added here in colour order per row.
template <int PLAYOUT, int SLAYOUT>
__global__ void fold_kernel(int64_t n, int m, const int* __restrict__ inv,
                            const int* __restrict__ img_cnt, const int* __restrict__ img_off,
                            const double* __restrict__ sf, double* __restrict__ force,
                            bool images, int ncol) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto get = [&](int r, int k) {
        const size_t e = SLAYOUT == AOS ? 3 * (size_t)r + k : (size_t)k * m + r;
        if (ncol == 0) return sf[e];
        double v[8];   // independent loads first, then the colour-order sum
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = q < ncol ? sf[(size_t)q * 3 * m + e] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < ncol) s += v[q];
        return s;
    };
    int r0 = inv[i];
    double fx = get(r0, 0), fy = get(r0, 1), fz = get(r0, 2);
    if (images) {
        int q0 = img_off[i], nq = img_cnt[i];
        // up to 7 images (3 periodic axes): their rows and forces loaded
        // together (independent loads), then added in combo order -- a
        // particle's chain of dependent loads is 3 deep, not 2 per image
        if (nq <= 7) {
            int rr[7];
#pragma unroll
            for (int q = 0; q < 7; ++q) rr[q] = q < nq ? inv[n + q0 + q] : r0;
            double gx[7], gy[7], gz[7];
#pragma unroll
            for (int q = 0; q < 7; ++q) {
                gx[q] = q < nq ? get(rr[q], 0) : 0.0;
                gy[q] = q < nq ? get(rr[q], 1) : 0.0;
                gz[q] = q < nq ? get(rr[q], 2) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 7; ++q)
                if (q < nq) {
                    fx += gx[q];
                    fy += gy[q];
                    fz += gz[q];
                }
        } else {
            for (int q = 0; q < nq; ++q) {
                int r = inv[n + q0 + q];
                fx += get(r, 0);
                fy += get(r, 1);
                fz += get(r, 2);
            }
        }
    }
    force[pidx<PLAYOUT>(i, 0, n)] = fx;
    force[pidx<PLAYOUT>(i, 1, n)] = fy;
    force[pidx<PLAYOUT>(i, 2, n)] = fz;
}

void lc_fold_forces(Context& c, Grid& gr, int layout, bool images) {
    if (c.n == 0) return;
    dim3 b(blocks_for(c.n, 256)), t(256);
    int m = (int)gr.m;
    const int ncol = gr.cpart_ncol;
    const double* sfp = ncol ? gr.cpart.p : gr.sforce.p;
    if (c.layout == AOS) {
        if (layout == AOS)
            fold_kernel<AOS, AOS><<<b, t, 0, c.stream>>>(c.n, m, gr.inv.p, gr.img_cnt.p, gr.img_off.p, sfp, c.force, images, ncol), note_launch();
        else
            fold_kernel<AOS, SOA><<<b, t, 0, c.stream>>>(c.n, m, gr.inv.p, gr.img_cnt.p, gr.img_off.p, sfp, c.force, images, ncol), note_launch();
    } else {
        if (layout == AOS)
            fold_kernel<SOA, AOS><<<b, t, 0, c.stream>>>(c.n, m, gr.inv.p, gr.img_cnt.p, gr.img_off.p, sfp, c.force, images, ncol), note_launch();
        else
            fold_kernel<SOA, SOA><<<b, t, 0, c.stream>>>(c.n, m, gr.inv.p, gr.img_cnt.p, gr.img_off.p, sfp, c.force, images, ncol), note_launch();
    }
}

}  // namespace mdg
