// Temperature, thermostat and live statistics on the device (SURVEY §8(f)
// rows 2 and 4), bit-identical to the reference's numpy arithmetic.
//
// Reference: integrator.py:72-78 (current_temperature), :81-95
// (apply_thermostat), simulation.py:186-188 (thermostat cadence),
// livestats.py:46-77 (compute_live_stats, the features the selectors read).
//
// Every sum the reference takes is np.sum / np.mean over a contiguous fp64
// array, i.e. numpy's pairwise reduction.  The PairwiseTree below replays
// exactly that association (planned on the host once per length): leaves
// are summed by one thread each with the same 8 strided accumulators, then
// the internal nodes are combined height by height in one block.  No float
// atomics anywhere, so the result is deterministic and equals np.sum.
#include <limits.h>
#include <math.h>

#include <algorithm>

#include "device.cuh"

namespace mdg {

constexpr int kPwBlock = 128;   // numpy PW_BLOCKSIZE

void PairwiseTree::release() {
    leaves.release();
    nodes.release();
    d_level_off.release();
    val.release();
    n = -1;
}

// ------------------------------------------------------------------ planning

namespace {

struct PlanState {
    std::vector<PwLeaf> leaves;
    std::vector<int4> nodes;      // {left, right, out(internal idx), height}
};

// returns {slot, height}; internal slots are encoded as -(k+1) until the
// leaf count is known
std::pair<int, int> plan_rec(PlanState& st, long long off, long long n) {
    if (n <= kPwBlock) {
        st.leaves.push_back(PwLeaf{off, (int)n, 0});
        return {(int)st.leaves.size() - 1, 0};
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    auto l = plan_rec(st, off, n2);
    auto r = plan_rec(st, off + n2, n - n2);
    int h = std::max(l.second, r.second) + 1;
    st.nodes.push_back(int4{l.first, r.first, 0, h});
    return {-(int)st.nodes.size(), h};
}

int plan(PairwiseTree& t, int64_t n, cudaStream_t s) {
    if (t.n == n) return 0;
    PlanState st;
    auto root = plan_rec(st, 0, n);
    int L = (int)st.leaves.size();
    auto slot = [L](int enc) { return enc >= 0 ? enc : L + (-enc - 1); };
    int nint = (int)st.nodes.size();
    std::vector<int> order(nint);
    for (int k = 0; k < nint; ++k) order[k] = k;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return st.nodes[a].w < st.nodes[b].w; });
    std::vector<int4> flat(std::max(nint, 1));
    t.level_off.assign(1, 0);
    int cur_h = 1;
    for (int k = 0; k < nint; ++k) {
        const int4& nd = st.nodes[order[k]];
        while (nd.w > cur_h) {
            t.level_off.push_back(k);
            ++cur_h;
        }
        flat[k] = int4{slot(nd.x), slot(nd.y), L + order[k], 0};
    }
    t.level_off.push_back(nint);
    t.nleaves = L;
    t.root = slot(root.first);
    t.leaves.ensure(L);
    t.nodes.ensure(flat.size());
    t.d_level_off.ensure(t.level_off.size());
    t.val.ensure((size_t)L + nint);
    if (!t.leaves.p || !t.nodes.p || !t.d_level_off.p || !t.val.p) {
        set_error("out of device memory (pairwise plan)");
        return -1;
    }
    MDG_CUDA(cudaMemcpyAsync(t.leaves.p, st.leaves.data(), L * sizeof(PwLeaf),
                             cudaMemcpyHostToDevice, s));
    MDG_CUDA(cudaMemcpyAsync(t.nodes.p, flat.data(), flat.size() * sizeof(int4),
                             cudaMemcpyHostToDevice, s));
    MDG_CUDA(cudaMemcpyAsync(t.d_level_off.p, t.level_off.data(),
                             t.level_off.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    // the staging vectors die here; make the copies complete first
    MDG_CUDA(cudaStreamSynchronize(s));
    t.n = n;
    return 0;
}

}  // namespace

// ------------------------------------------------------------------- kernels

// numpy pairwise_sum leaf (loops_utils.h): n < 8 sequential from -0.0, else
// 8 accumulators over the multiple-of-8 prefix, combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail sequentially.
template <class Elem>
__device__ double pw_leaf(const Elem& f, long long off, int n) {
    if (n < 8) {
        double res = -0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, f(off + i));
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(off + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(off + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, f(off + i));
    return res;
}

template <class Elem>
__global__ void pw_leaves_kernel(Elem f, const PwLeaf* __restrict__ leaves, int nleaves,
                                 double* __restrict__ val) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nleaves) return;
    PwLeaf lf = leaves[k];
    val[k] = pw_leaf(f, lf.off, lf.len);
}

// m_i * sum(v_i * v_i) with the row sum left to right (integrator.py:77:
// np.sum(masses * np.sum(v * v, axis=1)); a 3-element row reduces
// sequentially in numpy).
template <int LAYOUT>
struct KineticElem {
    const double* __restrict__ vel;
    const double* __restrict__ mass;
    const int* __restrict__ tid;
    int64_t n;
    __device__ __forceinline__ double operator()(long long i) const {
        double vx = vel[pidx<LAYOUT>(i, 0, n)];
        double vy = vel[pidx<LAYOUT>(i, 1, n)];
        double vz = vel[pidx<LAYOUT>(i, 2, n)];
        double s = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
        return __dmul_rn(mass[tid ? tid[i] : 0], s);
    }
};

// (counts - mean) ** 2 (livestats.py:63); numpy squares with x * x.
struct BinDevElem {
    const int* __restrict__ counts;
    double mean;
    __device__ __forceinline__ double operator()(long long i) const {
        double d = __dadd_rn((double)counts[i], -mean);
        return __dmul_rn(d, d);
    }
};

enum Epilogue { EPI_TEMPERATURE = 0, EPI_THERMOSTAT = 1, EPI_LIVE_STATS = 2 };

struct EpiArgs {
    int mode;
    int64_t n;            // particles (temperature) or bins (live stats)
    double target, max_dt;
    double mean;          // live stats: particles per bin
    const int* hist;      // live stats: histogram of bin counts (n_particles + 1)
    long long median_rank;
    unsigned long long* flags;
    double* out;          // temperature: out[0] = T, out[1] = velocity scale
};

// Height-by-height combine of the internal nodes, then the reference's
// scalar epilogue on thread 0.
__global__ void pw_combine_kernel(const int4* __restrict__ nodes, const int* __restrict__ level_off,
                                  int nlevels, double* __restrict__ val, int root, EpiArgs a) {
    for (int l = 0; l < nlevels; ++l) {
        int lo = level_off[l], hi = level_off[l + 1];
        for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
            int4 nd = nodes[k];
            val[nd.z] = __dadd_rn(val[nd.x], val[nd.y]);
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    double sum = val[root];
    if (a.mode == EPI_TEMPERATURE || a.mode == EPI_THERMOSTAT) {
        double t_cur = __ddiv_rn(sum, 3.0 * (double)a.n);
        double scale = 1.0;
        if (a.mode == EPI_THERMOSTAT) {
            if (t_cur == 0.0) {
                if (a.target > 0.0) atomicOr(a.flags, 2ull);
            } else {
                // np.clip(target - t_cur, -max, max) = min(max(x, lo), hi)
                double d = __dadd_rn(a.target, -t_cur);
                double lo = -a.max_dt, hi = a.max_dt;
                if (d < lo) d = lo;
                if (d > hi) d = hi;
                double t_next = __dadd_rn(t_cur, d);
                scale = __dsqrt_rn(__ddiv_rn(t_next, t_cur));
            }
        }
        a.out[0] = t_cur;
        a.out[1] = scale;
    } else {
        // livestats.py:61-73
        double rel = 0.0;
        if (a.mean > 0.0)
            rel = __ddiv_rn(__dsqrt_rn(__ddiv_rn(sum, (double)a.n)), a.mean);
        long long acc = 0;
        int median = 0;
        for (int v = 0;; ++v) {
            acc += a.hist[v];
            if (acc > a.median_rank) {
                median = v;
                break;
            }
        }
        a.out[2] = a.mean;
        a.out[3] = rel;
        a.out[4] = (double)median;
        a.out[6] = (double)a.n;
        a.out[7] = (double)a.hist[0];
        // out[5] (max) was written by bin_summary_kernel
    }
}

template <int LAYOUT>
__global__ void scale_velocity_kernel(double* __restrict__ vel, int64_t n,
                                      const double* __restrict__ scale) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    double s = scale[1];
    vel[i] = __dmul_rn(vel[i], s);   // vel[:] *= sqrt(t_next / t_cur)
}

struct BinGeom {
    double len[3];
    long long dims[3];
};

// livestats.py:57-60: floor(pos / lengths) clipped to [0, dims-1]
template <int LAYOUT>
__global__ void bin_count_kernel(const double* __restrict__ pos, int64_t n, BinGeom g,
                                 int* __restrict__ counts) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double q = floor(__ddiv_rn(pos[pidx<LAYOUT>(i, k, n)], g.len[k]));
        // astype(int64): NaN / out of range give INT64_MIN on x86, then the clip
        long long v = (q >= -9.223372036854775808e18 && q < 9.223372036854775808e18)
                          ? (long long)q : LLONG_MIN;
        if (v < 0) v = 0;
        if (v > g.dims[k] - 1) v = g.dims[k] - 1;
        c[k] = v;
    }
    atomicAdd(counts + (c[0] * g.dims[1] + c[1]) * g.dims[2] + c[2], 1);
}

// histogram of bin counts (for the median and the empty-bin count) + max
__global__ void bin_summary_kernel(const int* __restrict__ counts, int64_t nbins,
                                   int* __restrict__ hist, double* __restrict__ out) {
    __shared__ int smax;
    if (threadIdx.x == 0) smax = 0;
    __syncthreads();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int c = i < nbins ? counts[i] : 0;
    if (i < nbins) atomicAdd(hist + c, 1);
    int wmax = __reduce_max_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) atomicMax(&smax, wmax);
    __syncthreads();
    // out[5] holds the max as a double; counts are non-negative, so the
    // int bit pattern of the running max lives in out[8]
    if (threadIdx.x == 0) atomicMax(reinterpret_cast<int*>(out + 8), smax);
}

__global__ void finalize_max_kernel(double* out) {
    out[5] = (double)*reinterpret_cast<const int*>(out + 8);
}

// ------------------------------------------------------------------- drivers

static void launch_combine(Context& c, PairwiseTree& t, const EpiArgs& a) {
    int nlev = (int)t.level_off.size() - 1;
    pw_combine_kernel<<<1, 1024, 0, c.stream>>>(t.nodes.p, t.d_level_off.p, nlev, t.val.p,
                                                t.root, a), note_launch();
}

template <int LAYOUT>
static void launch_kinetic(Context& c) {
    KineticElem<LAYOUT> f{c.vel, c.d_mass.p, c.tid, c.n};
    PairwiseTree& t = c.pw_particles;
    pw_leaves_kernel<<<blocks_for(t.nleaves, 128), 128, 0, c.stream>>>(f, t.leaves.p, t.nleaves,
                                                                       t.val.p), note_launch();
}

static int temperature_common(Context& c, int mode, double target, double max_dt) {
    if (c.n == 0) {
        set_error("temperature of an empty particle set is undefined");
        return 1;
    }
    if (plan(c.pw_particles, c.n, c.stream)) return -1;
    c.st_out.ensure(16);
    if (!c.st_out.p) { set_error("out of device memory"); return -1; }
    if (c.layout == AOS) launch_kinetic<AOS>(c);
    else launch_kinetic<SOA>(c);
    EpiArgs a{};
    a.mode = mode;
    a.n = c.n;
    a.target = target;
    a.max_dt = max_dt;
    a.flags = c.scal.p + 2;
    a.out = c.st_out.p;
    launch_combine(c, c.pw_particles, a);
    return 0;
}

int stats_temperature(Context& c, double* t) {
    if (int e = temperature_common(c, EPI_TEMPERATURE, 0.0, 0.0)) return e;
    MDG_CUDA(cudaMemcpyAsync(t, c.st_out.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    MDG_CUDA(cudaStreamSynchronize(c.stream));
    return 0;
}

int stats_thermostat(Context& c, double target, double max_delta_t) {
    if (int e = temperature_common(c, EPI_THERMOSTAT, target, max_delta_t)) return e;
    int64_t nv = 3 * c.n;
    // the layout only changes the order of the components, not the scaling
    scale_velocity_kernel<AOS><<<blocks_for(nv, 256), 256, 0, c.stream>>>(c.vel, c.n,
                                                                          c.st_out.p), note_launch();
    return 0;
}

int stats_live(Context& c, double out[6]) {
    // livestats.py:50-53, host side exactly as numpy: floor(L / ell) with a
    // true division, lengths = L / dims
    double ell = c.cutoff + c.skin;
    BinGeom g;
    long long nbins = 1;
    for (int k = 0; k < 3; ++k) {
        double q = floor(c.L[k] / ell);
        g.dims[k] = std::max<long long>(1, (long long)q);
        g.len[k] = c.L[k] / (double)g.dims[k];
        nbins *= g.dims[k];
    }
    if (nbins > (1ll << 31) - 1) { set_error("too many live-statistics bins"); return 1; }
    if (plan(c.pw_bins, nbins, c.stream)) return -1;
    c.ls_counts.ensure(nbins);
    c.ls_hist.ensure(c.n + 1);
    c.st_out.ensure(16);
    if (!c.ls_counts.p || !c.ls_hist.p || !c.st_out.p) { set_error("out of device memory"); return -1; }
    MDG_CUDA(cudaMemsetAsync(c.ls_counts.p, 0, nbins * sizeof(int), c.stream));
    MDG_CUDA(cudaMemsetAsync(c.ls_hist.p, 0, (c.n + 1) * sizeof(int), c.stream));
    MDG_CUDA(cudaMemsetAsync(c.st_out.p, 0, 16 * sizeof(double), c.stream));
    if (c.n) {
        if (c.layout == AOS)
            bin_count_kernel<AOS><<<blocks_for(c.n, 256), 256, 0, c.stream>>>(c.pos, c.n, g, c.ls_counts.p), note_launch();
        else
            bin_count_kernel<SOA><<<blocks_for(c.n, 256), 256, 0, c.stream>>>(c.pos, c.n, g, c.ls_counts.p), note_launch();
    }
    bin_summary_kernel<<<blocks_for(nbins, 256), 256, 0, c.stream>>>(c.ls_counts.p, nbins,
                                                                    c.ls_hist.p, c.st_out.p), note_launch();
    finalize_max_kernel<<<1, 1, 0, c.stream>>>(c.st_out.p), note_launch();
    double mean = (double)c.n / (double)nbins;   // livestats.py:61
    BinDevElem f{c.ls_counts.p, mean};
    PairwiseTree& t = c.pw_bins;
    pw_leaves_kernel<<<blocks_for(t.nleaves, 128), 128, 0, c.stream>>>(f, t.leaves.p, t.nleaves,
                                                                       t.val.p), note_launch();
    EpiArgs a{};
    a.mode = EPI_LIVE_STATS;
    a.n = nbins;
    a.mean = mean;
    a.hist = c.ls_hist.p;
    a.median_rank = (nbins - 1) / 2;
    a.flags = c.scal.p + 2;
    a.out = c.st_out.p;
    launch_combine(c, t, a);
    double h[8];
    MDG_CUDA(cudaMemcpyAsync(h, c.st_out.p, 8 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    MDG_CUDA(cudaStreamSynchronize(c.stream));
    for (int k = 0; k < 6; ++k) out[k] = h[2 + k];
    return 0;
}

void stats_release(Context& c) {
    c.pw_particles.release();
    c.pw_bins.release();
    c.ls_counts.release();
    c.ls_hist.release();
    c.st_out.release();
}

}  // namespace mdg
