// Internal header of libmdg: the B200 (sm_100a) LJ force + neighbour path.
//
// Everything here is device-resident.  The C ABI (include/mdg.h, api.cu) is the
// only surface; no torch types cross it.  Reference behaviour each piece
// mirrors is cited at the kernel that implements it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

// Device-side bounds checks (the build's checked variant, `make CHECKS=1` ->
// _build_checks/libmdg.so; compute-sanitizer is closed on the GPU pool):
// every shared-memory gather / scatter index, list slot and atomic-claimed
// slot the kernels derive is checked against its buffer; a violation prints
// the site and traps.  Compiled out of the product library.
#ifdef MDG_DEVICE_CHECKS
#define MDG_DCHECK(c)                                                                   \
    do {                                                                                \
        if (!(c)) {                                                                     \
            printf("MDG_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #c, (int)blockIdx.x, (int)threadIdx.x);                              \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define MDG_DCHECK(c) \
    do {              \
    } while (0)
#endif

#include <string>
#include <vector>

namespace mdg {

constexpr int kMaxTypes = 4;       // by-value LJ tables (kernel parameter space)
constexpr int kMaxStencil = 124;   // pruned stencil at CSF 0.5 (cells.py:80-95)
constexpr int kNoShift = 13;       // shift code of (0,0,0)

enum Layout { AOS = 0, SOA = 1 };

// Lorentz-Berthelot tables, forces.py:12-22, passed by value to every kernel.
struct LJTab {
    int T;
    double rc2;
    double sig2[kMaxTypes * kMaxTypes];
    double eps24[kMaxTypes * kMaxTypes];
};

struct Stencil {
    int n;
    int d[kMaxStencil][3];
};

// cells.py:20-67 (make_geometry) restated on the host side of the library.
struct Geom {
    double L[3];
    int periodic[3];
    double ell, csf;
    int S[3];          // dims_owned
    double cl[3];      // cell_length
    int overlap[3];
    int H[3];          // halo layers
    int D[3];          // padded dims
    int64_t ncells;
};

Geom make_geometry(const double L[3], const int periodic[3], double ell, double csf);
Stencil pruned_stencil(const Geom& g);
Stencil forward_stencil(const Geom& g, int major);

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    void ensure(size_t n);
    void release();
};

// One binning of the particles over a padded cell grid (containers.py:78-123):
// entries = N owned particles followed by periodic images (cells.py:122-156),
// stably counting-sorted by cell.  Within a cell the stable order equals
// ascending entry id (all entries of one cell share one image combo).
struct Grid {
    Geom g{};
    Stencil pruned{}, fwd{}, fwd_sli{};
    int sli_major = 0;
    int sort_by_z = 0;                              // in-cell order: 0 = entry id (reference), 1 = z (VCL)
    int64_t n = 0, nimg = 0, m = 0;
    // sum over cells of (rows in the cell)^2 at the last build: occ2 / m is the
    // cell occupancy the average row sees (the tile plan's density; the plain
    // mean undercounts slabs, droplets and vacuum)
    double occ2 = 0.0;
    bool built = false;
    DBuf<int> cell_count, cell_start;              // ncells + 1
    int64_t counts_clear = 0;                       // cell_count is all zero over this many entries
    DBuf<int> img_cnt, img_off;                     // n + 1
    DBuf<int> img_src;                              // nimg
    DBuf<uint8_t> img_code;                         // nimg
    DBuf<int> tmp_ent, row_ent;                     // m
    DBuf<int> row_src, row_cell, row_tid, inv;      // m
    DBuf<uint8_t> row_code;                         // m
    // layout-specific scratch (LayoutBuffers, containers.py:126-171)
    int scratch_layout = -1;
    DBuf<double4> spos4;                            // AoS: x,y,z,type
    DBuf<double> spos3;                             // SoA: x[m],y[m],z[m]
    DBuf<double> sforce;                            // 3*m ((m,3) AoS or (3,m) SoA)
    DBuf<double> cpart;                             // small-system C08: per-colour partial forces, colours x 3*m
    int cpart_ncol = 0;                             // > 0: the last compute left its forces in cpart (the fold adds them)
    size_t cpart_zero = 0;                          // leading doubles of cpart known to be zero
    int64_t build_id = 0;                           // bumped by every grid_rebuild
    // small-system C08: per-unit staged partner lists of build c08l_for (lc.cu C08Lists)
    DBuf<int> c08l_tot, c08l_j;
    DBuf<uint8_t> c08l_f;
    int64_t c08l_for = -1;
    void release();
};

// Verlet lists (containers.py:343-375) in the CSF-1 grid's row space:
// per-row counts + warp-blocked column-major int32 entries of width `cap`.
struct Verlet {
    Grid grid;
    DBuf<int> cnt;             // per row
    DBuf<int> nbr;             // ceil(m/32)*32*cap row indices
    int cap = 0;
    DBuf<float4> b32;          // fp32 build positions (membership pre-filter)
    DBuf<float4> q32;          // fp32 cell-relative positions + packed cell (fp32 variant)
    DBuf<double4> s4;          // unwrapped sorted positions {x,y,z,type} (AoS variant)
    DBuf<double> s3;           // x[m], y[m], z[m] (SoA variant)
    bool s3_valid = false;
    bool built = false;
    // shared-memory tiles of the force walk (vltile.cu)
    bool tiled = false;
    bool rows_valid = false;   // row-space lists (cnt/nbr) built for every row
    int ntiles = 0, nbig = 0, cap4 = 0, win_rows = 0;
    DBuf<int> tdesc;           // ntiles descriptors (TileDesc)
    DBuf<int> tsize, tbase;    // per tile: padded entry count, exclusive prefix
    DBuf<uint16_t> tl;         // window-local lists, 4-entry groups per lane
    DBuf<int> tcnt;            // per tile row slot: list length
    DBuf<uint8_t> big_row;     // 1 = row walked by the global-gather kernel
    // dynamic pruning of the tile lists (vltile.cu): inner lists of the pairs
    // within rp of the positions at the last prune, walked while every owned
    // row has moved less than (rp - rc) / 2 since then
    bool prune = false;
    double prune_rp2 = 0.0;
    float prune_thr = 0.f;
    DBuf<uint16_t> tl_in;      // inner lists, the layout of tl
    DBuf<int> tcnt_in;         // inner list lengths, the layout of tcnt
    // per 32-row list block, the longest row's count: [0, nblk) the full
    // lists, [nblk, 2 nblk) the inner ones; the walk's producer prefetches
    // only that much of each block into L2 (not the padded capacity)
    DBuf<int> bmax;
    int64_t nblk = 0;
    DBuf<float> disp;          // per row: path length since the last prune (rounded up)
    bool prune_ready = false;  // disp / pst allocated before this build (vlt_prune_prepare)
    DBuf<int> pst;             // [0] the next walk prunes, [1] prune walks since the build
    // the tile build's host check (list capacity, overflow tiles) deferred to
    // the first use of the lists (vlt_finish), so the host does not wait on
    // the build kernel with the stream empty behind it
    bool build_pending = false;
    cudaEvent_t ev_build = nullptr;
    unsigned long long* h_build = nullptr;   // pinned (mapped): the build's scalars, written by vlt_bmax_kernel
    unsigned long long* d_h_build = nullptr;
    int plan[5] = {0, 0, 0, 0, 0};           // ngx, ngy, nzt, tz, window budget
    void release();
};

// numpy's pairwise summation order (np.add.reduce over a contiguous fp64
// array: leaves of <= 128 elements summed with 8 strided accumulators, split
// at n/2 rounded down to a multiple of 8) planned once per length, so device
// reductions are bit-identical to the reference's np.sum (stats.cu).
struct PwLeaf {
    long long off;
    int len;
    int pad;
};

struct PairwiseTree {
    int64_t n = -1;
    int nleaves = 0, root = 0;
    std::vector<int> level_off;     // internal nodes grouped by height
    DBuf<PwLeaf> leaves;
    DBuf<int4> nodes;               // {left slot, right slot, out slot, -}
    DBuf<int> d_level_off;
    DBuf<double> val;               // leaves then internal nodes
    void release();
};

// Verlet cluster lists (north_star VerletClusterLists, vcl.cu): clusters of 8
// consecutive rows of their own CSF-1 grid, fp64 bounding boxes of the build
// positions, per-cluster lists of j-clusters whose boxes are within
// cutoff + skin, walked on the unwrapped positions like the Verlet lists.
struct Vcl {
    Grid grid;
    int ncl = 0, capc = 0;
    DBuf<double4> bb_lo, bb_hi;    // per cluster (w: 1 if it holds an owned row)
    DBuf<int> ccnt, clist;         // list length, clist[ci * capc + k]
    DBuf<double4> s4;              // unwrapped positions (build copy / refresh)
    DBuf<double> s3;               // x[ms], y[ms], z[ms]
    bool s3_valid = false;
    bool built = false;
    void release();
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sm_count = 148;
    // system (SimulationParams + per-type tables)
    bool have_system = false;
    double L[3] = {0, 0, 0};
    int periodic[3] = {0, 0, 0};
    double cutoff = 0, skin = 0;
    LJTab tab{};
    std::vector<double> mass;
    DBuf<double> d_mass;
    // bound particle arrays (owned by the caller)
    int64_t n = 0;
    int layout = AOS;
    double *pos = nullptr, *vel = nullptr, *force = nullptr, *old_force = nullptr;
    const int* tid = nullptr;
    // containers
    Grid grids[2];             // [0] CSF 1, [1] CSF 0.5
    Verlet vl;
    double prune_delta = -1.0;  // inner-list radius rc + delta (mdg_set_prune); < 0 default, 0 off
    // rows whose source index is >= n_force get no force work in the tiled
    // Verlet walk (the decomposition's ghost rows, mdg_set_force_rows)
    int64_t n_force = INT64_MAX;
    // the caller's loop iteration of the next drift (mdg_set_iteration): the
    // blow-up check records the earliest failing one (scal[8])
    long long iter_tag = 0;
    DBuf<int> order_tmp;        // mdg_owned_order scratch
    Vcl vcl;
    // temperature / thermostat / live statistics (stats.cu)
    PairwiseTree pw_particles, pw_bins;
    DBuf<int> ls_counts, ls_hist;
    DBuf<double> st_out;            // device results (temperature, stats[6])
    // device scalars: [0] eval count, [1] scan total scratch, [2] status flags
    // (bit 0 blow-up, bit 1 thermostat at T = 0)
    DBuf<unsigned long long> scal;
    unsigned long long* h_scal = nullptr;   // pinned mirror
    unsigned long long* d_h_scal = nullptr; // its device address (mapped): kernels write it, no copy engine
    // cached steady-state step graph (mdg_step_graph)
    uint64_t gen = 0;                       // bumped by every rebuild / rebind
    // mdg_rebuild_checked: the status word rides on the rebuild's first host
    // synchronisation; nonzero abandons the rebuild there
    bool flags_probe = false;
    unsigned flags_seen = 0;
    cudaStream_t graph_stream = nullptr;
    cudaEvent_t graph_in = nullptr, graph_out = nullptr;
    cudaGraphExec_t step_exec = nullptr;
    unsigned char step_key[96] = {0};       // what the cached graph was captured for
    // mdg_run's steady steps replayed from graphs: one per force / old_force
    // order (the loop swaps them every step), keyed by everything a captured
    // step bakes in; the kick_drift node's iteration tag is patched per replay
    uint64_t build_gen = 0;                 // bumped by rebuilds, set_system, new n / layout / types
    struct RunGraph {
        unsigned char key[192];
        cudaGraph_t graph_inst = nullptr;   // instantiated from: its root is the node handle to patch
        cudaGraph_t graph_cur = nullptr;    // the latest capture (cudaGraphExecUpdate'd in): its params
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t root = nullptr;     // the kick_drift node (of graph_inst)
        cudaKernelNodeParams kp{};          // of graph_cur's kick_drift node
        uint64_t used = 0;
        // mdg_profile inside the graph: the two event-record nodes around the
        // force kernels (of graph_inst), re-pointed at pool events per replay
        cudaGraphNode_t pnode[2] = {nullptr, nullptr};
        int nkern = 0;                      // kernel nodes (mdg_launch_count counts them per replay)
    } rg[2];
    // capture of a step graph in progress: prof_mark records into these
    // placeholder events as event-record nodes (cudaEventRecordExternal)
    bool capturing = false;
    int cap_marks = 0;
    cudaEvent_t cap_ev[2] = {nullptr, nullptr};
    uint64_t rg_clock = 0;
    DBuf<unsigned long long> scan_tmp;      // single-pass scans: [0] ticket, [1..] tile status words
    unsigned scan_epoch = 0;                // tags the status words of one scan call
    // optional CUDA-event bracketing of the force kernels (mdg_profile)
    bool prof = false;
    std::vector<cudaEvent_t> chunk_ev;   // mdg_host_step's per-chunk copy events
    cudaStream_t copy_stream = nullptr;  // mdg_host_run's H2D stream (overlaps the D2H)
    // mdg_timings: events around build (rebuild + refresh) and force (compute)
    bool timing = false, build_open = false, build_done = false, force_done = false;
    cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t h2d_done = nullptr;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    void prof_mark();
};

// ---- scans (warp-shuffle block scan, three phases) ----
void exclusive_scan_i32(Context& c, const int* in, int* out, int64_t n, unsigned long long* total,
                        unsigned long long* sumsq = nullptr);
void exclusive_scan_i32_to_i64(Context& c, const int* in, long long* out, int64_t n,
                               unsigned long long* total);

// ---- pipeline pieces ----
int grid_rebuild(Context& c, Grid& gr, const double* pos, int layout);
void grid_bind_scratch(Context& c, Grid& gr, int layout);
void grid_refresh(Context& c, Grid& gr, int layout);
void lc_compute(Context& c, Grid& gr, int traversal, int newton3, int layout);
int lc_pairs(Context& c, Grid& gr, long long cap, int2* dev_out, long long* count);
void lc_fold_forces(Context& c, Grid& gr, int layout, bool images_written);
int vl_rebuild(Context& c);
void vl_compute(Context& c, int layout);
int vl_export(Context& c, int64_t* entries, int64_t* noff, int32_t* nbr);
int vl_energy(Context& c, double* pe);
void vl_compute32(Context& c);
int vlt_build(Context& c);
int grid_owned_order(Context& c, Grid& gr, int* out);
// completes a deferred tile build (host check, retries, overflow tiles, pruning); -1 = error
int vlt_finish(Context& c);
// the next tiled walk re-prunes (an s3 write that bypassed the displacement bound)
void vl_prune_invalidate(Context& c);
int vcl_rebuild(Context& c);
void vcl_compute(Context& c, int newton3);
void vl_refresh_into(Context& c, Grid& gr, double4* s4, double* s3, bool& s3_valid);
int vl_build_rows(Context& c, const uint8_t* only);
int vl_ensure_rows(Context& c);
void halo_pack(Context& c, const int64_t* idx, int64_t nl, int64_t cnt, int axis, double sl, double sr,
               double* out);
void halo_unpack(Context& c, const double* in, int64_t count, int64_t row0);
struct Rows4 {
    double* p[4];
};
void permutation(Context& c, int op, int64_t n, const int64_t* a, const int64_t* b, int64_t* out);
void gather_rows(Context& c, const int64_t* order, int64_t n, int layout, Rows4 src, Rows4 dst,
                 const int* tsrc, int* tdst);
// cell lengths for the fp32-compute Verlet walk (cell-relative positions)
struct Cells32 {
    float cl[3];
    double cld[3];
};
void vlt_compute32(Context& c, const Cells32& cc);

// finish_kick arguments for kernels that fuse it into their epilogue
struct KickArgs {
    double* vel;
    const double* old_force;
    const double* mass;   // per type
    const int* tid;       // per particle, may be null
    double dt, gravity;
    int has_gravity;
};
bool vlt_compute(Context& c, const KickArgs* kick = nullptr);
float* vlt_prune_prepare(Context& c);
bool vlt_speculate(Context& c);
void vlt_big_rows(Context& c);
template <int PLAYOUT, int SLAYOUT>
void vl_refresh_launch(Context& c, int* zero_me, unsigned long long* zero_cnt = nullptr);
template <int PLAYOUT>
void vl_force_rows_launch(Context& c, const uint8_t* only);
void integ_drift_wrap(Context& c, double dt);
void integ_finish_kick(Context& c, double dt, int has_gravity, double gravity);
void integ_kick_drift(Context& c, double dt, int has_gravity, double gravity, bool copy);
size_t integ_box_size();
size_t integ_box_tag_offset();
int integ_kick_drift_nparams();
void integ_sd_step(Context& c, double gamma, double max_disp);
int stats_temperature(Context& c, double* t);
int stats_thermostat(Context& c, double target, double max_delta_t);
int stats_live(Context& c, double out[6]);
void stats_release(Context& c);
void set_error(const std::string& msg);
// host-side count of kernel launches issued by the library (bench evidence)
void note_launch();
void note_launches(int k);
// scalars to a mapped pinned mirror by a one-thread kernel: a D2H copy in the
// stream costs a ~17 us bubble between the copy and compute engines
void scal_to_host(Context& c, const unsigned long long* src, int count, unsigned long long* dst_mapped);
unsigned long long launch_count();

#define MDG_CUDA(x)                                                             \
    do {                                                                        \
        cudaError_t _e = (x);                                                   \
        if (_e != cudaSuccess) {                                                \
            ::mdg::set_error(std::string(#x) + ": " + cudaGetErrorString(_e));  \
            return -1;                                                          \
        }                                                                       \
    } while (0)

// component stride of the unwrapped SoA copy (Verlet::s3): a multiple of 4
// rows, so every component array is 32-byte aligned (1-D bulk copies)
inline int s3_stride(int m) { return (m + 3) & ~3; }

inline int blocks_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace mdg
