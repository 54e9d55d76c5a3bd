// The C ABI (include/mdg.h) over the device pipeline.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>

#include <vector>
#include <nvtx3/nvToolsExt.h>
#include "../../include/mdg.h"
#include "device.cuh"

struct mdg_ctx {
    mdg::Context c;
};

namespace mdg {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

void Context::prof_mark() {
    if (!prof) return;
    if (capturing) {   // a step graph: an event-record node, re-pointed per replay
        if (cap_marks < 2) cudaEventRecordWithFlags(cap_ev[cap_marks], stream, cudaEventRecordExternal);
        ++cap_marks;
        return;
    }
    if (ev_used == ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ev_pool.push_back(e);
    }
    cudaEventRecord(ev_pool[ev_used++], stream);
}

static unsigned long long g_launches = 0;
void note_launch() { ++g_launches; }
void note_launches(int k) { g_launches += (unsigned long long)k; }
unsigned long long launch_count() { return g_launches; }

}  // namespace mdg

using namespace mdg;

#define CHECK_CTX(ctx)                                   \
    do {                                                 \
        if (!(ctx)) {                                    \
            set_error("null context");                   \
            return MDG_EINVAL;                           \
        }                                                \
        cudaSetDevice((ctx)->c.device);                  \
    } while (0)

static int cuda_status(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": " + cudaGetErrorString(e));
        return MDG_ECUDA;
    }
    return MDG_OK;
}

// Configuration.__post_init__ (configuration.py:30-50)
static int validate(const mdg_config* cfg) {
    if (!cfg) {
        set_error("null configuration");
        return MDG_EINVAL;
    }
    if (cfg->layout != MDG_AOS && cfg->layout != MDG_SOA) {
        set_error("unknown layout");
        return MDG_EINVAL;
    }
    if (cfg->container == MDG_VL) {
        if (cfg->traversal != MDG_LIST_ITER) {
            set_error("Verlet lists only support List_Iter");
            return MDG_EINVAL;
        }
        if (cfg->csf != 1.0) {
            set_error("Verlet lists fix the cell size factor at 1");
            return MDG_EINVAL;
        }
    } else if (cfg->container == MDG_VCL) {
        if (cfg->traversal != MDG_CLUSTER_ITER) {
            set_error("Verlet cluster lists only support ClusterIter");
            return MDG_EINVAL;
        }
        if (cfg->csf != 1.0) {
            set_error("Verlet cluster lists fix the cell size factor at 1");
            return MDG_EINVAL;
        }
    } else if (cfg->container == MDG_LC) {
        if (cfg->traversal < MDG_C01 || cfg->traversal > MDG_SLI) {
            set_error("linked cells do not support this traversal");
            return MDG_EINVAL;
        }
    } else {
        set_error("unknown container");
        return MDG_EINVAL;
    }
    if ((cfg->traversal == MDG_LIST_ITER || cfg->traversal == MDG_C01) && cfg->newton3) {
        set_error("C01 / List_Iter cannot use Newton-3 writes");
        return MDG_EINVAL;
    }
    if (cfg->csf != 1.0 && cfg->csf != 0.5) {
        set_error("cell size factor must be one of (1.0, 0.5)");
        return MDG_EINVAL;
    }
    if (cfg->precision != MDG_FP64 && cfg->precision != MDG_FP32) {
        set_error("unknown precision");
        return MDG_EINVAL;
    }
    if (cfg->precision == MDG_FP32 && cfg->container != MDG_VL) {
        set_error("the fp32-compute variant exists for Verlet lists only");
        return MDG_EINVAL;
    }
    return MDG_OK;
}

static Grid* grid_for(Context& c, double csf) { return csf == 1.0 ? &c.grids[0] : &c.grids[1]; }

static int need_system(mdg_ctx* ctx) {
    if (!ctx->c.have_system) {
        set_error("mdg_set_system has not been called");
        return MDG_ESTATE;
    }
    return MDG_OK;
}

// NVTX ranges around the ABI's phases (SURVEY §5 tracing): visible to Nsight
// tools in the "mdg" domain; without a tool attached a range is one pointer test.
namespace {
nvtxDomainHandle_t nvtx_domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("mdg");
    return d;
}
struct NvtxRange {
    explicit NvtxRange(const char* name) {
        nvtxEventAttributes_t a = {};
        a.version = NVTX_VERSION;
        a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        a.messageType = NVTX_MESSAGE_TYPE_ASCII;
        a.message.ascii = name;
        nvtxDomainRangePushEx(nvtx_domain(), &a);
    }
    ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace
#ifdef MDG_NO_NVTX
#define MDG_RANGE(name) ((void)0)
#else
#define MDG_RANGE(name) NvtxRange nvtx_range_(name)
#endif

extern "C" {

const char* mdg_version(void) { return "mdg 0.1 (sm_100a)"; }

uint64_t mdg_launch_count(void) { return (uint64_t)launch_count(); }

const char* mdg_last_error(void) { return g_err.c_str(); }

int mdg_create(int device, void* stream, mdg_ctx** out) {
    if (!out) {
        set_error("null output");
        return MDG_EINVAL;
    }
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return cuda_status("cudaSetDevice");
    mdg_ctx* ctx = new mdg_ctx();
    ctx->c.device = device;
    ctx->c.stream = (cudaStream_t)stream;
    cudaDeviceGetAttribute(&ctx->c.sm_count, cudaDevAttrMultiProcessorCount, device);
    ctx->c.scal.ensure(16);
    if (!ctx->c.scal.p || cudaHostAlloc((void**)&ctx->c.h_scal, 16 * sizeof(unsigned long long),
                                        cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&ctx->c.d_h_scal, ctx->c.h_scal, 0) != cudaSuccess) {
        delete ctx;
        return cuda_status("allocating context scalars");
    }
    cudaMemsetAsync(ctx->c.scal.p, 0, 8 * sizeof(unsigned long long), ctx->c.stream);
    cudaMemsetAsync(ctx->c.scal.p + 8, 0xff, 8 * sizeof(unsigned long long), ctx->c.stream);
    *out = ctx;
    return cuda_status("mdg_create");
}

int mdg_destroy(mdg_ctx* ctx) {
    if (!ctx) return MDG_OK;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    ctx->c.grids[0].release();
    ctx->c.grids[1].release();
    ctx->c.vl.release();
    ctx->c.vcl.release();
    stats_release(ctx->c);
    ctx->c.scal.release();
    ctx->c.scan_tmp.release();
    ctx->c.d_mass.release();
    if (ctx->c.h_scal) cudaFreeHost(ctx->c.h_scal);
    for (cudaEvent_t e : ctx->c.ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->c.chunk_ev) cudaEventDestroy(e);
    if (ctx->c.step_exec) cudaGraphExecDestroy(ctx->c.step_exec);
    for (cudaEvent_t e : ctx->c.cap_ev)
        if (e) cudaEventDestroy(e);
    for (auto& g : ctx->c.rg) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph_cur && g.graph_cur != g.graph_inst) cudaGraphDestroy(g.graph_cur);
        if (g.graph_inst) cudaGraphDestroy(g.graph_inst);
    }
    if (ctx->c.graph_in) cudaEventDestroy(ctx->c.graph_in);
    if (ctx->c.graph_out) cudaEventDestroy(ctx->c.graph_out);
    if (ctx->c.graph_stream) cudaStreamDestroy(ctx->c.graph_stream);
    if (ctx->c.h2d_done) cudaEventDestroy(ctx->c.h2d_done);
    for (cudaEvent_t e : ctx->c.tev)
        if (e) cudaEventDestroy(e);
    if (ctx->c.copy_stream) cudaStreamDestroy(ctx->c.copy_stream);
    delete ctx;
    return MDG_OK;
}

int mdg_set_stream(mdg_ctx* ctx, void* stream) {
    CHECK_CTX(ctx);
    ctx->c.stream = (cudaStream_t)stream;
    return MDG_OK;
}

int mdg_set_system(mdg_ctx* ctx, const double domain[3], const int periodic[3], double cutoff,
                   double skin, int ntypes, const double* sigma, const double* epsilon,
                   const double* mass) {
    CHECK_CTX(ctx);
    Context& c = ctx->c;
    ++c.build_gen;
    if (!(cutoff > 0)) { set_error("cutoff must be > 0"); return MDG_EINVAL; }
    if (!(skin >= 0)) { set_error("skin must be >= 0"); return MDG_EINVAL; }
    if (ntypes < 1 || ntypes > kMaxTypes) {
        set_error("ntypes must be in [1, " + std::to_string(kMaxTypes) + "]");
        return MDG_EINVAL;
    }
    double ell = cutoff + skin;
    for (int k = 0; k < 3; ++k) {
        if (!(domain[k] >= ell)) {
            set_error("domain size must be at least cutoff + skin in every dimension");
            return MDG_EINVAL;
        }
        if (periodic[k] && domain[k] < 2.0 * ell) {
            set_error("periodic axes require domain >= 2*(cutoff + skin)");
            return MDG_EINVAL;
        }
    }
    for (int k = 0; k < 3; ++k) {
        c.L[k] = domain[k];
        c.periodic[k] = periodic[k] ? 1 : 0;
    }
    c.cutoff = cutoff;
    c.skin = skin;
    // forces.py:12-22
    c.tab.T = ntypes;
    c.tab.rc2 = cutoff * cutoff;
    for (int a = 0; a < ntypes; ++a)
        for (int b = 0; b < ntypes; ++b) {
            double sm = 0.5 * (sigma[a] + sigma[b]);
            double em = sqrt(epsilon[a] * epsilon[b]);
            c.tab.sig2[a * ntypes + b] = sm * sm;
            c.tab.eps24[a * ntypes + b] = 24.0 * em;
        }
    c.mass.assign(mass, mass + ntypes);
    c.d_mass.ensure(ntypes);
    if (cudaMemcpy(c.d_mass.p, mass, ntypes * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
        return cuda_status("mass upload");
    const double csfs[2] = {1.0, 0.5};
    for (int g = 0; g < 2; ++g) {
        Grid& gr = c.grids[g];
        gr.g = make_geometry(c.L, c.periodic, ell, csfs[g]);
        gr.pruned = pruned_stencil(gr.g);
        gr.fwd = forward_stencil(gr.g, 0);
        int major = 0;  // SLI sweeps along argmax(dims_owned) (containers.py:225-227)
        for (int k = 1; k < 3; ++k)
            if (gr.g.S[k] > gr.g.S[major]) major = k;
        gr.sli_major = major;
        gr.fwd_sli = forward_stencil(gr.g, major);
        gr.built = false;
    }
    c.vl.grid.g = c.grids[0].g;
    c.vl.grid.pruned = c.grids[0].pruned;
    c.vl.grid.sort_by_z = 1;   // z-ordered cells: the tiled build scans a z-window (vltile.cu)
    c.vl.built = false;
    c.vcl.grid.g = c.grids[0].g;
    c.vcl.grid.pruned = c.grids[0].pruned;
    c.vcl.grid.sort_by_z = 1;
    c.vcl.built = false;
    c.have_system = true;
    return MDG_OK;
}

int mdg_bind(mdg_ctx* ctx, int64_t n, int layout, double* pos, double* vel, double* force,
             double* old_force, const int32_t* type_id) {
    CHECK_CTX(ctx);
    if (n < 0 || n > 0x7fffffffLL / 2) { set_error("particle count out of range"); return MDG_EINVAL; }
    if (layout != MDG_AOS && layout != MDG_SOA) { set_error("unknown layout"); return MDG_EINVAL; }
    Context& c = ctx->c;
    if (n != c.n) {
        c.grids[0].built = c.grids[1].built = false;
        c.vl.built = false;
        c.vcl.built = false;
    }
    if (n != c.n || layout != c.layout || pos != c.pos || vel != c.vel || force != c.force ||
        old_force != c.old_force || type_id != c.tid)
        ++c.gen;
    if (n != c.n || layout != c.layout || type_id != c.tid) ++c.build_gen;
    c.n = n;
    c.layout = layout;
    c.pos = pos;
    c.vel = vel;
    c.force = force;
    c.old_force = old_force;
    c.tid = type_id;
    return MDG_OK;
}

// mdg_timings' events (skipped while a stream is being captured into a graph)
static void tmark(Context& c, int k) {
    if (!c.timing) return;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(c.stream, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone) return;
    if (!c.tev[k] && cudaEventCreate(&c.tev[k]) != cudaSuccess) return;
    cudaEventRecord(c.tev[k], c.stream);
    if (k == 0) c.build_open = true;
    if (k == 1) { c.build_open = false; c.build_done = true; }
    if (k == 3) c.force_done = true;
}

int mdg_timings(mdg_ctx* ctx, int enable, int64_t* build_ns, int64_t* force_ns) {
    CHECK_CTX(ctx);
    Context& c = ctx->c;
    if (build_ns) *build_ns = -1;
    if (force_ns) *force_ns = -1;
    if (enable >= 0) {
        c.timing = enable != 0;
        c.build_open = c.build_done = c.force_done = false;
        return MDG_OK;
    }
    float ms = 0.f;
    if (c.build_done && build_ns && cudaEventSynchronize(c.tev[1]) == cudaSuccess &&
        cudaEventElapsedTime(&ms, c.tev[0], c.tev[1]) == cudaSuccess)
        *build_ns = (int64_t)((double)ms * 1e6);
    if (c.force_done && force_ns && cudaEventSynchronize(c.tev[3]) == cudaSuccess &&
        cudaEventElapsedTime(&ms, c.tev[2], c.tev[3]) == cudaSuccess)
        *force_ns = (int64_t)((double)ms * 1e6);
    return cuda_status("mdg_timings");
}

int mdg_set_prune(mdg_ctx* ctx, double delta) {
    CHECK_CTX(ctx);
    if (!(delta == delta)) {
        set_error("prune delta is NaN");
        return MDG_EINVAL;
    }
    ctx->c.prune_delta = delta < 0.0 ? -1.0 : delta;
    return MDG_OK;
}

int mdg_prune_count(mdg_ctx* ctx, int64_t* prunes) {
    CHECK_CTX(ctx);
    if (!prunes) {
        set_error("null output");
        return MDG_EINVAL;
    }
    Context& c = ctx->c;
    *prunes = -1;
    if (vlt_finish(c)) return MDG_ECUDA;
    if (!c.vl.prune || !c.vl.pst.p) return MDG_OK;
    int h = 0;
    if (cudaMemcpyAsync(&h, c.vl.pst.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c.stream) != cudaSuccess ||
        cudaStreamSynchronize(c.stream) != cudaSuccess)
        return cuda_status("mdg_prune_count");
    *prunes = h;
    return MDG_OK;
}

int mdg_rebuild(mdg_ctx* ctx, const mdg_config* cfg) {
    MDG_RANGE("mdg_rebuild");
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    if (int e = need_system(ctx)) return e;
    Context& c = ctx->c;
    tmark(c, 0);
    ++c.gen;
    ++c.build_gen;
    if (cfg->container == MDG_VL) {
        if (vl_rebuild(c)) return MDG_ECUDA;
    } else if (cfg->container == MDG_VCL) {
        if (vcl_rebuild(c)) return MDG_ECUDA;
    } else {
        Grid& gr = *grid_for(c, cfg->csf);
        if (grid_rebuild(c, gr, c.pos, c.layout)) return MDG_ECUDA;
        grid_bind_scratch(c, gr, cfg->layout);
    }
    return cuda_status("mdg_rebuild");
}

int mdg_rebuild_checked(mdg_ctx* ctx, const mdg_config* cfg, int* flags) {
    MDG_RANGE("mdg_rebuild_checked");
    CHECK_CTX(ctx);
    if (!flags) { set_error("null output"); return MDG_EINVAL; }
    *flags = 0;
    if (int e = validate(cfg)) return e;
    if (int e = need_system(ctx)) return e;
    Context& c = ctx->c;
    // the status word rides on grid_rebuild's copy of the scalars before its
    // host synchronisation (flags_probe)
    c.flags_probe = true;
    c.flags_seen = 0;
    int e = mdg_rebuild(ctx, cfg);
    if (c.flags_probe) {   // the rebuild stopped before that synchronisation: read it now
        c.flags_probe = false;
        if (cudaMemcpyAsync(c.h_scal + 2, c.scal.p + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            c.stream) != cudaSuccess ||
            cudaStreamSynchronize(c.stream) != cudaSuccess)
            return cuda_status("mdg_rebuild_checked");
        c.flags_seen = (unsigned)(c.h_scal[2] & 3ull);
    }
    if (c.flags_seen) {
        *flags = (int)c.flags_seen;
        c.vl.built = false;
        c.vcl.built = false;
        cudaMemsetAsync(c.scal.p + 2, 0, sizeof(unsigned long long), c.stream);
        set_error("");
        return cuda_status("mdg_rebuild_checked");
    }
    return e;
}

int mdg_refresh(mdg_ctx* ctx, const mdg_config* cfg) {
    MDG_RANGE("mdg_refresh");
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    Context& c = ctx->c;
    if (!c.build_open) tmark(c, 0);
    if (cfg->container == MDG_VL || cfg->container == MDG_VCL) {
        tmark(c, 1);
        return MDG_OK;
    }
    Grid& gr = *grid_for(c, cfg->csf);
    if (!gr.built) { set_error("refresh before rebuild"); return MDG_ESTATE; }
    if (gr.scratch_layout != cfg->layout) grid_bind_scratch(c, gr, cfg->layout);
    grid_refresh(c, gr, cfg->layout);
    tmark(c, 1);
    return cuda_status("mdg_refresh");
}

int mdg_compute(mdg_ctx* ctx, const mdg_config* cfg) {
    MDG_RANGE("mdg_compute");
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    Context& c = ctx->c;
    if (c.layout != cfg->layout) {
        set_error(std::string("particle layout ") + (c.layout == MDG_AOS ? "AoS" : "SoA") +
                  " does not match the configuration");
        return MDG_EINVAL;
    }
    tmark(c, 2);
    // the fp64 Verlet-list compute zeroes the eval count itself (in its
    // refresh kernel, or before its row-space walk): one launch less per step
    const bool vl64 = cfg->container == MDG_VL && cfg->precision != MDG_FP32 && c.n > 0 && c.vl.built;
    if (!vl64 && cudaMemsetAsync(c.scal.p, 0, sizeof(unsigned long long), c.stream) != cudaSuccess)
        return cuda_status("counter reset");
    if (c.n == 0) {
        tmark(c, 3);
        return MDG_OK;
    }
    if (cfg->container == MDG_VCL) {
        if (!c.vcl.built) { set_error("compute before rebuild"); return MDG_ESTATE; }
        vcl_compute(c, cfg->newton3);
    } else if (cfg->container == MDG_VL) {
        if (!c.vl.built) { set_error("compute before rebuild"); return MDG_ESTATE; }
        if (cfg->precision == MDG_FP32) vl_compute32(c);
        else vl_compute(c, cfg->layout);
    } else {
        Grid& gr = *grid_for(c, cfg->csf);
        if (!gr.built || gr.scratch_layout != cfg->layout) {
            set_error("compute before rebuild/refresh");
            return MDG_ESTATE;
        }
        lc_compute(c, gr, cfg->traversal, cfg->newton3, cfg->layout);
        lc_fold_forces(c, gr, cfg->layout, cfg->traversal != MDG_C01);
    }
    tmark(c, 3);
    return cuda_status("mdg_compute");
}

int mdg_lc_pairs(mdg_ctx* ctx, double csf, int64_t cap, int32_t* pairs, int64_t* count) {
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    if (csf != 1.0 && csf != 0.5) { set_error("csf must be 1 or 0.5"); return MDG_EINVAL; }
    if (!count) { set_error("null count"); return MDG_EINVAL; }
    Context& c = ctx->c;
    Grid& gr = *grid_for(c, csf);
    if (!gr.built) { set_error("LC grid not built (mdg_rebuild with an LC configuration first)"); return MDG_ESTATE; }
    DBuf<int2> buf;
    if (pairs && cap > 0) {
        buf.ensure((size_t)cap);
        if (!buf.p) { set_error("out of device memory (pair export)"); return MDG_ECUDA; }
    }
    long long n = 0;
    if (lc_pairs(c, gr, pairs ? cap : 0, buf.p, &n)) return cuda_status("mdg_lc_pairs");
    *count = n;
    if (pairs && cap > 0 && n > 0)
        cudaMemcpy(pairs, buf.p, (size_t)std::min<long long>(n, cap) * sizeof(int2), cudaMemcpyDeviceToHost);
    buf.release();
    return cuda_status("mdg_lc_pairs");
}

int mdg_compute_kick(mdg_ctx* ctx, const mdg_config* cfg, double dt, int has_gravity,
                     double gravity) {
    MDG_RANGE("mdg_compute_kick");
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    if (int e = need_system(ctx)) return e;
    Context& c = ctx->c;
    Verlet& v = c.vl;
    // Measured on B200, config 2: the fused epilogue's scattered
    // per-particle vel / old_force accesses cost more (walk 0.186 -> 0.228 ms)
    // than the coalesced kick pass they replace, so fusion is opt-in
    // (MDG_FUSE_KICK=1).
    static int fuse_env = -1;
    if (fuse_env < 0) {
        const char* e = getenv("MDG_FUSE_KICK");
        fuse_env = e ? atoi(e) : 0;
    }
    if (fuse_env && cfg->container == MDG_VL && v.build_pending && vlt_finish(c)) {
        // the tiled build failed: the row-space lists take over (as in vl_compute)
        v.tiled = false;
        v.prune = false;
        if (vl_ensure_rows(c)) return cuda_status("mdg_compute_kick: row-space lists");
    }
    bool fuse = fuse_env && cfg->container == MDG_VL && cfg->precision == MDG_FP64 &&
                c.layout == cfg->layout && v.built && v.tiled && v.nbig == 0 && c.n > 0;
    if (fuse) {
        if (cudaMemsetAsync(c.scal.p, 0, sizeof(unsigned long long), c.stream) != cudaSuccess)
            return cuda_status("counter reset");
        v.s3.ensure(3 * (size_t)s3_stride((int)v.grid.m) + 8);
        KickArgs k{c.vel, c.old_force, c.d_mass.p, c.tid, dt, gravity, has_gravity};
        vlt_compute(c, &k);
        return cuda_status("mdg_compute_kick");
    }
    if (int e = mdg_compute(ctx, cfg)) return e;
    integ_finish_kick(c, dt, has_gravity, gravity);
    return cuda_status("mdg_compute_kick");
}

int mdg_step_graph(mdg_ctx* ctx, const mdg_config* cfg, double dt, int has_gravity, double gravity) {
    MDG_RANGE("mdg_step_graph");
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    if (int e = need_system(ctx)) return e;
    Context& c = ctx->c;
    if (c.layout != cfg->layout) {
        set_error("particle layout does not match the configuration");
        return MDG_EINVAL;
    }
    bool built = cfg->container == MDG_VL ? c.vl.built
               : cfg->container == MDG_VCL ? c.vcl.built
               : grid_for(c, cfg->csf)->built;
    if (!built) { set_error("mdg_step_graph before rebuild"); return MDG_ESTATE; }
    if (cfg->container == MDG_VL && vlt_finish(c)) {   // no host wait inside a capture
        // the tiled build failed: build the row-space lists now, outside the capture
        c.vl.tiled = false;
        c.vl.prune = false;
        if (vl_ensure_rows(c)) return cuda_status("mdg_step_graph: row-space lists");
    }
    if (!c.graph_stream) {
        if (cudaStreamCreateWithFlags(&c.graph_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c.graph_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c.graph_out, cudaEventDisableTiming) != cudaSuccess)
            return cuda_status("graph stream");
    }
    struct Key {
        mdg_config cfg;
        double dt, gravity;
        int has_gravity;
        uint64_t gen;
        const void* stream;
    } key;
    memset(&key, 0, sizeof key);
    key.cfg = *cfg;
    key.dt = dt;
    key.gravity = gravity;
    key.has_gravity = has_gravity;
    key.gen = c.gen;
    key.stream = c.stream;
    static_assert(sizeof(Key) <= sizeof(c.step_key), "graph key");
    if (!c.step_exec || memcmp(&key, c.step_key, sizeof key) != 0) {
        if (c.step_exec) {
            cudaGraphExecDestroy(c.step_exec);
            c.step_exec = nullptr;
        }
        // capture drift + refresh + compute + kick on the private stream
        cudaStream_t home = c.stream;
        bool prof = c.prof;
        c.stream = c.graph_stream;
        c.prof = false;
        cudaGraph_t graph = nullptr;
        int err = MDG_OK;
        if (cudaStreamBeginCapture(c.graph_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            err = MDG_ECUDA;
        } else {
            integ_drift_wrap(c, dt);
            if (cfg->container == MDG_LC) {
                Grid& gr = *grid_for(c, cfg->csf);
                grid_refresh(c, gr, cfg->layout);
            }
            cudaMemsetAsync(c.scal.p, 0, sizeof(unsigned long long), c.stream);
            if (cfg->container == MDG_VCL) {
                vcl_compute(c, cfg->newton3);
            } else if (cfg->container == MDG_VL) {
                if (cfg->precision == MDG_FP32) vl_compute32(c);
                else vl_compute(c, cfg->layout);
            } else {
                Grid& gr = *grid_for(c, cfg->csf);
                lc_compute(c, gr, cfg->traversal, cfg->newton3, cfg->layout);
                lc_fold_forces(c, gr, cfg->layout, cfg->traversal != MDG_C01);
            }
            integ_finish_kick(c, dt, has_gravity, gravity);
            if (cudaStreamEndCapture(c.graph_stream, &graph) != cudaSuccess || !graph) err = MDG_ECUDA;
        }
        c.stream = home;
        c.prof = prof;
        if (err == MDG_OK && cudaGraphInstantiate(&c.step_exec, graph, 0) != cudaSuccess) err = MDG_ECUDA;
        if (graph) cudaGraphDestroy(graph);
        if (err != MDG_OK) {
            c.step_exec = nullptr;
            return cuda_status("step graph capture");
        }
        memcpy(c.step_key, &key, sizeof key);
    }
    // order against the context stream on both sides
    if (cudaEventRecord(c.graph_in, c.stream) != cudaSuccess ||
        cudaStreamWaitEvent(c.graph_stream, c.graph_in, 0) != cudaSuccess ||
        cudaGraphLaunch(c.step_exec, c.graph_stream) != cudaSuccess ||
        cudaEventRecord(c.graph_out, c.graph_stream) != cudaSuccess ||
        cudaStreamWaitEvent(c.stream, c.graph_out, 0) != cudaSuccess)
        return cuda_status("step graph launch");
    note_launch();
    return MDG_OK;
}

int mdg_eval_count(mdg_ctx* ctx, int64_t* count) {
    CHECK_CTX(ctx);
    Context& c = ctx->c;
    if (cudaMemcpyAsync(c.h_scal, c.scal.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        c.stream) != cudaSuccess ||
        cudaStreamSynchronize(c.stream) != cudaSuccess)
        return cuda_status("mdg_eval_count");
    *count = (int64_t)c.h_scal[0];
    return MDG_OK;
}

int mdg_drift_wrap(mdg_ctx* ctx, double dt) {
    MDG_RANGE("mdg_drift_wrap");
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    integ_drift_wrap(ctx->c, dt);
    return cuda_status("mdg_drift_wrap");
}

int mdg_finish_kick(mdg_ctx* ctx, double dt, int has_gravity, double gravity) {
    MDG_RANGE("mdg_finish_kick");
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    integ_finish_kick(ctx->c, dt, has_gravity, gravity);
    return cuda_status("mdg_finish_kick");
}

int mdg_kick_drift(mdg_ctx* ctx, double dt, int has_gravity, double gravity, int copy_old_force) {
    MDG_RANGE("mdg_kick_drift");
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    integ_kick_drift(ctx->c, dt, has_gravity, gravity, copy_old_force != 0);
    return cuda_status("mdg_kick_drift");
}

// One steady step's device work after the drift (refresh + compute, as
// mdg_refresh / mdg_compute do it for a built container), for capture.
static void steady_step_kernels(Context& c, const mdg_config* cfg) {
    if (cfg->container == MDG_LC) grid_refresh(c, *grid_for(c, cfg->csf), cfg->layout);
    if (!(cfg->container == MDG_VL && cfg->precision != MDG_FP32))   // vl_compute zeroes it
        cudaMemsetAsync(c.scal.p, 0, sizeof(unsigned long long), c.stream);
    if (cfg->container == MDG_VCL) {
        vcl_compute(c, cfg->newton3);
    } else if (cfg->container == MDG_VL) {
        if (cfg->precision == MDG_FP32) vl_compute32(c);
        else vl_compute(c, cfg->layout);
    } else {
        Grid& gr = *grid_for(c, cfg->csf);
        lc_compute(c, gr, cfg->traversal, cfg->newton3, cfg->layout);
        lc_fold_forces(c, gr, cfg->layout, cfg->traversal != MDG_C01);
    }
}

// MDG_RUN_GRAPH: 1 (default) mdg_run replays steady steps from graphs, 0 eager
static int run_graph_env() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_RUN_GRAPH");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// A steady step (kick + drift, refresh, compute) from a cached graph: 0 done,
// 1 not possible here (the caller runs it eagerly), < 0 error.
static int run_graph_step(Context& c, const mdg_config* cfg, double dt, int has_gravity, double gravity) {
    if (c.n == 0) return 1;
    bool built = cfg->container == MDG_VL ? c.vl.built
               : cfg->container == MDG_VCL ? c.vcl.built
               : grid_for(c, cfg->csf)->built && grid_for(c, cfg->csf)->scratch_layout == cfg->layout;
    // mdg_timings brackets kernels with events per call: eager (mdg_profile's
    // marks become event-record nodes of the graph)
    if (!built || c.layout != cfg->layout || c.timing) return 1;
    // first uses after a rebuild (host checks, lazy allocations and list
    // builds) run eagerly: a capture must only record steady-state work
    if (cfg->container == MDG_VL && (c.vl.build_pending || (!c.vl.tiled && !c.vl.rows_valid))) return 1;
    if (!c.graph_stream) {
        if (cudaStreamCreateWithFlags(&c.graph_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c.graph_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c.graph_out, cudaEventDisableTiming) != cudaSuccess)
            return -1;
    }
    struct Key {
        mdg_config cfg;
        double dt, gravity, prune_delta;
        int has_gravity, layout;
        uint64_t build_gen;
        int64_t n, n_force;
        const void *pos, *vel, *force, *old_force, *tid, *stream;
        int prof;
    } key;
    static_assert(sizeof(Key) <= sizeof(c.rg[0].key), "run graph key");
    memset(&key, 0, sizeof key);
    key.cfg = *cfg;
    key.dt = dt;
    key.gravity = gravity;
    key.prune_delta = c.prune_delta;
    key.has_gravity = has_gravity;
    key.layout = c.layout;
    key.build_gen = c.build_gen;
    key.n = c.n;
    key.n_force = c.n_force;
    key.pos = c.pos; key.vel = c.vel; key.force = c.force; key.old_force = c.old_force;
    key.tid = c.tid; key.stream = c.stream;
    key.prof = c.prof ? 1 : 0;
    if (c.prof && !c.cap_ev[0]) {
        if (cudaEventCreate(&c.cap_ev[0]) != cudaSuccess || cudaEventCreate(&c.cap_ev[1]) != cudaSuccess) return 1;
    }
    Context::RunGraph* g = nullptr;
    for (auto& s : c.rg)
        if (s.exec && memcmp(s.key, &key, sizeof key) == 0) g = &s;
    if (!g) {
        // capture this step; update the least recently used slot's executable
        // graph with it (same topology after a rebuild: no re-instantiation),
        // else instantiate anew
        g = c.rg[0].used <= c.rg[1].used ? &c.rg[0] : &c.rg[1];
        cudaStream_t home = c.stream;
        c.stream = c.graph_stream;
        c.capturing = true;
        c.cap_marks = 0;
        cudaGraph_t graph = nullptr;
        bool ok = cudaStreamBeginCapture(c.graph_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            // as the eager step: kick + drift, then the force into the other buffer
            integ_kick_drift(c, dt, has_gravity, gravity, false);
            std::swap(c.force, c.old_force);
            steady_step_kernels(c, cfg);
            std::swap(c.force, c.old_force);   // the caller swaps after the replay
            ok = cudaStreamEndCapture(c.graph_stream, &graph) == cudaSuccess && graph;
        }
        c.stream = home;
        c.capturing = false;
        ok = ok && (!c.prof || c.cap_marks == 2);   // the force path marks exactly twice
        cudaGraphNode_t root = nullptr;
        cudaKernelNodeParams kp{};
        size_t nroot = 1;
        ok = ok && cudaGraphGetRootNodes(graph, &root, &nroot) == cudaSuccess && nroot == 1 &&
             cudaGraphKernelNodeGetParams(root, &kp) == cudaSuccess;
        // the graph's kernel nodes (launch accounting) and its two event-record
        // nodes (profiling), found by their placeholder events
        cudaGraphNode_t pn[2] = {nullptr, nullptr};
        int nkern = 0;
        if (ok) {
            size_t nn = 0;
            cudaGraphGetNodes(graph, nullptr, &nn);
            std::vector<cudaGraphNode_t> nodes(nn);
            if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType ty;
                if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess) continue;
                if (ty == cudaGraphNodeTypeKernel) ++nkern;
                cudaEvent_t ev = nullptr;
                if (c.prof && ty == cudaGraphNodeTypeEventRecord &&
                    cudaGraphEventRecordNodeGetEvent(nd, &ev) == cudaSuccess)
                    for (int k = 0; k < 2; ++k)
                        if (ev == c.cap_ev[k]) pn[k] = nd;
            }
            if (c.prof) ok = pn[0] && pn[1];
        }
        bool updated = false;
        if (ok && g->exec) {
            cudaGraphExecUpdateResultInfo info;
            updated = cudaGraphExecUpdate(g->exec, graph, &info) == cudaSuccess;
            if (!updated) cudaGetLastError();
        }
        if (ok && !updated) {
            if (g->exec) cudaGraphExecDestroy(g->exec);
            if (g->graph_cur && g->graph_cur != g->graph_inst) cudaGraphDestroy(g->graph_cur);
            if (g->graph_inst) cudaGraphDestroy(g->graph_inst);
            g->exec = nullptr;
            g->graph_inst = g->graph_cur = nullptr;
            ok = cudaGraphInstantiate(&g->exec, graph, 0) == cudaSuccess;
            if (ok) {
                g->graph_inst = g->graph_cur = graph;
                g->root = root;
                g->pnode[0] = pn[0];
                g->pnode[1] = pn[1];
            }
        } else if (ok) {
            if (g->graph_cur && g->graph_cur != g->graph_inst) cudaGraphDestroy(g->graph_cur);
            g->graph_cur = graph;
        }
        if (!ok) {
            if (graph && graph != g->graph_inst) cudaGraphDestroy(graph);
            if (g->exec && !g->graph_inst) {
                cudaGraphExecDestroy(g->exec);
                g->exec = nullptr;
            }
            memset(g->key, 0, sizeof g->key);
            cudaGetLastError();
            return 1;   // not capturable here: eager
        }
        g->kp = kp;
        g->nkern = nkern;
        memcpy(g->key, &key, sizeof key);
    }
    g->used = ++c.rg_clock;
    // this step's iteration tag into the captured kick_drift launch
    alignas(16) unsigned char box[256];
    const size_t bs = integ_box_size();
    if (bs > sizeof box) return -1;
    memcpy(box, g->kp.kernelParams[0], bs);
    const unsigned long long tag = (unsigned long long)c.iter_tag;
    memcpy(box + integ_box_tag_offset(), &tag, sizeof tag);
    void* args[16];
    const int na = integ_kick_drift_nparams();
    for (int k = 0; k < na; ++k) args[k] = g->kp.kernelParams[k];
    args[0] = box;
    cudaKernelNodeParams kp = g->kp;
    kp.kernelParams = args;
    kp.extra = nullptr;
    // (captured on the private stream; launched straight into the context
    // stream, legacy default stream included)
    if (cudaGraphExecKernelNodeSetParams(g->exec, g->root, &kp) != cudaSuccess) return -1;
    if (c.prof) {   // this replay's force-kernel marks: the next two pool events
        for (int k = 0; k < 2; ++k) {
            if (c.ev_used == c.ev_pool.size()) {
                cudaEvent_t e;
                if (cudaEventCreate(&e) != cudaSuccess) return -1;
                c.ev_pool.push_back(e);
            }
            if (cudaGraphExecEventRecordNodeSetEvent(g->exec, g->pnode[k], c.ev_pool[c.ev_used++]) != cudaSuccess)
                return -1;
        }
    }
    if (cudaGraphLaunch(g->exec, c.stream) != cudaSuccess) return -1;
    note_launches(g->nkern);
    return 0;
}

int mdg_run(mdg_ctx* ctx, const mdg_config* cfg, int64_t steps, double dt, int has_gravity,
            double gravity, int rebuild_interval, int64_t iteration0, int rebuild_now, int* since,
            int* kick_due, int* swaps, int64_t* done, int* flags) {
    MDG_RANGE("mdg_run");
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    if (int e = need_system(ctx)) return e;
    if (!since || !kick_due || !swaps || !done || !flags || steps < 0 || rebuild_interval < 0) {
        set_error("mdg_run: bad arguments");
        return MDG_EINVAL;
    }
    Context& c = ctx->c;
    *done = 0;
    *flags = 0;
    for (int64_t k = 0; k < steps; ++k) {
        c.iter_tag = iteration0 + k;
        const bool rebuild = rebuild_now || *since >= rebuild_interval;
        if (!rebuild && *kick_due && run_graph_env()) {
            const int r = run_graph_step(c, cfg, dt, has_gravity, gravity);
            if (r < 0) return cuda_status("mdg_run: step graph");
            if (r == 0) {
                std::swap(c.force, c.old_force);
                ++c.gen;
                ++*swaps;
                *since += 1;
                *done = k + 1;
                continue;
            }
        }
        if (*kick_due) {
            if (int e = mdg_kick_drift(ctx, dt, has_gravity, gravity, 0)) return e;
            std::swap(c.force, c.old_force);
            ++c.gen;
            ++*swaps;
            *kick_due = 0;
        } else if (int e = mdg_drift_wrap(ctx, dt)) {
            return e;
        }
        if (rebuild) {
            int f = 0;
            if (int e = mdg_rebuild_checked(ctx, cfg, &f)) return e;
            if (f) {
                *flags = f;
                return MDG_OK;
            }
            rebuild_now = 0;
        }
        if (int e = mdg_refresh(ctx, cfg)) return e;
        if (int e = mdg_compute(ctx, cfg)) return e;
        *kick_due = 1;
        *since = rebuild ? 0 : *since + 1;
        *done = k + 1;
    }
    return MDG_OK;
}

int mdg_ghost_pack(mdg_ctx* ctx, const int64_t* idx, int64_t n_left, int64_t n_right, int axis,
                   double shift_left, double shift_right, double* out) {
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    Context& c = ctx->c;
    if (axis < 0 || axis > 2 || n_left < 0 || n_right < 0 || ((n_left + n_right) && (!idx || !out))) {
        set_error("mdg_ghost_pack: bad arguments");
        return MDG_EINVAL;
    }
    halo_pack(c, idx, n_left, n_left + n_right, axis, shift_left, shift_right, out);
    return cuda_status("mdg_ghost_pack");
}

int mdg_ghost_unpack(mdg_ctx* ctx, const double* in, int64_t count, int64_t row0) {
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    Context& c = ctx->c;
    if (count < 0 || row0 < 0 || row0 + count > c.n || (count && !in)) {
        set_error("mdg_ghost_unpack: rows outside the bound set");
        return MDG_EINVAL;
    }
    halo_unpack(c, in, count, row0);
    return cuda_status("mdg_ghost_unpack");
}

int mdg_gather_rows(mdg_ctx* ctx, const int64_t* order, int64_t n, int layout, const double* const* src,
                    double* const* dst, const int* tid_src, int* tid_dst) {
    CHECK_CTX(ctx);
    if (n < 0 || (n && (!order || !src || !dst)) || (layout != MDG_AOS && layout != MDG_SOA) ||
        (!tid_src != !tid_dst)) {
        set_error("mdg_gather_rows: bad arguments");
        return MDG_EINVAL;
    }
    Rows4 s, d;
    for (int k = 0; k < 4; ++k) {
        s.p[k] = const_cast<double*>(src[k]);
        d.p[k] = dst[k];
        if (n && (!s.p[k] || !d.p[k])) {
            set_error("mdg_gather_rows: null array");
            return MDG_EINVAL;
        }
    }
    gather_rows(ctx->c, order, n, layout, s, d, tid_src, tid_dst);
    return cuda_status("mdg_gather_rows");
}

int mdg_permutation(mdg_ctx* ctx, int op, int64_t n, const int64_t* a, const int64_t* b, int64_t* out) {
    CHECK_CTX(ctx);
    if (n < 0 || op < 0 || op > 2 || (n && (!a || !out || (op == 0 && !b)))) {
        set_error("mdg_permutation: bad arguments");
        return MDG_EINVAL;
    }
    permutation(ctx->c, op, n, a, b, out);
    return cuda_status("mdg_permutation");
}

int mdg_set_force_rows(mdg_ctx* ctx, int64_t n_force) {
    CHECK_CTX(ctx);
    ctx->c.n_force = n_force < 0 ? INT64_MAX : n_force;
    return MDG_OK;
}

int mdg_sd_step(mdg_ctx* ctx, double gamma, double max_disp) {
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    integ_sd_step(ctx->c, gamma, max_disp);
    return cuda_status("mdg_sd_step");
}

int mdg_blowup(mdg_ctx* ctx, int* flag, int reset) {
    CHECK_CTX(ctx);
    Context& c = ctx->c;
    if (cudaMemcpyAsync(c.h_scal + 2, c.scal.p + 2, sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, c.stream) != cudaSuccess ||
        cudaStreamSynchronize(c.stream) != cudaSuccess)
        return cuda_status("mdg_blowup");
    *flag = (int)(c.h_scal[2] & 3ull);
    if (reset) cudaMemsetAsync(c.scal.p + 2, 0, sizeof(unsigned long long), c.stream);
    return cuda_status("mdg_blowup");
}

int mdg_set_iteration(mdg_ctx* ctx, int64_t iteration) {
    CHECK_CTX(ctx);
    ctx->c.iter_tag = iteration;
    return MDG_OK;
}

int mdg_blowup_iteration(mdg_ctx* ctx, int64_t* iteration) {
    CHECK_CTX(ctx);
    if (!iteration) { set_error("null output"); return MDG_EINVAL; }
    Context& c = ctx->c;
    if (cudaMemcpyAsync(c.h_scal + 8, c.scal.p + 8, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        c.stream) != cudaSuccess ||
        cudaStreamSynchronize(c.stream) != cudaSuccess)
        return cuda_status("mdg_blowup_iteration");
    *iteration = c.h_scal[8] == ~0ull ? -1 : (int64_t)c.h_scal[8];
    cudaMemsetAsync(c.scal.p + 8, 0xff, sizeof(unsigned long long), c.stream);   // read and reset
    return cuda_status("mdg_blowup_iteration");
}

int mdg_temperature(mdg_ctx* ctx, double* temperature) {
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    if (!temperature) { set_error("null output"); return MDG_EINVAL; }
    int r = stats_temperature(ctx->c, temperature);
    if (r > 0) return MDG_EINVAL;
    if (r < 0) return MDG_ECUDA;
    return cuda_status("mdg_temperature");
}

int mdg_thermostat(mdg_ctx* ctx, double target, double max_delta_t) {
    MDG_RANGE("mdg_thermostat");
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    int r = stats_thermostat(ctx->c, target, max_delta_t);
    if (r > 0) return MDG_EINVAL;
    if (r < 0) return MDG_ECUDA;
    return cuda_status("mdg_thermostat");
}

int mdg_live_stats(mdg_ctx* ctx, double out[6]) {
    MDG_RANGE("mdg_live_stats");
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    if (!out) { set_error("null output"); return MDG_EINVAL; }
    int r = stats_live(ctx->c, out);
    if (r > 0) return MDG_EINVAL;
    if (r < 0) return MDG_ECUDA;
    return cuda_status("mdg_live_stats");
}

int mdg_profile(mdg_ctx* ctx, int enable) {
    CHECK_CTX(ctx);
    Context& c = ctx->c;
    c.prof = enable != 0;
    c.ev_used = 0;
    // enable > 1: that many bracketed launches reserved now, so a timed loop
    // creates no events (the pool otherwise grows on demand, two per launch)
    if (enable > 1) {
        while (c.ev_pool.size() < 2 * (size_t)enable) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return cuda_status("mdg_profile: events");
            c.ev_pool.push_back(e);
        }
    }
    return MDG_OK;
}

int mdg_profile_read(mdg_ctx* ctx, double* total_ms, int64_t* launches) {
    CHECK_CTX(ctx);
    Context& c = ctx->c;
    if (cudaStreamSynchronize(c.stream) != cudaSuccess) return cuda_status("mdg_profile_read");
    double tot = 0.0;
    for (size_t k = 0; k + 1 < c.ev_used; k += 2) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c.ev_pool[k], c.ev_pool[k + 1]);
        tot += ms;
    }
    *total_ms = tot;
    *launches = (int64_t)(c.ev_used / 2);
    c.ev_used = 0;
    return cuda_status("mdg_profile_read");
}

int mdg_synchronize(mdg_ctx* ctx) {
    CHECK_CTX(ctx);
    if (cudaStreamSynchronize(ctx->c.stream) != cudaSuccess) return cuda_status("synchronize");
    return cuda_status("synchronize");
}

int mdg_h2d(mdg_ctx* ctx, void* dev, const void* host, size_t bytes) {
    CHECK_CTX(ctx);
    if (!bytes) return MDG_OK;
    if (cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->c.stream) != cudaSuccess)
        return cuda_status("mdg_h2d");
    return MDG_OK;
}

int mdg_d2h(mdg_ctx* ctx, void* host, const void* dev, size_t bytes) {
    CHECK_CTX(ctx);
    if (!bytes) return MDG_OK;
    if (cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->c.stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->c.stream) != cudaSuccess)
        return cuda_status("mdg_d2h");
    return MDG_OK;
}

int mdg_host_step(mdg_ctx* ctx, const mdg_config* cfg, double* pos, double* vel, double* force,
                  double* old_force, const int32_t* type_id, const double* mass, double dt,
                  int has_gravity, double gravity, int rebuild, int chunks, int* blowup) {
    return mdg_host_step_ex(ctx, cfg, pos, vel, force, old_force, type_id, mass, dt, has_gravity,
                            gravity, rebuild, chunks, 0, blowup);
}

int mdg_host_step_ex(mdg_ctx* ctx, const mdg_config* cfg, double* pos, double* vel, double* force,
                     double* old_force, const int32_t* type_id, const double* mass, double dt,
                     int has_gravity, double gravity, int rebuild, int chunks, int flags, int* blowup) {
    MDG_RANGE("mdg_host_step_ex");
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    if (int e = need_system(ctx)) return e;
    Context& c = ctx->c;
    if (blowup) *blowup = 0;
    int64_t n = c.n;
    if (n == 0) return MDG_OK;
    if (!c.pos || !c.force) { set_error("mdg_host_step: bind the device arrays first"); return MDG_ESTATE; }
    int K = std::max(1, std::min<int>(chunks, (int)std::min<int64_t>(n, 64)));
    while ((int)c.chunk_ev.size() < K) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return cuda_status("event");
        c.chunk_ev.push_back(e);
    }
    int periodic[3] = {c.periodic[0], c.periodic[1], c.periodic[2]};
    // pieces (byte offset, bytes) of particles [a, b) in the bound layout
    auto copy = [&](double* dst, const double* src, int64_t a, int64_t b, cudaMemcpyKind kind) {
        if (c.layout == AOS)
            return cudaMemcpyAsync(dst + 3 * a, src + 3 * a, 24 * (b - a), kind, c.stream);
        for (int k = 0; k < 3; ++k) {
            cudaError_t e = cudaMemcpyAsync(dst + k * n + a, src + k * n + a, 8 * (b - a), kind, c.stream);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    };
    static int timing = getenv("MDG_HOST_STEP_TIMING") ? 1 : 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    int bad = 0;
    for (int k = 0; k < K; ++k) {
        int64_t a = n * k / K, b = n * (k + 1) / K;
        int bk = 0;
        mdg_host_drift_wrap_range_ex(n, a, b, c.layout, pos, vel, force, old_force, type_id, mass,
                                     c.L, periodic, dt, flags & MDG_HOST_STEP_SWAPPED, &bk);
        bad |= bk;
        if (copy(c.pos, pos, a, b, cudaMemcpyHostToDevice) != cudaSuccess) return cuda_status("h2d");
    }
    if (bad) {
        if (blowup) *blowup = 1;
        cudaStreamSynchronize(c.stream);
        return cuda_status("mdg_host_step");
    }
    auto t1 = now();
    if (rebuild)
        if (int e = mdg_rebuild(ctx, cfg)) return e;
    if (int e = mdg_refresh(ctx, cfg)) return e;
    if (int e = mdg_compute(ctx, cfg)) return e;
    for (int k = 0; k < K; ++k) {
        int64_t a = n * k / K, b = n * (k + 1) / K;
        if (copy(force, c.force, a, b, cudaMemcpyDeviceToHost) != cudaSuccess) return cuda_status("d2h");
        cudaEventRecord(c.chunk_ev[k], c.stream);
    }
    auto t2 = now();
    double wait_us = 0.0;
    for (int k = 0; k < K; ++k) {
        int64_t a = n * k / K, b = n * (k + 1) / K;
        auto w0 = now();
        if (cudaEventSynchronize(c.chunk_ev[k]) != cudaSuccess) return cuda_status("d2h wait");
        wait_us += std::chrono::duration<double, std::micro>(now() - w0).count();
        mdg_host_finish_kick_range(n, a, b, c.layout, vel, force, old_force, type_id, mass, dt,
                                   has_gravity, gravity);
    }
    if (timing) {
        auto t3 = now();
        auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
        fprintf(stderr, "host_step: drift+h2d %.0f us, device enqueue %.0f us, d2h waits %.0f us, "
                        "kicks %.0f us, total %.0f us%s\n",
                us(t0, t1), us(t1, t2), wait_us, us(t2, t3) - wait_us, us(t0, t3), rebuild ? " (rebuild)" : "");
    }
    return cuda_status("mdg_host_step");
}

int mdg_host_run(mdg_ctx* ctx, const mdg_config* cfg, double* pos, double* vel, double* force,
                 double* old_force, const int32_t* type_id, const double* mass, double dt,
                 int has_gravity, double gravity, int steps, int rebuild_interval, int since,
                 int rebuild_first, int chunks, int* blowup, int* steps_done) {
    MDG_RANGE("mdg_host_run");
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    if (int e = need_system(ctx)) return e;
    Context& c = ctx->c;
    if (blowup) *blowup = 0;
    if (steps_done) *steps_done = 0;
    if (steps < 0 || rebuild_interval < 0) { set_error("mdg_host_run: negative steps"); return MDG_EINVAL; }
    int64_t n = c.n;
    if (n == 0 || steps == 0) {
        if (steps_done) *steps_done = n == 0 ? steps : 0;
        return MDG_OK;
    }
    if (!c.pos || !c.force) { set_error("mdg_host_run: bind the device arrays first"); return MDG_ESTATE; }
    int K = std::max(1, std::min<int>(chunks, (int)std::min<int64_t>(n, 64)));
    while ((int)c.chunk_ev.size() < K) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return cuda_status("event");
        c.chunk_ev.push_back(e);
    }
    if (!c.copy_stream) {
        if (cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c.h2d_done, cudaEventDisableTiming) != cudaSuccess)
            return cuda_status("mdg_host_run streams");
    }
    int periodic[3] = {c.periodic[0], c.periodic[1], c.periodic[2]};
    auto copy = [&](double* dst, const double* src, int64_t a, int64_t b, cudaMemcpyKind kind,
                    cudaStream_t st) {
        if (c.layout == AOS) return cudaMemcpyAsync(dst + 3 * a, src + 3 * a, 24 * (b - a), kind, st);
        for (int k = 0; k < 3; ++k) {
            cudaError_t e = cudaMemcpyAsync(dst + k * n + a, src + k * n + a, 8 * (b - a), kind, st);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    };
    static int timing = getenv("MDG_HOST_STEP_TIMING") ? 1 : 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
    double t_enq = 0, t_wait = 0, t_host = 0, t_first = 0;
    auto T0 = now();
    // error exits drain both streams first: no copy may still be reading or
    // writing the caller's host arrays when the call returns
    auto drained = [&](int code) {
        cudaStreamSynchronize(c.copy_stream);
        cudaStreamSynchronize(c.stream);
        return code;
    };
    // the caller's buffers arrive swapped (MDG_HOST_STEP_SWAPPED): old_force
    // holds the current forces, force is free; the roles alternate per step
    double* cur = old_force;
    double* oth = force;
    // drift of the first step, chunks uploaded on the copy stream as they finish
    int bad = 0;
    for (int k = 0; k < K; ++k) {
        int64_t a = n * k / K, b = n * (k + 1) / K;
        int bk = 0;
        mdg_host_drift_wrap_range_ex(n, a, b, c.layout, pos, vel, nullptr, cur, type_id, mass, c.L,
                                     periodic, dt, 1, &bk);
        bad |= bk;
        if (copy(c.pos, pos, a, b, cudaMemcpyHostToDevice, c.copy_stream) != cudaSuccess) return drained(cuda_status("h2d"));
    }
    cudaEventRecord(c.h2d_done, c.copy_stream);
    if (bad) {
        cudaStreamSynchronize(c.copy_stream);
        if (blowup) *blowup = 1;
        return cuda_status("mdg_host_run");
    }
    for (int s = 0; s < steps; ++s) {
        bool last = s == steps - 1;
        bool rebuild = (s == 0 && rebuild_first) || since >= rebuild_interval;
        auto ta = now();
        if (cudaStreamWaitEvent(c.stream, c.h2d_done, 0) != cudaSuccess) return drained(cuda_status("wait h2d"));
        if (rebuild)
            if (int e = mdg_rebuild(ctx, cfg)) return drained(e);
        if (int e = mdg_refresh(ctx, cfg)) return drained(e);
        if (int e = mdg_compute(ctx, cfg)) return drained(e);
        for (int k = 0; k < K; ++k) {
            int64_t a = n * k / K, b = n * (k + 1) / K;
            if (copy(oth, c.force, a, b, cudaMemcpyDeviceToHost, c.stream) != cudaSuccess) return drained(cuda_status("d2h"));
            cudaEventRecord(c.chunk_ev[k], c.stream);
        }
        auto tb = now();
        t_enq += us(ta, tb);
        // each chunk as it lands: kick of this step, drift of the next, upload
        // (the H2D runs on the copy stream, overlapping the remaining D2H)
        for (int k = 0; k < K; ++k) {
            int64_t a = n * k / K, b = n * (k + 1) / K;
            auto w0 = now();
            if (cudaEventSynchronize(c.chunk_ev[k]) != cudaSuccess) return drained(cuda_status("d2h wait"));
            auto w1 = now();
            t_wait += us(w0, w1);
            if (k == 0) t_first += us(w0, w1);
            struct Acc {
                double& t; std::chrono::steady_clock::time_point s;
                ~Acc() { t += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - s).count(); }
            } acc{t_host, w1};
            if (last) {
                mdg_host_finish_kick_range(n, a, b, c.layout, vel, oth, cur, type_id, mass, dt,
                                           has_gravity, gravity);
                continue;
            }
            int bk = 0;
            mdg_host_kick_drift_range(n, a, b, c.layout, pos, vel, oth, cur, type_id, mass, c.L,
                                      periodic, dt, has_gravity, gravity, &bk);
            bad |= bk;
            if (copy(c.pos, pos, a, b, cudaMemcpyHostToDevice, c.copy_stream) != cudaSuccess) return drained(cuda_status("h2d"));
        }
        if (!last) cudaEventRecord(c.h2d_done, c.copy_stream);
        since = rebuild ? 0 : since + 1;
        std::swap(cur, oth);
        if (steps_done) *steps_done = s + 1;
        if (bad) {   // the next step's drift left the domain: stop before its force pass
            cudaStreamSynchronize(c.copy_stream);
            if (blowup) *blowup = 1;
            break;
        }
    }
    if (timing && steps_done && *steps_done > 0) {
        double k = *steps_done;
        fprintf(stderr, "host_run: %d steps x %d chunks: per step %.0f us = device enqueue %.0f, "
                        "d2h waits %.0f (first chunk %.0f), host kick+drift+h2d enqueue %.0f\n",
                *steps_done, K, us(T0, now()) / k, t_enq / k, t_wait / k, t_first / k, t_host / k);
    }
    return cuda_status("mdg_host_run");
}

int mdg_d2h_async(mdg_ctx* ctx, void* host, const void* dev, size_t bytes) {
    CHECK_CTX(ctx);
    if (!bytes) return MDG_OK;
    if (cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->c.stream) != cudaSuccess)
        return cuda_status("mdg_d2h_async");
    return MDG_OK;
}

int mdg_geometry(mdg_ctx* ctx, double csf, int dims_owned[3], double cell_length[3],
                 int overlap[3], int halo[3], int dims[3]) {
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    if (csf != 1.0 && csf != 0.5) { set_error("csf must be 1 or 0.5"); return MDG_EINVAL; }
    const Geom& g = grid_for(ctx->c, csf)->g;
    for (int k = 0; k < 3; ++k) {
        dims_owned[k] = g.S[k];
        cell_length[k] = g.cl[k];
        overlap[k] = g.overlap[k];
        halo[k] = g.H[k];
        dims[k] = g.D[k];
    }
    return MDG_OK;
}

int mdg_stencil(mdg_ctx* ctx, double csf, int kind, int major, int* count, int* out) {
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    if (csf != 1.0 && csf != 0.5) { set_error("csf must be 1 or 0.5"); return MDG_EINVAL; }
    if (major < 0 || major > 2) { set_error("major axis must be 0..2"); return MDG_EINVAL; }
    const Geom& g = grid_for(ctx->c, csf)->g;
    Stencil s = kind == 0 ? pruned_stencil(g) : forward_stencil(g, major);
    *count = s.n;
    if (out) memcpy(out, s.d, sizeof(int) * 3 * s.n);
    return MDG_OK;
}

int mdg_geometry_for(const double domain[3], const int periodic[3], double ell, double csf,
                     int dims_owned[3], double cell_length[3], int overlap[3], int halo[3],
                     int dims[3]) {
    if (!(ell > 0) || (csf != 1.0 && csf != 0.5)) { set_error("bad geometry arguments"); return MDG_EINVAL; }
    Geom g = make_geometry(domain, periodic, ell, csf);
    for (int k = 0; k < 3; ++k) {
        dims_owned[k] = g.S[k];
        cell_length[k] = g.cl[k];
        overlap[k] = g.overlap[k];
        halo[k] = g.H[k];
        dims[k] = g.D[k];
    }
    return MDG_OK;
}

int mdg_stencil_for(const double domain[3], const int periodic[3], double ell, double csf,
                    int kind, int major, int* count, int* out) {
    if (!(ell > 0) || (csf != 1.0 && csf != 0.5) || major < 0 || major > 2) {
        set_error("bad stencil arguments");
        return MDG_EINVAL;
    }
    Geom g = make_geometry(domain, periodic, ell, csf);
    Stencil s = kind == 0 ? pruned_stencil(g) : forward_stencil(g, major);
    *count = s.n;
    if (out) memcpy(out, s.d, sizeof(int) * 3 * s.n);
    return MDG_OK;
}

int mdg_get_grid(mdg_ctx* ctx, double csf, int64_t* m, int64_t* ncells, int32_t* src,
                 int8_t* shift_code, int32_t* start) {
    CHECK_CTX(ctx);
    if (csf != 1.0 && csf != 0.5) { set_error("csf must be 1 or 0.5"); return MDG_EINVAL; }
    Grid& gr = *grid_for(ctx->c, csf);
    if (!gr.built) { set_error("grid not built"); return MDG_ESTATE; }
    cudaStreamSynchronize(ctx->c.stream);
    if (m) *m = gr.m;
    if (ncells) *ncells = gr.g.ncells;
    if (src && gr.m) cudaMemcpy(src, gr.row_src.p, gr.m * sizeof(int), cudaMemcpyDeviceToHost);
    if (shift_code && gr.m)
        cudaMemcpy(shift_code, gr.row_code.p, gr.m, cudaMemcpyDeviceToHost);
    if (start) cudaMemcpy(start, gr.cell_start.p, (gr.g.ncells + 1) * sizeof(int), cudaMemcpyDeviceToHost);
    return cuda_status("mdg_get_grid");
}

int mdg_owned_order(mdg_ctx* ctx, const mdg_config* cfg, int32_t* order) {
    CHECK_CTX(ctx);
    if (int e = validate(cfg)) return e;
    if (!order) { set_error("null output"); return MDG_EINVAL; }
    Context& c = ctx->c;
    Grid& gr = cfg->container == MDG_VL ? c.vl.grid : cfg->container == MDG_VCL ? c.vcl.grid : *grid_for(c, cfg->csf);
    if (!gr.built || gr.n != c.n) { set_error("grid not built for the bound particles"); return MDG_ESTATE; }
    if (grid_owned_order(c, gr, order)) return MDG_ECUDA;
    return cuda_status("mdg_owned_order");
}

int mdg_potential_energy(mdg_ctx* ctx, int rebuild, double* pe) {
    CHECK_CTX(ctx);
    if (int e = need_system(ctx)) return e;
    if (!pe) { set_error("null output"); return MDG_EINVAL; }
    Context& c = ctx->c;
    if (rebuild || !c.vl.built)
        if (vl_rebuild(c)) return MDG_ECUDA;
    if (vl_energy(c, pe)) return MDG_ECUDA;
    return cuda_status("mdg_potential_energy");
}

int mdg_get_verlet(mdg_ctx* ctx, int64_t* entries, int64_t* noff, int32_t* nbr) {
    CHECK_CTX(ctx);
    Verlet& v = ctx->c.vl;
    if (!v.built) { set_error("Verlet lists not built"); return MDG_ESTATE; }
    int64_t e = 0;
    if (vl_export(ctx->c, &e, noff, nbr)) return MDG_ECUDA;
    if (entries) *entries = e;
    return cuda_status("mdg_get_verlet");
}

}  // extern "C"
