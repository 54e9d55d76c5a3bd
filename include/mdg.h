/*
 * mdg.h — C ABI of libmdg, the B200-native (sm_100a) Lennard-Jones force and
 * neighbour-identification path of the mdtune reference
 * (arXiv 2505.03438 re-creation, /root/reference/pkg/src/mdtune).
 *
 * The reference's drop-in boundary for this path is the Python protocol
 * `ForceCalculator(particles, params)` with `rebuild / refresh / compute /
 * last_eval_count` (containers.py:378-488), looked up as a module global by
 * `simulate` (simulation.py:21,144) and `measure_configuration_costs`
 * (dataset.py:21,114), plus the Verlet update around it (integrator.py:31-128).
 * Every entry point below replaces one piece of that surface; the mapping is
 * given per function.  All pointers are plain device pointers unless a
 * parameter is documented as host memory; no torch types cross this ABI.
 *
 * Return value of every int function: 0 = ok, MDG_EINVAL = invalid argument
 * (the reference raises ValueError), MDG_ECUDA = CUDA failure (RuntimeError),
 * MDG_ESTATE = called out of order (e.g. compute before rebuild).
 * mdg_last_error() returns the thread-local message of the last failure.
 *
 * Threading: one context per GPU, driven from one host thread; all work is
 * enqueued on the context's stream (containers.py / SPEC.md:105-106: the
 * calculator is single-threaded from the caller's side).
 */
#ifndef MDG_H
#define MDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDG_OK 0
#define MDG_EINVAL 1
#define MDG_ECUDA 2
#define MDG_ESTATE 3

/* configuration.py:7-17; MDG_VCL / MDG_CLUSTER_ITER are the north_star's
 * VerletClusterLists container (no reference implementation; GPU-only ids
 * appended to the space). */
enum { MDG_LC = 0, MDG_VL = 1, MDG_VCL = 2 };
enum { MDG_C01 = 0, MDG_C08 = 1, MDG_C18 = 2, MDG_SLI = 3, MDG_LIST_ITER = 4, MDG_CLUSTER_ITER = 5 };
/* particles.py:10-11 */
enum { MDG_AOS = 0, MDG_SOA = 1 };

/* Arithmetic of the force functor (north_star): fp64 throughout, or fp32
 * compute with fp64 accumulation (Verlet lists only; tolerance 1e-4). */
enum { MDG_FP64 = 0, MDG_FP32 = 1 };

/* One point of the search space: Configuration (configuration.py:20-50),
 * plus the precision of the extended space (the reference's 30 are fp64). */
typedef struct {
    int container;  /* MDG_LC / MDG_VL / MDG_VCL */
    int traversal;  /* MDG_C01 .. MDG_CLUSTER_ITER */
    int newton3;    /* 0 / 1 */
    int layout;     /* MDG_AOS / MDG_SOA */
    double csf;     /* cell size factor, 1.0 or 0.5 */
    int precision;  /* MDG_FP64 / MDG_FP32 */
} mdg_config;

typedef struct mdg_ctx mdg_ctx;

/* Library version string. */
const char* mdg_version(void);
/* Number of kernel launches libmdg has issued in this process (evidence for
 * bench.py's gpu_launches). */
uint64_t mdg_launch_count(void);
/* Thread-local message of the last failing call ("" if none). */
const char* mdg_last_error(void);

/* Context on `device`, enqueuing on `stream` (a cudaStream_t, may be NULL for
 * the legacy default stream).  Replaces ForceCalculator.__init__'s allocation
 * of GridState / LayoutBuffers / VerletListState (containers.py:385-401). */
int mdg_create(int device, void* stream, mdg_ctx** out);
int mdg_destroy(mdg_ctx* ctx);
int mdg_set_stream(mdg_ctx* ctx, void* stream);

/* SimulationParams (params.py:35-101) + per-type LJ parameters
 * (particles.py:60-70) -> mixing tables (forces.py:12-22) and the CSF-1 /
 * CSF-0.5 geometries (cells.py:55-67, containers.py:390-396).  Validates like
 * SimulationParams.__post_init__.  sigma/epsilon/mass: host arrays of ntypes. */
int mdg_set_system(mdg_ctx* ctx, const double domain[3], const int periodic[3], double cutoff,
                   double skin, int ntypes, const double* sigma, const double* epsilon,
                   const double* mass);

/* Bind the caller-owned particle arrays (ParticleSet, particles.py:31-98):
 * pos/vel/force/old_force are fp64 device arrays in `layout` (AoS (n,3),
 * SoA (3,n)); type_id is int32 on the device (may be NULL for one type). */
int mdg_bind(mdg_ctx* ctx, int64_t n, int layout, double* pos, double* vel, double* force,
             double* old_force, const int32_t* type_id);

/* ForceCalculator.rebuild (containers.py:403-412): cell binning (stable
 * counting sort incl. periodic images) or Verlet-list build.  Synchronises
 * once (sizes of the image / list arrays). */
int mdg_rebuild(mdg_ctx* ctx, const mdg_config* cfg);
/* mdg_rebuild preceded by the loop's error check (simulation.py:158-166 with
 * the blow-up / thermostat status of mdg_blowup): the status word is read at
 * the rebuild's own first host synchronisation instead of a separate one.
 * *flags = the MDG_FLAG_* bits raised since the last reset (then reset); when
 * nonzero the rebuild was abandoned and the container must be rebuilt. */
int mdg_rebuild_checked(mdg_ctx* ctx, const mdg_config* cfg, int* flags);
/* ForceCalculator.refresh (containers.py:429-439): gather pos[src]+shift into
 * the cell-sorted scratch (no-op for Verlet lists).  Asynchronous. */
int mdg_refresh(mdg_ctx* ctx, const mdg_config* cfg);
/* ForceCalculator.compute (containers.py:441-488): overwrite `force` with the
 * LJ forces.  Asynchronous; the within-cutoff evaluation count accumulates on
 * the device (read it with mdg_eval_count).  MDG_EINVAL on layout mismatch
 * (containers.py:445-448). */
int mdg_compute(mdg_ctx* ctx, const mdg_config* cfg);
/* mdg_compute followed by apply_gravity + finish_kick (simulation.py:169-185,
 * integrator.py:40-51): the velocity update is fused into the force walk's
 * epilogue where the configuration allows it (tiled Verlet lists), else run
 * as its own kernel.  Same arithmetic either way.  Asynchronous. */
int mdg_compute_kick(mdg_ctx* ctx, const mdg_config* cfg, double dt, int has_gravity,
                     double gravity);
/* One steady-state loop iteration (no rebuild due): drift_wrap + refresh +
 * compute + finish_kick, replayed from a CUDA graph captured on first use and
 * re-captured whenever the configuration, dt / gravity, the bound arrays or
 * the container (any rebuild) changed.  Ordered on the context stream;
 * asynchronous.  MDG_ESTATE before the first rebuild. */
int mdg_step_graph(mdg_ctx* ctx, const mdg_config* cfg, double dt, int has_gravity, double gravity);
/* ForceCalculator.last_eval_count (containers.py:454): synchronises. */
int mdg_eval_count(mdg_ctx* ctx, int64_t* count);
/* Shifted LJ potential energy of the bound positions (no reference
 * ForceCalculator counterpart; the reference's energy test helper,
 * tests/test_integrator.py:227-247): 1/2 sum over within-cutoff pairs of
 * 4 eps [(s/r)^12 - (s/r)^6 - (s/rc)^12 + (s/rc)^6].  Uses the Verlet lists
 * (built first when `rebuild` != 0 or none exist).  Synchronises. */
int mdg_potential_energy(mdg_ctx* ctx, int rebuild, double* pe);

/* drift_with_force + apply_boundaries + copy force->old_force
 * (integrator.py:31-37, :98-128; simulation.py:151-153), fused. */
int mdg_drift_wrap(mdg_ctx* ctx, double dt);
/* apply_gravity + finish_kick (integrator.py:40-51; simulation.py:177,185). */
int mdg_finish_kick(mdg_ctx* ctx, double dt, int has_gravity, double gravity);
/* finish_kick of the previous step fused with this step's drift_wrap, one
 * pass over the bound state, bit-identical to mdg_finish_kick then
 * mdg_drift_wrap (integrator.py:31-51, 98-128).  copy_old_force = 0 skips the
 * F -> F_old copy: the caller then swaps its force / old_force buffers (and
 * re-binds) before the next compute. */
int mdg_kick_drift(mdg_ctx* ctx, double dt, int has_gravity, double gravity, int copy_old_force);
/* The reference loop for ONE configuration on the bound device state
 * (simulation.py:144-189 under a FixedStrategy, no timing / records, no
 * thermostat), iterations iteration0 .. iteration0 + steps - 1, as
 * Simulation.step runs them with the kick deferred into the next drift:
 * per iteration kick_drift (when *kick_due, force / old_force swapped instead
 * of copied) or drift_wrap; mdg_rebuild_checked when *since >= R or
 * *rebuild_now; refresh; compute.  One native call instead of ~10 ctypes
 * calls per iteration (small systems are host-bound otherwise).  In/out:
 * *since (iterations since the last rebuild), *kick_due (a kick is owed on
 * return: run mdg_finish_kick or pass it back in), *swaps (incremented per
 * force / old_force swap: the caller swaps its buffers when odd),
 * *done (iterations completed).  A raised status bit at a rebuild stops the
 * loop before that rebuild: *flags = the bits (as mdg_rebuild_checked).  The
 * eval count afterwards is that of the last compute. */
int mdg_run(mdg_ctx* ctx, const mdg_config* cfg, int64_t steps, double dt, int has_gravity,
            double gravity, int rebuild_interval, int64_t iteration0, int rebuild_now, int* since,
            int* kick_due, int* swaps, int64_t* done, int* flags);
/* Ghost exchange of the spatial domain decomposition (no
 * reference counterpart -- the decomposed stand-in for the periodic images of
 * cells.py:122-156).  pack: bound rows idx[0 .. n_left+n_right) -> AoS
 * (n_left+n_right, 3) `out` (device), + shift_left on `axis` for the first
 * n_left rows and + shift_right for the others.  unpack: AoS (count, 3) `in`
 * (device) -> bound rows [row0, row0+count) in the bound layout. */
int mdg_ghost_pack(mdg_ctx* ctx, const int64_t* idx, int64_t n_left, int64_t n_right, int axis,
                   double shift_left, double shift_right, double* out);
int mdg_ghost_unpack(mdg_ctx* ctx, const double* in, int64_t count, int64_t row0);
/* Row gather of the particle state (device pointers): dst_k[i] = src_k[order[i]]
 * for pos, vel, force, old_force (layout MDG_AOS (N,3) / MDG_SOA (3,N)) and,
 * when both are given, the int32 type ids -- the cell-order permutation of
 * Simulation(reorder=K) in one pass; no reference counterpart. */
int mdg_gather_rows(mdg_ctx* ctx, const int64_t* order, int64_t n, int layout, const double* const* src,
                    double* const* dst, const int* tid_src, int* tid_dst);
/* Index permutations of the cell reorder (no reference counterpart), on the
 * context stream: op 0 out[i] = a[b[i]] (composition), 1 out[a[i]] = i
 * (inverse), 2 out[i] = ((const int32_t*)a)[i] (mdg_owned_order's output
 * widened to int64; b unused).  Device pointers, n entries. */
int mdg_permutation(mdg_ctx* ctx, int op, int64_t n, const int64_t* a, const int64_t* b, int64_t* out);
/* Rows whose particle index is >= n_force get no force work (zero force, no
 * eval count) in the tiled Verlet walk: the decomposition's ghost rows, whose
 * forces are never used (n_force < 0: every row).  Exact for the owned rows
 * (NoN3L: a row's force is its own list's sum). */
int mdg_set_force_rows(mdg_ctx* ctx, int64_t n_force);
/* The caller's loop iteration of the drifts that follow (tagging only; no
 * device work), and the earliest tagged iteration whose drift raised the
 * blow-up bit since the last read (-1: none; read and reset; synchronises): the
 * loop reports the reference's failing iteration (integrator.py:108-116,
 * raised inside that iteration's apply_boundaries) although it checks the
 * status bit only at rebuilds. */
int mdg_set_iteration(mdg_ctx* ctx, int64_t iteration);
int mdg_blowup_iteration(mdg_ctx* ctx, int64_t* iteration);
/* Capped steepest-descent step x += F/|F| min(gamma|F|, max_disp) (input
 * relaxation for BASELINE configs 2/4; no reference counterpart). */
int mdg_sd_step(mdg_ctx* ctx, double gamma, double max_disp);
/* Device status bits raised since the last reset.  Synchronises.
 *   bit 0 (MDG_FLAG_BLOWUP): BlowUpError, integrator.py:108-116, set by any
 *          drift;
 *   bit 1 (MDG_FLAG_THERMO_ZERO): apply_thermostat met T = 0 with a positive
 *          target (the ValueError of integrator.py:84-88). */
#define MDG_FLAG_BLOWUP 1
#define MDG_FLAG_THERMO_ZERO 2
int mdg_blowup(mdg_ctx* ctx, int* flag, int reset);

/* current_temperature (integrator.py:72-78): T = sum m|v|^2 / (3N) over the
 * bound particles, summed in numpy's pairwise order so the value is
 * bit-identical to the reference.  MDG_EINVAL when N = 0.  Synchronises. */
int mdg_temperature(mdg_ctx* ctx, double* temperature);
/* apply_thermostat (integrator.py:81-95; simulation.py:186-188): velocity
 * rescaling toward `target`, |dT| clipped to `max_delta_t`, computed and
 * applied on the device without a host round trip.  The T = 0 / target > 0
 * error is reported through MDG_FLAG_THERMO_ZERO (velocities untouched).
 * MDG_EINVAL when N = 0. */
int mdg_thermostat(mdg_ctx* ctx, double target, double max_delta_t);
/* compute_live_stats (livestats.py:46-77) over the bound positions: CSF-1
 * bin counts with dims = max(1, floor(L/(cutoff+skin))), reduced to
 * out[0..5] = {mean, rel_std_dev, median, max, num_bins, num_empty} per bin,
 * bit-identical to the reference.  Synchronises. */
int mdg_live_stats(mdg_ctx* ctx, double out[6]);
/* Bracket every force-kernel launch with CUDA events on the context stream
 * (enable != 0; resets the record; enable > 1 also creates the events of that
 * many launches up front, so that a timed loop creates none).
 * mdg_profile_read synchronises and returns the summed kernel time and the
 * number of bracketed launches. */
int mdg_profile(mdg_ctx* ctx, int enable);
int mdg_profile_read(mdg_ctx* ctx, double* total_ms, int64_t* launches);
/* Wait for all work of the context's stream. */
int mdg_synchronize(mdg_ctx* ctx);

/* Host <-> device copies on the context stream (host-copy drop-in mode).
 * `host` should be pinned for full bandwidth.  d2h synchronises. */
int mdg_h2d(mdg_ctx* ctx, void* dev, const void* host, size_t bytes);
int mdg_d2h(mdg_ctx* ctx, void* host, const void* dev, size_t bytes);
/* device -> host copy enqueued on the context stream without waiting (the
 * pipelined host loop waits on an event per chunk). */
int mdg_d2h_async(mdg_ctx* ctx, void* host, const void* dev, size_t bytes);

/* The particles in the row order of the container `cfg` selects, as of its
 * last rebuild: order[k] = the particle of the k-th owned row (a permutation
 * of 0..n-1, written to the DEVICE buffer `order`, n int32).  No reference
 * counterpart: the device loop uses it to keep the particle arrays in cell
 * order (Simulation(reorder=...)), restoring the caller's order on flush. */
int mdg_owned_order(mdg_ctx* ctx, const mdg_config* cfg, int32_t* order);

/* Debug / parity exports (host buffers). */
/* make_geometry (cells.py:55-67) for csf. */
int mdg_geometry(mdg_ctx* ctx, double csf, int dims_owned[3], double cell_length[3],
                 int overlap[3], int halo[3], int dims[3]);
/* kind 0 = pruned_stencil (cells.py:80-95), 1 = forward_stencil with `major`
 * (cells.py:98-111).  out: 3*124 ints; *count = number of offsets. */
int mdg_stencil(mdg_ctx* ctx, double csf, int kind, int major, int* count, int* out);
/* GridState after the last rebuild of `csf` (containers.py:93-118): *m rows,
 * *ncells cells; src (m, int32), shift_code (m; (sx+1)*9+(sy+1)*3+(sz+1)),
 * start (ncells+1).  Any output pointer may be NULL (size query). */
int mdg_get_grid(mdg_ctx* ctx, double csf, int64_t* m, int64_t* ncells, int32_t* src,
                 int8_t* shift_code, int32_t* start);
/* VerletListState after the last VL rebuild (containers.py:352-375): noff
 * (n+1, int64) and nbr (entries, int32).  NULL outputs = size query. */
int mdg_get_verlet(mdg_ctx* ctx, int64_t* entries, int64_t* noff, int32_t* nbr);

/* The pairs every LC traversal evaluates within rc on the CSF-`csf` grid of
 * the last LC rebuild (r^2 < rc^2 on pos[src] + shift, kernels.py:36-40), as
 * owner pairs (src_i, src_j), src_i < src_j, in no particular order (the
 * caller sorts): the "LC pair set" of SURVEY §8(c)(ii).  *count = number of
 * pairs; at most `cap` are written to pairs (2 x int32 each); pairs may be
 * NULL (size query). */
int mdg_lc_pairs(mdg_ctx* ctx, double csf, int64_t cap, int32_t* pairs, int64_t* count);

/* Device timings of the reference's timing hooks (simulation.py:155-181):
 * build = mdg_rebuild (when called) + mdg_refresh, force = mdg_compute,
 * measured with CUDA events on the context stream.  enable >= 0 switches the
 * events on (1) or off (0) and returns; enable < 0 reads the last completed
 * intervals in ns (-1 = not measured), waiting for them. */
int mdg_timings(mdg_ctx* ctx, int enable, int64_t* build_ns, int64_t* force_ns);

/* Dynamic pruning of the tiled Verlet-list walk (no reference counterpart;
 * an execution detail of vl_force_aos/_soa, kernels.py:730-818).  After each
 * VL rebuild the walk writes inner lists of the entries within rc + delta and
 * walks them while every particle has moved less than delta / 2 since; a
 * larger move re-prunes from the full lists.  Pair sets within rc, counts and
 * forces are those of the full walk (forces up to the grouping of the
 * batched reciprocal, ~1e-16 relative).  delta < 0: default (env
 * MDG_VL_PRUNE_DELTA, else skin / 3; MDG_VL_PRUNE=0 disables); 0: off;
 * > 0: that delta (off if >= skin).  Applies from the next rebuild. */
int mdg_set_prune(mdg_ctx* ctx, double delta);
/* Prune walks since the last VL rebuild (-1 when pruning is off); synchronises. */
int mdg_prune_count(mdg_ctx* ctx, int64_t* prunes);

/* Context-free host versions of the two exports above (no device needed). */
int mdg_geometry_for(const double domain[3], const int periodic[3], double interaction_length,
                     double csf, int dims_owned[3], double cell_length[3], int overlap[3],
                     int halo[3], int dims[3]);
int mdg_stencil_for(const double domain[3], const int periodic[3], double interaction_length,
                    double csf, int kind, int major, int* count, int* out);

/* Host-side integrator of the host-resident drop-in path (host arrays, OpenMP,
 * same rounding as mdg_drift_wrap / mdg_finish_kick and the reference's numpy
 * sequence, integrator.py:31-51, :98-128).  mass: per type; type_id may be
 * NULL (one type); *blowup set when a coordinate left [-L, 2L] or is NaN. */
int mdg_host_drift_wrap(int64_t n, int layout, double* pos, double* vel, const double* force,
                        double* old_force, const int32_t* type_id, const double* mass,
                        const double domain[3], const int periodic[3], double dt, int* blowup);
int mdg_host_finish_kick(int64_t n, int layout, double* vel, double* force, const double* old_force,
                         const int32_t* type_id, const double* mass, double dt, int has_gravity,
                         double gravity);
/* The same on particles [begin, end) of an n-particle set (SoA stride n), so
 * a host loop can overlap the update of one chunk with the copy of another. */
int mdg_host_drift_wrap_range(int64_t n, int64_t begin, int64_t end, int layout, double* pos,
                              double* vel, const double* force, double* old_force,
                              const int32_t* type_id, const double* mass, const double domain[3],
                              const int periodic[3], double dt, int* blowup);
int mdg_host_finish_kick_range(int64_t n, int64_t begin, int64_t end, int layout, double* vel,
                               double* force, const double* old_force, const int32_t* type_id,
                               const double* mass, double dt, int has_gravity, double gravity);

/* One full reference-loop iteration (simulation.py:150-185) on HOST state
 * with the device force path, pipelined: the host drift of particle chunk k
 * runs while chunk k-1's positions copy to the bound device `pos`; then
 * rebuild (when `rebuild`) + refresh + compute; then the forces copy back in
 * chunks and each chunk is kicked on the host as soon as it lands.  Host
 * arrays pos/vel/force/old_force (layout of the bound set, pinned for DMA
 * speed) are the caller's ParticleSet; the device arrays are those of
 * mdg_bind.  Same arithmetic as mdg_host_drift_wrap / mdg_host_finish_kick,
 * bit-identical to the unpipelined sequence.  *blowup set (and nothing after
 * the drift done) when a coordinate left [-L, 2L].  Returns when the step is
 * complete on the host. */
int mdg_host_step(mdg_ctx* ctx, const mdg_config* cfg, double* pos, double* vel, double* force,
                  double* old_force, const int32_t* type_id, const double* mass, double dt,
                  int has_gravity, double gravity, int rebuild, int chunks, int* blowup);
/* The same with flags: MDG_HOST_STEP_SWAPPED = the caller swapped its force
 * and old_force buffers before the call (old_force holds the current forces,
 * force is scratch), which makes the drift's F -> F_old copy unnecessary; the
 * state after the step is identical. */
#define MDG_HOST_STEP_SWAPPED 1
int mdg_host_step_ex(mdg_ctx* ctx, const mdg_config* cfg, double* pos, double* vel, double* force,
                     double* old_force, const int32_t* type_id, const double* mass, double dt,
                     int has_gravity, double gravity, int rebuild, int chunks, int flags, int* blowup);
/* mdg_host_drift_wrap_range reading the current forces from old_force
 * without copying (swapped != 0), see MDG_HOST_STEP_SWAPPED. */
int mdg_host_drift_wrap_range_ex(int64_t n, int64_t begin, int64_t end, int layout, double* pos,
                                 double* vel, const double* force, double* old_force,
                                 const int32_t* type_id, const double* mass, const double domain[3],
                                 const int periodic[3], double dt, int swapped, int* blowup);

/* `steps` reference-loop iterations on HOST state in one call, pipelined
 * across step boundaries: after the force pass of step s the forces copy back
 * in `chunks` pieces, and as each lands the host runs the kick of step s and
 * the drift of step s+1 on it in one pass (mdg_host_kick_drift_range) and
 * uploads its positions on a second stream, so the H2D of step s+1 overlaps
 * the D2H of step s and the next force pass waits only for the last chunk.
 * Buffers as for MDG_HOST_STEP_SWAPPED on entry (old_force = current forces);
 * the two force buffers alternate roles per step, so after an EVEN number of
 * completed steps the latest forces are in old_force (the caller swaps its
 * names back).  Rebuild before step s when (s == 0 && rebuild_first) or
 * `since` (steps since the last rebuild, updated per step) >= rebuild_interval
 * (simulation.py:158-159, 179).  Per particle the arithmetic and its order
 * are those of mdg_host_step, so the state after k steps is bit-identical to
 * k calls of it.  *steps_done = completed steps; *blowup set when a drift
 * left [-L, 2L] (the run stops before that step's force pass). */
int mdg_host_run(mdg_ctx* ctx, const mdg_config* cfg, double* pos, double* vel, double* force,
                 double* old_force, const int32_t* type_id, const double* mass, double dt,
                 int has_gravity, double gravity, int steps, int rebuild_interval, int since,
                 int rebuild_first, int chunks, int* blowup, int* steps_done);
/* Kick of step s then drift of step s+1 on particles [begin, end) in one
 * pass: gravity into fnew.z, v += (fnew + fold) dt/(2m), x += v dt,
 * x += fnew dt^2/(2m), wrap/reflect (integrator.py:31-51, 98-128); fnew is
 * not copied to fold (swapped buffers). */
int mdg_host_kick_drift_range(int64_t n, int64_t begin, int64_t end, int layout, double* pos,
                              double* vel, double* fnew, const double* fold,
                              const int32_t* type_id, const double* mass, const double domain[3],
                              const int periodic[3], double dt, int has_gravity, double gravity,
                              int* blowup);

/* Measured FP64 FMA throughput of this device (roofline denominator):
 * dependent-chain DFMA microbenchmark, TFLOP/s (2 flops per DFMA). */
int mdg_measure_fp64_peak(mdg_ctx* ctx, double* tflops, double* sm_mhz_hint);

#ifdef __cplusplus
}
#endif

#endif /* MDG_H */
