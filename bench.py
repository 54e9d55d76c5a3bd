"""Benchmark of the LJ force + neighbour path on the BASELINE configurations.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mdg|reference]
                    [--workload config2|config3|config4|config5] [--config ID]
                    [--tune none|predictive|fullsearch]

N = 1 (default): BASELINE.json configs[1] (the configuration the metric is
quoted on): 1,048,576 LJ particles, uniform random at rho = 0.75 in a periodic
cube (side 111.82 sigma), overlaps relaxed by 50 capped steepest-descent
steps, Maxwell-Boltzmann T = 0.7, r_c = 2.5, skin 0.3, dt = 0.002, rebuild
every R+1 = 11 steps (reference cadence with R = 10), fp64, 1,000 steps.

N > 1 (torchrun, one rank per GPU): the north_star's decomposed
configuration 5 -- 67,108,864 particles on a jittered FCC lattice -- strong
scaled over a 2x1x1 / 2x2x1 / 2x2x2 process grid (configs 2-4 run as z-slabs
with --workload); ghost positions packed by libmdg and exchanged point to
point every step, migration every rebuild; ``--tune predictive`` gives every
rank its own reference TuningController fed by that rank's device timings.

A *step* is one full MD iteration of the reference loop (drift + boundaries,
rebuild when due, refresh, force, kick).  ``value`` = MUPS (particle updates
per second) of the whole system, state resident in HBM, time = max over
ranks; ``e2e`` (N = 1) = the same metric through the reference-facing host
drop-in (state in pinned host arrays, positions H2D and forces D2H every
step).  The L2 (126 MB) is flushed between timed steps by writing a 256 MB
buffer outside the timed events.

--impl reference times the reference algorithm on the host CPU (the oracle
port of the numba kernels, oracle/, all host threads) on the same workload
(a bounded sample of it for configs 4 and 5).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LJ force MUPS (particle-updates/s) at 1/2/4/8 B200; % of FP64/HBM roofline"
UNIT = "MUPS"
FLOPS_PER_PAIR = 26          # per unique within-cutoff pair
DEFAULT_CONFIG = "VL-List_Iter-NoN3L-SoA"
CPU_CONFIG = "LC-SLI-N3L-SoA-CSF1"   # fastest reference CPU configuration


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


WORKLOADS = {
    "config2": "config2: homogeneous LJ liquid, 1,048,576 particles, rho=0.75, SD-relaxed, T=0.7, "
               "rc=2.5, skin=0.3, dt=0.002, rebuild every 11 steps",
    "config3": "config3: FCC slab (rho=0.8) + vacuum, 2,097,152 particles, 128 x 128 x 640, "
               "T=2.0 + linear z ramp, rc=2.5, skin=0.3, dt=0.001, rebuild every 11 steps",
    "config4": "config4: LJ fluid at rho=0.4, 4,194,304 particles, SD-relaxed, equilibrated at "
               "T=1.4 then quenched to T=0.7 (droplets), rc=2.5, skin=0.3, dt=0.002",
    "config5": "config5: FCC 256^3 cells, 67,108,864 particles, rho=0.8, jittered, T=0.9, rc=2.5, "
               "skin=0.3, dt=0.002, rebuild every 11 steps",
}


DATA = {"config2": "uniform + 50 steepest-descent steps",
        "config3": "FCC slab sites + jitter",
        "config4": "uniform + steepest descent + T=1.4 equilibration + quench to T=0.7 on the device",
        "config5": "jittered FCC lattice"}


def default_workload(world):
    """N = 1: BASELINE configs[1] (the metric's single-GPU configuration);
    N > 1: the north_star's decomposed configuration 5, strong-scaled."""
    return "config2" if world == 1 else "config5"


def grid_dims(workload, world):
    """Process grid: config 5 as a 3-D grid (2x1x1, 2x2x1, 2x2x2 at 2/4/8),
    configs 2-4 as z-slabs."""
    if workload == "config5":
        table = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
        if world in table:
            return table[world]
        f = [1, 1, 1]
        n, q, k = world, 2, 0
        while n > 1:
            while n % q == 0:
                f[k % 3] *= q
                n //= q
                k += 1
            q += 1
        return tuple(f)
    return (1, 1, world)


def workload_config(args, n_gpus):
    out = {"workload": WORKLOADS[args.workload], "n_particles": args.n_total,
           "configuration": args.config}
    if n_gpus > 1:
        dims = grid_dims(args.workload, n_gpus)
        out.update({"decomposition": "x".join(str(d) for d in dims),
                    "parallelism": f"domain decomposition {'x'.join(str(d) for d in dims)} over "
                                   f"{n_gpus} GPUs (one rank per GPU): ghost positions packed by libmdg "
                                   "and exchanged point to point every step, migration at rebuilds, "
                                   "strong scaling (the whole system fixed)",
                    "tuning": args.tune})
    else:
        out["parallelism"] = "single"
        out["cell_reorder"] = (f"particle arrays permuted to the Verlet grid's cell order every "
                               f"{args.reorder} rebuild(s), inside the timed steps; caller order "
                               "restored by the final flush" if args.reorder else "off")
    out["l2"] = "flushed between timed steps (256 MB write, untimed)"
    return out


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every millisecond
    during the timed region through NVML (the counters nvidia-smi reports;
    one nvidia-smi call takes longer than a short timed region).  NVML is
    initialised before the timed region starts, so the first sample lands at
    its start; the main thread waits in CUDA calls (GIL released)."""

    def __init__(self, gpu_index, period_s=0.001):
        self.idx = gpu_index
        self.period = period_s
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._nv = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                          "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                          "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                          "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                          "hw_power_brake": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
            self._nv = nv
        except Exception as exc:   # no NVML: record why instead of failing the bench
            self.error = f"{type(exc).__name__}: {exc}"
            return

        def run():
            nv, h = self._nv, self._h
            try:
                while not self._stop.is_set():
                    mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((mhz, [k for k, b in self._bits.items() if rs & b]))
                    self._stop.wait(self.period)
            except Exception as exc:
                self.error = f"{type(exc).__name__}: {exc}"
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [r[0] for r in self.rows]
        reasons = sorted({x for r in self.rows for x in r[1]})
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": reasons,
               "samples": len(self.rows), "source": "NVML, 1 ms period, timed region only"}
        if getattr(self, "error", None):
            out["error"] = self.error
        return out


# --------------------------------------------------------------------- GPU arm

def global_inputs(args, on_device=True):
    """Seeded inputs of the workload as numpy (pos, vel, params); configs 2 and
    4 are relaxed (and 4 quenched) on the current GPU."""
    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200 import systems
    w = args.workload
    if w == "config2":
        pos, vel, params = systems.config2_inputs(n=args.n, seed=args.seed)
        parts = P.ParticleSet(pos, vel)
        systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
        return parts.numpy("pos"), parts.numpy("vel"), params
    if w == "config3":
        return systems.config3_inputs()
    if w == "config4":
        return systems.config4_state(equil_steps=args.quench // 2, quench_steps=args.quench)
    return systems.config5_inputs(n_side=args.n5_side)


def build_system(args, rank):
    import paper_2505_03438_b200 as P
    pos, vel, params = global_inputs(args)
    args.n_total = len(pos)
    return P.ParticleSet(pos, vel), params


def build_decomposed(args, rank, world, cfg, dist):
    """N > 1: the whole system of the workload, strong-scaled over a process
    grid (grid_dims).  Configs 3 and 5 are generated identically by every rank
    (seeded numpy); configs 2 and 4 are relaxed / quenched on rank 0's GPU and
    broadcast.  Each rank keeps the particles of its subdomain."""
    import torch

    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200.decomp import DeviceDecomposedSimulation, GridDecomposition
    dev = torch.device("cuda", torch.cuda.current_device())
    if args.workload in ("config2", "config4"):
        cd = "cpu" if args.dist_backend == "gloo" else dev
        if rank == 0:
            pos, vel, params = global_inputs(args)
            meta = torch.tensor([len(pos), *params.domain_size], dtype=torch.float64)
        else:
            meta = torch.zeros(4, dtype=torch.float64)
        meta = meta.to(cd)
        dist.broadcast(meta, 0)
        n = int(meta[0].item())
        buf = (torch.as_tensor(np.concatenate([pos, vel], 1)) if rank == 0
               else torch.empty((n, 6), dtype=torch.float64)).to(cd)
        dist.broadcast(buf, 0)
        buf = buf.cpu().numpy()
        pos, vel = buf[:, :3], buf[:, 3:]
        # configs 2 and 4 share their parameters (systems.config2_inputs /
        # config4_inputs); the box is rank 0's
        params = P.SimulationParams(domain_size=meta[1:].cpu().numpy().astype(np.float64), cutoff=2.5,
                                    skin=0.3, rebuild_interval=10, delta_t=2e-3,
                                    boundary=(P.PERIODIC,) * 3)
    else:
        pos, vel, params = global_inputs(args)
    args.n_total = len(pos)
    dims = grid_dims(args.workload, world)
    dec = GridDecomposition(params, rank, world, dims)
    mine = np.flatnonzero(dec.owner_of_positions(pos) == rank)
    owned = P.ParticleSet(pos[mine], vel[mine], device=dev)
    ids = torch.as_tensor(mine, device=dev)
    controller = None
    if args.tune != "none":
        controller = _rank_controller(args, cfg)
    comm = "cpu" if args.dist_backend == "gloo" else None
    sim = DeviceDecomposedSimulation(dec, owned, params, cfg, ids=ids, comm_device=comm,
                                     controller=controller)
    if controller is not None:
        controller.stats_provider = lambda: sim.calc.live_stats(sim.ps)
    return sim, params


def _rank_controller(args, cfg):
    """One reference TuningController per rank, fed by this
    rank's device timings; needs the staged reference (baseline/_ref)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.append(ref)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mdg_numba_cache")
    from mdtune import tuning

    import paper_2505_03438_b200 as P
    strategy = {"predictive": tuning.PredictiveStrategy, "fullsearch": tuning.FullSearchStrategy}[args.tune]()
    total = args.warmup + args.steps
    return tuning.TuningController(P.enumerate_configurations(), strategy, samples_per_config=2,
                                   tuning_interval=max(70, total // 2), rebuild_interval=10,
                                   total_iterations=total)


def gpu_arm(args, rank, world, dist):
    import torch

    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200 import _lib
    from paper_2505_03438_b200.simulation import Simulation

    local = _env_int("LOCAL_RANK", 0) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = P.parse_configuration(args.config)
    if world > 1:
        sim, params = build_decomposed(args, rank, world, cfg, dist)
        host_pos = host_vel = None
    else:
        parts, params = build_system(args, rank)
        host_pos = parts.numpy("pos")
        host_vel = parts.numpy("vel")
        parts.convert_layout(cfg.layout)
        # kick of step s fused into the drift of step s+1 (bit-identical,
        # tests/test_gpu_parity.py::test_fused_kick_drift_loop_is_bit_identical)
        # the particle arrays kept in cell order (bit-identical forces,
        # tests/test_gpu_parity.py::test_cell_reorder_is_invisible)
        sim = Simulation(parts, params, cfg, fuse_kick_drift=True, reorder=args.reorder)
    calc = sim.calc

    fp64_peak = _measure_fp64_peak(calc)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    for _ in range(args.warmup):
        sim.step()
    sim.check()
    warm_extra = 0
    if hasattr(sim, "warm_reorder"):
        sim.warm_reorder()
        # on through the loop's next cell reorder, untimed: the first reorder
        # taken inside step() (the first to compose permutations and to hand
        # the spare arrays back) stalled the host for 3-14 ms in ~10% of the
        # runs during some periods on the GPU pool -- always that one, never a
        # later reorder (profiles/round2_reorder_spike.txt)
        if (args.reorder and dist is None and cfg.container == P.VERLET_LISTS
                and not os.environ.get("MDG_BENCH_NO_WARM_EXTRA")):   # (the probe's way back to the stall)
            # (the reorder falls on the rebuild `reorder` rebuild intervals after this
            # point; one more interval brings the loop back to a rebuild step, so the
            # timed steps start on a rebuild as they always did)
            warm_extra = (args.reorder + 1) * (params.rebuild_interval + 1)
            for _ in range(warm_extra):
                sim.step()
            sim.check()
    torch.cuda.synchronize()

    clocks = ClockSampler(local, period_s=float(os.environ.get("MDG_BENCH_CLOCK_PERIOD", "0.001")))
    clocks.start()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.lib().mdg_launch_count()
    calc.profile(True, reserve=args.steps + 16)   # its events created here, not in the loop
    # the per-step events too: created (first record) before the timed loop
    step_ms = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    for a, b in step_ms:
        a.record()
        b.record()
    torch.cuda.synchronize()
    gc.disable()   # no collector pause stalls the host's launches inside the timed steps
    dev_allocs0 = torch.cuda.memory_stats(dev).get("num_device_alloc", 0)
    if os.environ.get("MDG_BENCH_STEPS"):
        print("timed loop starts", file=sys.stderr, flush=True)
    host_ms = [] if os.environ.get("MDG_BENCH_STEPS") else None   # host time of each step() call
    for k in range(args.steps):
        flush.zero_()
        a, b = step_ms[k]
        a.record()
        t0 = time.perf_counter() if host_ms is not None else 0.0
        sim.step()
        if k == args.steps - 1:
            sim.flush()   # the last step's (deferred) kick inside the timed region
        b.record()
        if host_ms is not None:
            host_ms.append(round((time.perf_counter() - t0) * 1e3, 4))
    torch.cuda.synchronize()
    gc.enable()
    launches = _lib.lib().mdg_launch_count() - launches0
    kernel_ms, kernel_launches = calc.profile_read()
    calc.profile(False)
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in step_ms)
    if os.environ.get("MDG_BENCH_STEPS"):
        print(json.dumps([round(a.elapsed_time(b), 4) for a, b in step_ms]), file=sys.stderr)
        print("host_ms " + json.dumps(host_ms), file=sys.stderr)
        from paper_2505_03438_b200 import simulation as _simmod
        print("reorder steps (iteration, reorder, rebuild, refresh + compute host ms): " + json.dumps(_simmod.STEP_TRACE), file=sys.stderr)
        print("cudaMallocs by torch inside the timed loop: %d" % (torch.cuda.memory_stats(dev).get("num_device_alloc", 0) - dev_allocs0), file=sys.stderr)
    sim.check()

    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64,
                         device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # unique within-cutoff pairs of the last force evaluation (the roofline unit)
    count = calc.last_eval_count
    pairs = count if cfg.newton3 else count // 2
    if rank != 0:
        return None
    ms_per_step = total_ms / args.steps
    value = args.n_total * args.steps / (total_ms * 1e-3) / 1e6
    avg_kernel_ms = kernel_ms / max(kernel_launches, 1)
    achieved = FLOPS_PER_PAIR * pairs / (avg_kernel_ms * 1e-3) / 1e12
    roofline = {"bound": "fp64", "achieved": round(achieved, 3), "peak": round(fp64_peak, 2),
                "unit": "TFLOP/s", "frac": round(achieved / fp64_peak, 4),
                "traffic": _ncu_traffic(args.config),
                "peak_source": "measured on-box DFMA microbenchmark (mdg_measure_fp64_peak); "
                               "MEASURED_PEAKS.json has no fp64 figure",
                "kernel": "force traversal kernels of " + args.config,
                "kernel_ms_avg": round(avg_kernel_ms, 4), "kernel_launches": kernel_launches,
                "unique_pairs": pairs, "flops_per_pair": FLOPS_PER_PAIR,
                "kernel_share_of_step": round(kernel_ms / total_ms, 3)}
    out = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
           "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": f"synthetic, seeded ({args.workload}: {DATA[args.workload]})",
           "config": workload_config(args, world), "roofline": roofline,
           "pair_interactions_per_s": round(pairs / (avg_kernel_ms * 1e-3), 1),
           "gpu_launches": int(launches), "clocks": clk}
    if warm_extra:
        out["config"]["warmup_extra"] = (f"{warm_extra} further untimed steps after the {args.warmup} warm-up steps take the "
                                         "loop through its next cell reorder (one-time first-use costs); the "
                                         "timed steps keep the reorder cadence")
    if world == 1 and not args.no_e2e and args.workload == "config2":
        out["e2e"] = e2e_arm(args, host_pos, host_vel, params)
    if world == 1 and not args.no_cpu and args.workload == "config2":
        out["cpu_baseline"] = cpu_baseline(args, host_pos, host_vel, params)
    if world > 1:
        out["e2e"] = None
        out["e2e_note"] = ("the host-array drop-in path (HostForceCalculator, mdg_host_run) is a "
                           "single-process API; N > 1 runs keep the state resident on each rank")
        out["comm"] = comm_info(args, world)
        if args.workload == "config5":
            out["strong_scaling_baseline"] = (
                "the same system on one GPU: bench.py --workload config5 (one GPU holds all "
                "67,108,864 particles); the default N = 1 line is config 2, BASELINE's single-GPU "
                "configuration, so per-N values of the default runs do not form one strong-scaling series")
        if args.tune != "none":
            out["tuning_trials"] = len(sim.trial_log)
            out["phase_selections"] = list(getattr(sim.controller, "phase_selections", []))
    return out


def comm_info(args, world):
    """The communicator the decomposed run used (NCCL version, ranks, process
    grid), so the line shows the multi-rank data path that ran."""
    import torch
    info = {"backend": args.dist_backend, "ranks": world,
            "process_grid": "x".join(str(d) for d in grid_dims(args.workload, world))}
    try:
        v = torch.cuda.nccl.version()
        info["nccl_version"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    except Exception as exc:   # pragma: no cover
        info["nccl_version"] = f"unavailable: {exc}"
    return info


def _measure_fp64_peak(calc):
    import ctypes

    from paper_2505_03438_b200 import _lib
    t, mhz = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib().mdg_measure_fp64_peak(calc.ctx.h, ctypes.byref(t), ctypes.byref(mhz)))
    return float(t.value)


def _ncu_traffic(config_id):
    """DRAM bytes per force launch from the committed `ncu --set full` capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            doc = json.load(fh)
        return doc.get(config_id)
    except (OSError, ValueError):
        return None


def e2e_arm(args, host_pos, host_vel, params):
    """The reference-facing drop-in end to end: state in (pinned) host memory,
    the reference loop order (simulation.py:150-188) with HostForceCalculator as
    the force backend -- positions H2D and forces D2H every step -- and the
    host-side Verlet update in libmdg's native integrator."""
    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200.hostloop import HostParticleSet, HostSimulation
    cfg = P.parse_configuration(args.config)
    steps = min(args.steps, 1000)
    p = HostParticleSet(host_pos, host_vel)
    sim = HostSimulation(p, params, cfg)
    sim.run(2)                      # allocations + first rebuild outside the timed region
    n = len(host_pos)
    # three timed windows of `steps` steps on one trajectory, the median
    # reported (the host-memory-bound loop varies run to run)
    runs = []
    for _ in range(3):
        t0 = time.perf_counter()
        sim.run(steps)
        runs.append(n * steps / (time.perf_counter() - t0) / 1e6)
    h2d = 24 * n   # positions once per step (rebuilds reuse the uploaded copy)
    return {"value": round(statistics.median(runs), 3), "unit": UNIT, "steps": steps,
            "windows": [round(r, 1) for r in runs],
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 24 * n,
            "path": "hostloop.HostSimulation.run: pinned host state, reference loop order, "
                    "H2D positions and D2H forces every step in 16 chunks, native host kick+drift "
                    "per chunk as its forces land (mdg_host_run)"}


def _cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(args, host_pos, host_vel, params):
    """Oracle port (the reference's algorithm restated in C + numpy) on the
    host cores, on a bounded sample of the same workload: one rebuild, two
    refresh+force evaluations and one integrator pass on the relaxed snapshot;
    MUPS = N / (force + refresh + integrator + rebuild/(R+1))."""
    from oracle import port
    cfg = port.parse(CPU_CONFIG)
    threads = _cpu_threads()
    per = tuple(port.PERIODIC if f else port.REFLECTIVE for f in params.periodic_flags())
    pp = port.Params(domain_size=params.domain_size, cutoff=params.cutoff, skin=params.skin,
                     rebuild_interval=params.rebuild_interval, delta_t=params.delta_t,
                     boundary=per, thread_count=threads)
    p = port.Particles(host_pos, host_vel)
    p.convert_layout(cfg.layout)
    calc = port.ForceCalculator(p, pp)
    with port.Pool(threads) as pool:
        t0 = time.perf_counter()
        calc.rebuild(p, cfg)
        t1 = time.perf_counter()
        tf, tr = [], []
        for _ in range(2):
            a = time.perf_counter()
            calc.refresh(p, cfg)
            b = time.perf_counter()
            calc.compute(p, cfg, pool)
            c = time.perf_counter()
            tr.append(b - a)
            tf.append(c - b)
        a = time.perf_counter()
        port.drift_with_force(p, pp.delta_t)
        port.apply_boundaries(p, pp)
        np.copyto(p.view("old_force"), p.view("force"))
        port.finish_kick(p, pp.delta_t)
        ti = time.perf_counter() - a
        step = min(tf) + min(tr) + ti + (t1 - t0) / (params.rebuild_interval + 1)
        # the GPU arm's own configuration on the same snapshot (like-for-like)
        same = port.parse(args.config)
        p.convert_layout(same.layout)
        s0 = time.perf_counter()
        calc.rebuild(p, same)
        s1 = time.perf_counter()
        calc.refresh(p, same)
        b = time.perf_counter()
        calc.compute(p, same, pool)
        tfs = time.perf_counter() - b
    step_same = tfs + ti + (s1 - s0) / (params.rebuild_interval + 1)
    return {"value": round(len(host_pos) / step / 1e6, 4), "unit": UNIT, "cores": threads,
            "kind": "port", "config": CPU_CONFIG,
            "sample": f"1 rebuild + 2 refresh/force + 1 integrator pass on the relaxed {len(host_pos):,}-"
                      f"particle snapshot the GPU arm starts from ({threads} threads; rebuild amortised "
                      "over 11 steps); the fastest reference CPU configuration",
            "force_s": round(min(tf), 4), "rebuild_s": round(t1 - t0, 4),
            "integrator_s": round(ti, 4),
            "same_config": {"configuration": args.config, "value": round(len(host_pos) / step_same / 1e6, 4),
                            "force_s": round(tfs, 4), "rebuild_s": round(s1 - s0, 4),
                            "sample": "the GPU arm's configuration on the same snapshot: 1 rebuild + "
                                      "1 force + the integrator pass"}}


# --------------------------------------------------------------- reference arm

def reference_arm(args):
    """The reference algorithm on the host CPU (oracle port, all threads) on the
    same workload; each timed step is one full reference-loop MD step."""
    from oracle import port

    from paper_2505_03438_b200 import systems
    threads = _cpu_threads()
    cfg = port.parse(CPU_CONFIG)
    w = args.workload
    relax = w in ("config2", "config4")
    if w == "config2":
        pos, vel, params = systems.config2_inputs(n=args.n, seed=args.seed)
        what = f"the {len(pos):,}-particle config-2 system"
    elif w == "config3":
        pos, vel, params = systems.config3_inputs()
        what = "the 2,097,152-particle config-3 slab"
    elif w == "config4":   # bounded sample: a 1/16 box at the same density (relaxed, not quenched)
        pos, vel, params = systems.config4_inputs(n=262_144)
        what = "a 262,144-particle box at config 4's density (rho = 0.4; relaxed, not quenched)"
    else:                  # bounded sample: a 64^3-cell block of the same lattice, density and T
        pos, vel, params = systems.config5_inputs(n_side=64)
        what = "a 64^3-cell (1,048,576-particle) periodic block of config 5's FCC lattice (rho = 0.8, T = 0.9)"
    per = tuple(port.PERIODIC if f else port.REFLECTIVE for f in params.periodic_flags())
    pp = port.Params(domain_size=params.domain_size, cutoff=params.cutoff, skin=params.skin,
                     rebuild_interval=params.rebuild_interval, delta_t=params.delta_t,
                     boundary=per, thread_count=threads)
    p = port.Particles(pos, vel)
    n = len(pos)
    with port.Pool(threads) as pool:
        if relax:
            port.sd_relax(p, pp, cfg, systems.SD_STEPS, systems.SD_GAMMA, systems.SD_MAX_DISP, pool)
        snap = (np.array(p.positions), np.array(p.velocities))
        steps = max(1, min(args.steps, 11))
        warm = max(0, min(args.warmup, 1))
        port.simulate_fixed(p, pp, cfg, steps=warm, pool=pool)
        t0 = time.perf_counter()
        port.simulate_fixed(p, pp, cfg, steps=steps, pool=pool)
        dt = time.perf_counter() - t0
    value = n * steps / dt / 1e6
    sample = (f"{steps} full MD steps (one rebuild window of 11) of {what} after {warm} warm-up "
              f"step(s); {threads} host threads; {CPU_CONFIG}")
    extra = {}
    if os.environ.get("MDG_REF_NUMBA", "1") != "0":
        extra["reference_mdtune"] = _time_mdtune(snap, params, steps, threads)
    return {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "impl": "reference",
            "n_gpus": 1, "steps": steps, "warmup": warm, "ms_per_step": round(dt / steps * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic, seeded ({w}: {DATA[w]})",
            "config": {"workload": WORKLOADS[w], "n_particles": n, "sample": what,
                       "configuration": CPU_CONFIG, "parallelism": f"{threads} CPU threads"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}, **extra}


def _time_mdtune(snap, params, steps, threads):
    """The unmodified reference itself (mdtune's simulate with numba kernels,
    staged under baseline/_ref) on the same relaxed snapshot and configuration,
    next to the oracle port's number; skipped when the package is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mdtune")):
        return {"unavailable": "reference not staged under baseline/_ref"}
    if ref not in sys.path:
        sys.path.append(ref)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mdg_numba_cache")
    try:
        from mdtune.configuration import parse_configuration
        from mdtune.params import PERIODIC, SimulationParams
        from mdtune.particles import ParticleSet
        from mdtune.simulation import simulate
        from mdtune.tuning import FixedStrategy

        def run(k):
            prm = SimulationParams(domain_size=tuple(params.domain_size), cutoff=params.cutoff,
                                   skin=params.skin, rebuild_interval=params.rebuild_interval,
                                   delta_t=params.delta_t, total_iterations=k, boundary=(PERIODIC,) * 3,
                                   thread_count=threads)
            ps = ParticleSet(snap[0].copy(), velocities=snap[1].copy())
            t0 = time.perf_counter()
            rep = simulate(ps, prm, FixedStrategy(parse_configuration(CPU_CONFIG)), tuning_interval=10 ** 9,
                           raise_errors=True)
            return time.perf_counter() - t0, rep
        run(1)                       # numba JIT / cache load outside the timing
        dt, _ = run(steps)
        import numba
        return {"value": round(len(snap[0]) * steps / dt / 1e6, 4), "unit": UNIT, "steps": steps,
                "configuration": CPU_CONFIG, "threads": threads, "numba": numba.__version__,
                "sample": f"{steps} steps of mdtune.simulation.simulate (FixedStrategy) on the same snapshot"}
    except Exception as exc:   # informational only: the port's number is the line's value
        return {"unavailable": f"{type(exc).__name__}: {exc}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=11)
    ap.add_argument("--impl", default="mdg", choices=("mdg", "reference"))
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--particles", "--n", dest="n", type=int, default=1_048_576,
                    help="config 2 particle count")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None,
                    help="BASELINE configuration (default: config2 at N=1, config5 at N>1)")
    ap.add_argument("--n5-side", type=int, default=256, help="config 5 FCC cells per axis")
    ap.add_argument("--quench", type=int, default=2000,
                    help="config 4: quench steps at T=0.7 (after half as many at T=1.4)")
    ap.add_argument("--tune", choices=("none", "predictive", "fullsearch"), default="none",
                    help="N>1: one reference TuningController per rank (needs baseline/_ref)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--reorder", type=int, default=_env_int("MDG_BENCH_REORDER", 16),
                    help="permute the particle arrays to cell order every K-th rebuild (0 = off)")
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"),
                    help="gloo (messages staged on the host) only to smoke-test the N > 1 path "
                         "with several ranks on one GPU; never a performance number")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "mdg":
        args.warmup = 3
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    if args.workload is None:
        args.workload = default_workload(world)
    args.n_total = args.n

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(reference_arm(args)), flush=True)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(_env_int("LOCAL_RANK", 0) % max(1, torch.cuda.device_count()))
        tdist.init_process_group(args.dist_backend)
        dist = tdist
    out = gpu_arm(args, rank, world, dist)
    if out is not None:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
