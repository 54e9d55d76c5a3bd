"""Benchmark of the LJ force + neighbour path on BASELINE config 2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mdg|reference]
                    [--config ID] [--n N]

Workload (BASELINE.json configs[1], the configuration the metric is quoted
on): 1,048,576 LJ particles, uniform random at rho = 0.75 in a periodic cube
(side 111.82 sigma), overlaps relaxed by 50 capped steepest-descent steps,
Maxwell-Boltzmann T = 0.7, r_c = 2.5, skin 0.3, dt = 0.002, rebuild every
R+1 = 11 steps (reference cadence with R = 10), fp64.  Seeded synthetic data.

A *step* is one full MD iteration of the reference loop (drift + boundaries,
rebuild when due, refresh, force, kick).  ``value`` = MUPS (particle updates
per second) over all ranks with state resident in HBM; ``e2e`` = the same
metric through the reference-facing host drop-in (HostForceCalculator driving
the reference-shaped simulate loop on host numpy arrays, positions H2D and
forces D2H every step).  The L2 (126 MB) is flushed between timed steps by
writing a 256 MB buffer outside the timed events.

--impl reference times the reference algorithm on the host CPU (the oracle
port of the numba kernels, oracle/, all host threads) on the same workload.
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


def workload_config(args, n_gpus):
    if n_gpus > 1:
        return {"workload": f"config2 boxes stacked along z: {n_gpus} x {args.n:,} particles in one "
                            f"periodic box L x L x {n_gpus}L (rho=0.75, SD-relaxed, T=0.7, rc=2.5, "
                            "skin=0.3, dt=0.002, rebuild every 11 steps)",
                "n_particles": args.n * n_gpus, "n_particles_per_gpu": args.n,
                "configuration": args.config,
                "parallelism": f"zslab{n_gpus}: domain decomposition, ghost positions over NCCL "
                               "every step, migration at rebuilds",
                "l2": "flushed between timed steps (256 MB write, untimed)"}
    return {"workload": "config2: homogeneous LJ liquid, 1,048,576 particles, rho=0.75, "
                        "SD-relaxed, T=0.7, rc=2.5, skin=0.3, dt=0.002, rebuild every 11 steps",
            "n_particles": args.n, "configuration": args.config, "parallelism": "single",
            "cell_reorder": (f"particle arrays permuted to the Verlet grid's cell order every "
                             f"{args.reorder} rebuild(s), inside the timed steps; caller order "
                             "restored by the final flush" if args.reorder else "off"),
            "l2": "flushed between timed steps (256 MB write, untimed)"}


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every few ms during the
    timed region through NVML (the same counters nvidia-smi reports; one
    nvidia-smi call takes longer than the whole timed region)."""

    def __init__(self, gpu_index, period_s=0.005):
        self.idx = gpu_index
        self.period = period_s
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            try:
                import pynvml as nv
                nv.nvmlInit()
                h = nv.nvmlDeviceGetHandleByIndex(self.idx)
                self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                        "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                        "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                        "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                        "hw_power_brake": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
                while not self._stop.is_set():
                    mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((mhz, [k for k, b in bits.items() if rs & b]))
                    self._stop.wait(self.period)
            except Exception as exc:   # no NVML: record why instead of failing the bench
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
               "samples": len(self.rows), "source": "NVML, 5 ms period, timed region only"}
        if getattr(self, "error", None):
            out["error"] = self.error
        return out


# --------------------------------------------------------------------- GPU arm

def build_system(args, rank):
    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200 import systems
    pos, vel, params = systems.config2_inputs(n=args.n, seed=args.seed + rank)
    parts = P.ParticleSet(pos, vel)
    relax_cfg = P.parse_configuration("LC-SLI-N3L-AoS-CSF1")
    systems.relax_on_device(parts, params, relax_cfg)
    return parts, params


def build_decomposed(args, rank, world, cfg):
    """N > 1: one config-2 box per rank, stacked along z into one periodic
    system of N x n particles, z-slab decomposed.  Every rank
    relaxes the same seeded box, so the interfaces between slabs are as
    relaxed as the box's own periodic faces; velocities are drawn per rank."""
    import numpy as np
    import torch

    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200.decomp import DeviceDecomposedSimulation, GridDecomposition
    parts, params = build_system(args, 0)
    L = np.asarray(params.domain_size, dtype=np.float64)
    rng = np.random.default_rng(args.seed + 7919 * (rank + 1))
    vel = rng.normal(0.0, np.sqrt(0.7), (args.n, 3))
    vel -= vel.mean(0)
    pos = parts.view("pos").clone()
    pos[:, 2] += rank * L[2]
    gparams = P.SimulationParams(domain_size=(L[0], L[1], world * L[2]), cutoff=params.cutoff,
                                 skin=params.skin, rebuild_interval=params.rebuild_interval,
                                 delta_t=params.delta_t, boundary=params.boundary)
    dec = GridDecomposition(gparams, rank, world, (1, 1, world))
    owned = P.ParticleSet(pos, torch.as_tensor(vel), device=parts.device)
    ids = torch.arange(args.n, device=parts.device) + rank * args.n
    comm = "cpu" if args.dist_backend == "gloo" else None
    return DeviceDecomposedSimulation(dec, owned, gparams, cfg, ids=ids, comm_device=comm), gparams


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
        sim, params = build_decomposed(args, rank, world, cfg)
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
    if hasattr(sim, "warm_reorder"):
        sim.warm_reorder()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.lib().mdg_launch_count()
    calc.profile(True)
    gc.disable()   # no collector pause stalls the host's launches inside the timed steps
    step_ms = []
    for k in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sim.step()
        if k == args.steps - 1:
            sim.flush()   # the last step's (deferred) kick inside the timed region
        b.record()
        step_ms.append((a, b))
    torch.cuda.synchronize()
    gc.enable()
    launches = _lib.lib().mdg_launch_count() - launches0
    kernel_ms, kernel_launches = calc.profile_read()
    calc.profile(False)
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in step_ms)
    if os.environ.get("MDG_BENCH_STEPS"):
        print(json.dumps([round(a.elapsed_time(b), 4) for a, b in step_ms]), file=sys.stderr)
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
    value = args.n * world * args.steps / (total_ms * 1e-3) / 1e6
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
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded uniform + steepest-descent relaxation, BASELINE config 2)",
           "config": workload_config(args, world), "roofline": roofline,
           "pair_interactions_per_s": round(pairs / (avg_kernel_ms * 1e-3), 1),
           "gpu_launches": int(launches), "clocks": clk}
    if world == 1 and not args.no_e2e:
        out["e2e"] = e2e_arm(args, host_pos, host_vel, params)
    if world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args, host_pos, host_vel, params)
    return out


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
    return {"value": round(len(host_pos) / step / 1e6, 4), "unit": UNIT, "cores": threads,
            "kind": "port", "config": CPU_CONFIG,
            "sample": f"1 rebuild + 2 refresh/force + 1 integrator pass on the relaxed {len(host_pos):,}-"
                      f"particle snapshot ({threads} threads; rebuild amortised over 11 steps)",
            "force_s": round(min(tf), 4), "rebuild_s": round(t1 - t0, 4),
            "integrator_s": round(ti, 4)}


# --------------------------------------------------------------- reference arm

def reference_arm(args):
    """The reference algorithm on the host CPU (oracle port, all threads) on the
    same workload; each timed step is one full reference-loop MD step."""
    from oracle import port

    from paper_2505_03438_b200 import systems
    threads = _cpu_threads()
    cfg = port.parse(CPU_CONFIG)
    pos, vel, params = systems.config2_inputs(n=args.n, seed=args.seed)
    per = tuple(port.PERIODIC if f else port.REFLECTIVE for f in params.periodic_flags())
    pp = port.Params(domain_size=params.domain_size, cutoff=params.cutoff, skin=params.skin,
                     rebuild_interval=params.rebuild_interval, delta_t=params.delta_t,
                     boundary=per, thread_count=threads)
    p = port.Particles(pos, vel)
    with port.Pool(threads) as pool:
        port.sd_relax(p, pp, cfg, systems.SD_STEPS, systems.SD_GAMMA, systems.SD_MAX_DISP, pool)
        steps = max(1, min(args.steps, 11))
        warm = max(0, min(args.warmup, 1))
        port.simulate_fixed(p, pp, cfg, steps=warm, pool=pool)
        t0 = time.perf_counter()
        port.simulate_fixed(p, pp, cfg, steps=steps, pool=pool)
        dt = time.perf_counter() - t0
    value = args.n * steps / dt / 1e6
    sample = (f"{steps} full MD steps (one rebuild window of 11) of the {args.n:,}-particle "
              f"system after {warm} warm-up step(s); {threads} host threads; {CPU_CONFIG}")
    return {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "impl": "reference",
            "n_gpus": 1, "steps": steps, "warmup": warm, "ms_per_step": round(dt / steps * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform + steepest-descent relaxation, BASELINE config 2)",
            "config": {"workload": "config2 (see GPU arm)", "n_particles": args.n,
                       "configuration": CPU_CONFIG, "parallelism": f"{threads} CPU threads"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=110)
    ap.add_argument("--warmup", type=int, default=11)
    ap.add_argument("--impl", default="mdg", choices=("mdg", "reference"))
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--particles", "--n", dest="n", type=int, default=1_048_576)
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
