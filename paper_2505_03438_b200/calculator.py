"""The force calculator on the GPU: the reference's drop-in boundary.

``ForceCalculator`` mirrors mdtune.containers.ForceCalculator
(containers.py:378-488) member for member -- ``rebuild``, ``refresh``,
``compute`` (returns the within-cutoff evaluation count), ``last_eval_count``
-- on a device-resident :class:`~paper_2505_03438_b200.particles.ParticleSet`.
Every call goes through libmdg's C ABI (include/mdg.h); there is no CPU path.

``HostForceCalculator`` is the same protocol over the reference's HOST
ParticleSet (numpy arrays): positions are copied host->device at rebuild /
refresh (and at compute for Verlet lists, which read positions directly,
containers.py:435-436), forces device->host after compute.  It is what gets
installed into ``mdtune.simulation.ForceCalculator`` /
``mdtune.dataset.ForceCalculator`` (see plugin.py) so the reference's own
simulate loop and tuning strategies drive the GPU unchanged.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import FLAG_BLOWUP, check, config_struct, lib


@dataclass
class Timings:
    force_ns: int = 0
    build_ns: int = 0


def _dptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class Context:
    """Owns one mdg_ctx on a CUDA device, enqueuing on torch's current stream."""

    def __init__(self, device=None, stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2505_03438_b200 needs a CUDA device (no CPU fallback)")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        self.stream = stream or torch.cuda.current_stream(idx)
        h = ctypes.c_void_p()
        check(lib().mdg_create(idx, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)),
              "mdg_create")
        self.h = h

    def set_system(self, params, sigma, epsilon, mass):
        L = np.ascontiguousarray(params.domain_size, dtype=np.float64)
        per = np.ascontiguousarray(params.periodic_flags().astype(np.int32))
        sig = np.ascontiguousarray(sigma, dtype=np.float64)
        eps = np.ascontiguousarray(epsilon, dtype=np.float64)
        m = np.ascontiguousarray(mass, dtype=np.float64)
        check(lib().mdg_set_system(self.h, L.ctypes.data, per.ctypes.data, float(params.cutoff),
                                   float(params.skin), len(sig), sig.ctypes.data,
                                   eps.ctypes.data, m.ctypes.data), "mdg_set_system")

    def bind(self, n, layout, pos, vel, force, old_force, type_id):
        check(lib().mdg_bind(self.h, int(n), _lib.AOS if layout == "AoS" else _lib.SOA,
                             _dptr(pos), _dptr(vel), _dptr(force), _dptr(old_force),
                             _dptr(type_id)), "mdg_bind")

    def eval_count(self) -> int:
        c = ctypes.c_int64()
        check(lib().mdg_eval_count(self.h, ctypes.byref(c)), "mdg_eval_count")
        return int(c.value)

    def close(self):
        if getattr(self, "h", None):
            lib().mdg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ForceCalculator:
    """Force evaluation under any enumerated configuration, on the GPU."""

    def __init__(self, particles, params):
        self.params = params
        self.ctx = Context(particles.device)
        self.ctx.set_system(params, particles.sigma, particles.epsilon, particles.mass)
        self._count_pending = False
        self._count = 0

    # -- binding -------------------------------------------------------------
    def bind(self, p):
        self._bound_n = p.n
        self.ctx.bind(p.n, p.layout, p.pos, p.vel, p.force, p.old_force,
                      p.type_id if p.ntypes > 1 else None)

    # -- the reference protocol ---------------------------------------------
    # bumped by every call that may rebuild a container (Simulation's cell
    # reorder checks it: a grid rebuilt on other indexing invalidates its order)
    generation = 0

    def rebuild(self, particles, config):
        self.generation += 1
        self.bind(particles)
        check(lib().mdg_rebuild(self.ctx.h, ctypes.byref(config_struct(config))), "rebuild")

    def rebuild_checked(self, particles, config) -> int:
        """rebuild() with the loop's status check folded into the rebuild's
        own host synchronisation (mdg_rebuild_checked): returns the status
        bits (then reset); nonzero means the rebuild was abandoned."""
        self.generation += 1
        self.bind(particles)
        f = ctypes.c_int()
        check(lib().mdg_rebuild_checked(self.ctx.h, ctypes.byref(config_struct(config)),
                                        ctypes.byref(f)), "rebuild")
        return int(f.value)

    def owned_order(self, config, out=None, tmp=None):
        """Device int64 tensor: the particles in the row (cell) order of the
        container of `config` as of its last rebuild (mdg_owned_order).
        ``out`` (int64) / ``tmp`` (int32), n elements each, are used when given:
        a caller inside a timed loop passes its own buffers, because a fresh
        block from the caching allocator can mean a cudaMalloc (milliseconds)."""
        n = self._bound_n
        dev = self.ctx.device
        if tmp is None or tmp.numel() != n or tmp.dtype != torch.int32 or tmp.device != dev:
            tmp = torch.empty(n, dtype=torch.int32, device=dev)
        check(lib().mdg_owned_order(self.ctx.h, ctypes.byref(config_struct(config)), tmp.data_ptr()),
              "owned_order")
        if out is None or out.numel() != n or out.dtype != torch.int64 or out.device != dev:
            out = torch.empty(n, dtype=torch.int64, device=dev)
        self.permutation(2, tmp, None, out)   # widened in libmdg, not by an eager torch cast
        return out

    def permutation(self, op, a, b, out):
        """mdg_permutation on device tensors: op 0 out = a[b], 1 out[a] =
        arange, 2 out = int64(a) (a int32)."""
        check(lib().mdg_permutation(self.ctx.h, int(op), int(out.numel()), ctypes.c_void_p(a.data_ptr()),
                                    ctypes.c_void_p(b.data_ptr() if b is not None else 0),
                                    ctypes.c_void_p(out.data_ptr())), "permutation")

    def refresh(self, particles, config):
        self.bind(particles)
        check(lib().mdg_refresh(self.ctx.h, ctypes.byref(config_struct(config))), "refresh")

    def compute_async(self, particles, config):
        """compute() without the host synchronisation for the count."""
        if particles.layout != config.layout:
            raise ValueError(f"particle layout {particles.layout} does not match "
                             f"configuration {config.id}")
        self.bind(particles)
        check(lib().mdg_compute(self.ctx.h, ctypes.byref(config_struct(config))), "compute")
        self._count_pending = True

    def compute(self, particles, config, workforce=None) -> int:
        self.compute_async(particles, config)
        return self.last_eval_count

    def step_graph(self, particles, config, dt, gravity=None):
        """One steady-state iteration (drift + refresh + compute + kick) from
        a cached CUDA graph (mdg_step_graph); asynchronous."""
        if particles.layout != config.layout:
            raise ValueError(f"particle layout {particles.layout} does not match "
                             f"configuration {config.id}")
        self.bind(particles)
        check(lib().mdg_step_graph(self.ctx.h, ctypes.byref(config_struct(config)), float(dt),
                                   int(gravity is not None), float(gravity or 0.0)), "step_graph")
        self._count_pending = True

    def compute_kick_async(self, particles, config, dt, gravity=None):
        """compute + apply_gravity + finish_kick (simulation.py:169-185), the
        kick fused into the force walk where the configuration allows."""
        if particles.layout != config.layout:
            raise ValueError(f"particle layout {particles.layout} does not match "
                             f"configuration {config.id}")
        self.bind(particles)
        check(lib().mdg_compute_kick(self.ctx.h, ctypes.byref(config_struct(config)), float(dt),
                                     int(gravity is not None), float(gravity or 0.0)), "compute_kick")
        self._count_pending = True

    @property
    def last_eval_count(self) -> int:
        if self._count_pending:
            self._count = self.ctx.eval_count()
            self._count_pending = False
        return self._count

    # -- integrator on the bound arrays (integrator.py) ------------------------
    def drift_wrap(self, particles, dt):
        self.bind(particles)
        check(lib().mdg_drift_wrap(self.ctx.h, float(dt)), "drift")

    def finish_kick(self, particles, dt, gravity=None):
        self.bind(particles)
        check(lib().mdg_finish_kick(self.ctx.h, float(dt), int(gravity is not None),
                                    float(gravity or 0.0)), "finish_kick")

    def kick_drift(self, particles, dt, gravity=None, copy_old_force=True):
        """finish_kick of the previous step + this step's drift_wrap in one
        pass (mdg_kick_drift); with ``copy_old_force=False`` the caller swaps
        ``particles.force`` / ``old_force`` afterwards."""
        self.bind(particles)
        check(lib().mdg_kick_drift(self.ctx.h, float(dt), int(gravity is not None),
                                   float(gravity or 0.0), int(bool(copy_old_force))), "kick_drift")

    def run_fixed(self, particles, config, steps, dt, gravity, rebuild_interval, iteration0,
                  since, kick_due, rebuild_now=False):
        """mdg_run: `steps` iterations of the fixed-configuration loop in one
        native call (see include/mdg.h).  Swaps ``particles.force`` /
        ``old_force`` as the native loop did.  Returns (done, since, kick_due,
        flags)."""
        if particles.layout != config.layout:
            raise ValueError(f"particle layout {particles.layout} does not match "
                             f"configuration {config.id}")
        self.bind(particles)
        s, kd, sw, fl = ctypes.c_int(int(since)), ctypes.c_int(int(bool(kick_due))), ctypes.c_int(0), ctypes.c_int(0)
        done = ctypes.c_int64(0)
        rc = lib().mdg_run(self.ctx.h, ctypes.byref(config_struct(config)), int(steps), float(dt),
                           int(gravity is not None), float(gravity or 0.0), int(rebuild_interval),
                           int(iteration0), int(bool(rebuild_now)), ctypes.byref(s), ctypes.byref(kd),
                           ctypes.byref(sw), ctypes.byref(done), ctypes.byref(fl))
        if sw.value & 1:
            particles.force, particles.old_force = particles.old_force, particles.force
        if done.value:
            if rebuild_now or s.value < int(since) + done.value:   # the loop rebuilt the container
                self.generation += 1
            self._count_pending = True
        check(rc, "run")
        return int(done.value), int(s.value), bool(kd.value), int(fl.value)

    def set_force_rows(self, n_force=None):
        """mdg_set_force_rows: only rows of particles [0, n_force) get force
        work in the tiled Verlet walk (None: every row)."""
        check(lib().mdg_set_force_rows(self.ctx.h, -1 if n_force is None else int(n_force)),
              "set_force_rows")

    def ghost_pack(self, particles, idx, n_left, axis, shift_left, shift_right, out):
        """mdg_ghost_pack: rows ``idx`` (int64 device tensor) of the bound
        positions into the AoS ``out`` (len(idx), 3), shifted along ``axis``
        by ``shift_left`` for the first ``n_left`` rows, ``shift_right`` after."""
        self.bind(particles)
        n = int(idx.numel())
        check(lib().mdg_ghost_pack(self.ctx.h, ctypes.c_void_p(idx.data_ptr()), int(n_left),
                                   int(n - n_left), int(axis), float(shift_left), float(shift_right),
                                   ctypes.c_void_p(out.data_ptr())), "ghost_pack")

    def ghost_unpack(self, particles, buf, row0):
        """mdg_ghost_unpack: the AoS (k, 3) ``buf`` into bound rows [row0, row0+k)."""
        self.bind(particles)
        check(lib().mdg_ghost_unpack(self.ctx.h, ctypes.c_void_p(buf.data_ptr()), int(buf.shape[0]),
                                     int(row0)), "ghost_unpack")

    def lc_pairs(self, csf):
        """The LC pair set (mdg_lc_pairs) of the last LC rebuild at `csf`: the
        (k, 2) sorted unique owner pairs (i < j) with r^2 < rc^2."""
        n = ctypes.c_int64()
        check(lib().mdg_lc_pairs(self.ctx.h, float(csf), 0, None, ctypes.byref(n)), "lc_pairs")
        out = np.zeros((max(n.value, 1), 2), dtype=np.int32)
        check(lib().mdg_lc_pairs(self.ctx.h, float(csf), n.value, out.ctypes.data, ctypes.byref(n)),
              "lc_pairs")
        out = out[:n.value].astype(np.int64)
        return np.unique(out, axis=0) if len(out) else out

    def timings(self, enable=None):
        """mdg_timings: enable/disable the build/force events, or read the
        last (build_ns, force_ns) (-1 = not measured)."""
        b, f = ctypes.c_int64(), ctypes.c_int64()
        check(lib().mdg_timings(self.ctx.h, -1 if enable is None else int(bool(enable)),
                                ctypes.byref(b), ctypes.byref(f)), "timings")
        return None if enable is not None else (b.value, f.value)

    def set_prune(self, delta=None):
        """mdg_set_prune: dynamic pruning of the tiled VL walk from the next
        rebuild (None = default skin / 3, 0 = off, > 0 = that inner skin)."""
        check(lib().mdg_set_prune(self.ctx.h, -1.0 if delta is None else float(delta)), "set_prune")

    def prune_count(self) -> int:
        """Prune walks since the last VL rebuild (-1 = pruning off)."""
        n = ctypes.c_int64()
        check(lib().mdg_prune_count(self.ctx.h, ctypes.byref(n)), "prune_count")
        return int(n.value)

    def sd_step(self, particles, gamma, max_disp):
        self.bind(particles)
        check(lib().mdg_sd_step(self.ctx.h, float(gamma), float(max_disp)), "sd_step")

    def potential_energy(self, particles, rebuild=True) -> float:
        """Shifted LJ potential energy of the current positions (north_star PE
        output; tests/test_integrator.py:227-247 of the reference)."""
        self.generation += 1
        self.bind(particles)
        pe = ctypes.c_double()
        check(lib().mdg_potential_energy(self.ctx.h, int(rebuild), ctypes.byref(pe)),
              "potential_energy")
        return float(pe.value)

    def profile(self, enable=True, reserve=0):
        """Bracket each force-kernel launch with CUDA events on the context stream;
        ``reserve``: launches whose events are created now instead of on demand."""
        check(lib().mdg_profile(self.ctx.h, max(1, int(reserve)) if enable else 0), "profile")

    def profile_read(self):
        """(summed force-kernel milliseconds, bracketed launches) since profile()."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        check(lib().mdg_profile_read(self.ctx.h, ctypes.byref(ms), ctypes.byref(n)), "profile_read")
        return float(ms.value), int(n.value)

    def status_flags(self, reset=True) -> int:
        """Device status bits since the last reset (FLAG_BLOWUP, FLAG_THERMO_ZERO)."""
        f = ctypes.c_int()
        check(lib().mdg_blowup(self.ctx.h, ctypes.byref(f), int(reset)), "blowup")
        return int(f.value)

    def blowup(self, reset=True) -> bool:
        return bool(self.status_flags(reset) & FLAG_BLOWUP)

    def set_iteration(self, iteration):
        """mdg_set_iteration: tag the following drifts with the loop iteration."""
        lib().mdg_set_iteration(self.ctx.h, int(iteration))

    def blowup_iteration(self) -> int:
        """mdg_blowup_iteration: the earliest tagged iteration whose drift left the
        domain (-1: none); read and reset."""
        it = ctypes.c_int64()
        check(lib().mdg_blowup_iteration(self.ctx.h, ctypes.byref(it)), "blowup_iteration")
        return int(it.value)

    # -- temperature, thermostat, live statistics (stats.cu) -------------------
    def temperature(self, particles) -> float:
        """current_temperature (integrator.py:72-78), bit-identical."""
        self.bind(particles)
        t = ctypes.c_double()
        check(lib().mdg_temperature(self.ctx.h, ctypes.byref(t)), "temperature")
        return float(t.value)

    def thermostat(self, particles, target, max_delta_t):
        """apply_thermostat (integrator.py:81-95) on the device, asynchronous.
        The T = 0 error surfaces through status_flags() (FLAG_THERMO_ZERO)."""
        self.bind(particles)
        check(lib().mdg_thermostat(self.ctx.h, float(target), float(max_delta_t)), "thermostat")

    def live_stats(self, particles):
        """compute_live_stats (livestats.py:46-77) on the device."""
        from .livestats import LiveStatistics
        self.bind(particles)
        out = np.zeros(6, dtype=np.float64)
        check(lib().mdg_live_stats(self.ctx.h, out.ctypes.data), "live_stats")
        return LiveStatistics(
            mean_particles_per_bin=float(out[0]), rel_std_dev_particles_per_bin=float(out[1]),
            median_particles_per_bin=float(out[2]), max_particles_per_bin=float(out[3]),
            num_bins=int(out[4]), num_empty_bins=int(out[5]),
            thread_count=self.params.thread_count, skin=self.params.skin)

    # -- parity exports --------------------------------------------------------
    def grid_state(self, csf):
        m, nc = ctypes.c_int64(), ctypes.c_int64()
        check(lib().mdg_get_grid(self.ctx.h, float(csf), ctypes.byref(m), ctypes.byref(nc),
                                 None, None, None), "get_grid")
        src = np.zeros(m.value, dtype=np.int32)
        code = np.zeros(m.value, dtype=np.int8)
        start = np.zeros(nc.value + 1, dtype=np.int32)
        check(lib().mdg_get_grid(self.ctx.h, float(csf), ctypes.byref(m), ctypes.byref(nc),
                                 src.ctypes.data, code.ctypes.data, start.ctypes.data), "get_grid")
        L = np.asarray(self.params.domain_size, dtype=np.float64)
        combo = np.stack([code // 9 - 1, (code // 3) % 3 - 1, code % 3 - 1], axis=1)
        return {"src": src.astype(np.int64), "shift": combo.astype(np.float64) * L,
                "start": start[:-1].astype(np.int64), "end": start[1:].astype(np.int64)}

    def verlet_lists(self):
        e = ctypes.c_int64()
        check(lib().mdg_get_verlet(self.ctx.h, ctypes.byref(e), None, None), "get_verlet")
        n = self._bound_n
        noff = np.zeros(n + 1, dtype=np.int64)
        nbr = np.zeros(e.value, dtype=np.int32)
        check(lib().mdg_get_verlet(self.ctx.h, ctypes.byref(e), noff.ctypes.data,
                                   nbr.ctypes.data), "get_verlet")
        return noff, nbr.astype(np.int64)

    def close(self):
        self.ctx.close()


def compute_forces(particles, config, params, workers=None, timer=None):
    """One-shot build + refresh + compute (containers.py:494-511), device-timed."""
    calc = ForceCalculator(particles, params)
    particles.convert_layout(config.layout)
    torch.cuda.synchronize(particles.device)
    t0 = time.perf_counter_ns()
    calc.rebuild(particles, config)
    calc.refresh(particles, config)
    torch.cuda.synchronize(particles.device)
    t1 = time.perf_counter_ns()
    count = calc.compute(particles, config)
    t2 = time.perf_counter_ns()
    calc.close()
    return Timings(force_ns=t2 - t1, build_ns=t1 - t0), count


class HostForceCalculator:
    """ForceCalculator protocol over HOST particle sets (the mdtune drop-in).

    Every public method synchronises before returning, so the reference's
    wall-clock ``timer()`` around build and compute (simulation.py:160-169)
    measures the GPU work including the host<->device copies.
    """

    def __init__(self, particles, params):
        self.params = params
        self.ctx = Context()
        dev = self.ctx.device
        self.ctx.set_system(params, particles.sigma, particles.epsilon, particles.mass)
        n = particles.n
        self.n = n
        self._buf = {k: torch.zeros(3 * n, dtype=torch.float64, device=dev)
                     for k in ("pos", "vel", "force", "old_force")}
        self._tid = None
        if len(particles.mass) > 1 and n:
            self._tid = torch.as_tensor(np.asarray(particles.type_id, dtype=np.int32)).to(dev)
        self.last_eval_count = 0

    def _bind(self, p):
        self.ctx.bind(self.n, p.layout, self._buf["pos"], self._buf["vel"], self._buf["force"],
                      self._buf["old_force"], self._tid)

    def _upload_positions(self, p):
        # straight from the caller's array (DMA speed when it is pinned, e.g.
        # hostloop.HostParticleSet; driver-staged for pageable numpy arrays)
        if not self.n:
            return
        src = p.pos if p.pos.flags.c_contiguous else np.ascontiguousarray(p.pos)
        check(lib().mdg_h2d(self.ctx.h, ctypes.c_void_p(self._buf["pos"].data_ptr()),
                            ctypes.c_void_p(src.ctypes.data), 24 * self.n), "h2d")

    def rebuild(self, particles, config):
        self._upload_positions(particles)
        self._bind(particles)
        check(lib().mdg_rebuild(self.ctx.h, ctypes.byref(config_struct(config))), "rebuild")

    # -- chunked pieces for the pipelined host loop (hostloop.HostSimulation) --
    def _ranges(self, p, a, b):
        """(byte offset, bytes) pieces of particles [a, b) in p's layout."""
        if p.layout == "AoS":
            return [(24 * a, 24 * (b - a))]
        return [(8 * (k * self.n + a), 8 * (b - a)) for k in range(3)]

    def upload_range(self, p, a, b):
        """Asynchronous H2D of positions [a, b) (p.pos must be pinned and contiguous)."""
        base_d, base_h = self._buf["pos"].data_ptr(), p.pos.ctypes.data
        for off, nb in self._ranges(p, a, b):
            check(lib().mdg_h2d(self.ctx.h, ctypes.c_void_p(base_d + off),
                                ctypes.c_void_p(base_h + off), nb), "h2d")

    def download_range(self, p, a, b):
        """Asynchronous D2H of forces [a, b) on the context stream."""
        base_d, base_h = self._buf["force"].data_ptr(), p.force.ctypes.data
        for off, nb in self._ranges(p, a, b):
            check(lib().mdg_d2h_async(self.ctx.h, ctypes.c_void_p(base_h + off),
                                      ctypes.c_void_p(base_d + off), nb), "d2h")

    def device_step(self, particles, config, rebuild):
        """rebuild (if due) + refresh + compute on positions already uploaded;
        asynchronous except for the rebuild's own size check."""
        self._bind(particles)
        cs = ctypes.byref(config_struct(config))
        if rebuild:
            check(lib().mdg_rebuild(self.ctx.h, cs), "rebuild")
        check(lib().mdg_refresh(self.ctx.h, cs), "refresh")
        check(lib().mdg_compute(self.ctx.h, cs), "compute")

    def refresh(self, particles, config):
        if config.container in ("VL", "VCL"):   # list containers refresh inside compute
            return
        self._upload_positions(particles)
        self._bind(particles)
        check(lib().mdg_refresh(self.ctx.h, ctypes.byref(config_struct(config))), "refresh")
        check(lib().mdg_synchronize(self.ctx.h), "sync")

    def compute(self, particles, config, workforce=None) -> int:
        if particles.layout != config.layout:
            raise ValueError(f"particle layout {particles.layout} does not match "
                             f"configuration {config.id}")
        if config.container in ("VL", "VCL"):
            self._upload_positions(particles)
        self._bind(particles)
        h = self.ctx.h
        check(lib().mdg_compute(h, ctypes.byref(config_struct(config))), "compute")
        if self.n:
            dst = particles.force
            if dst.flags.c_contiguous:
                check(lib().mdg_d2h(h, ctypes.c_void_p(dst.ctypes.data),
                                    ctypes.c_void_p(self._buf["force"].data_ptr()), 24 * self.n), "d2h")
            else:
                tmp = np.empty(dst.shape)
                check(lib().mdg_d2h(h, ctypes.c_void_p(tmp.ctypes.data),
                                    ctypes.c_void_p(self._buf["force"].data_ptr()), 24 * self.n), "d2h")
                dst[...] = tmp
        else:
            particles.force.fill(0.0)
        self.last_eval_count = self.ctx.eval_count()
        return self.last_eval_count
