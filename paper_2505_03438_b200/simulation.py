"""Device-resident simulation loop (mirror of mdtune.simulation.simulate,
simulation.py:126-197), for a fixed configuration or driven by a tuning
controller.

Per iteration, in the reference's order: drift with the previous forces,
boundaries, F -> F_old (one fused kernel, integrator.py:31-37/98-128,
simulation.py:151-153); ask the controller for this iteration's
configuration (tuning.py:200-210); layout conversion + rebuild when due +
refresh (timed as build); compute + gravity + finish_kick (timed as force;
the kick is fused into the tiled Verlet walk, its own kernel elsewhere); the
thermostat every ``interval_iterations``
(simulation.py:186-188, on the device, stats.cu).  The rebuild cadence is
the reference's: rebuild when forced (first sample of a trial), when the
configuration changed, or when ``since_rebuild >= R`` (so every R+1
iterations, simulation.py:158-159,179); forces start at zero, so iteration 0
drifts ballistically.

Timings are CUDA events on the context stream.  Steady-state iterations are
read once at the end, so they never synchronise with the host; trial
iterations synchronise on their compute event, because the controller
advances its candidate queue on every ``record_timings`` (tuning.py:212-227).
In steady mode the reference's ``record_timings`` is a no-op (tuning.py:213),
so it is not called.  A failing candidate is reported with
``record_failure`` and the iteration is retried with the next one
(simulation.py:155-176).  Device errors (BlowUpError, the thermostat's T = 0
ValueError) are flags checked at every rebuild (which synchronises anyway)
and at the end of the run.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import torch

from ._lib import FLAG_BLOWUP, FLAG_THERMO_ZERO
from .calculator import ForceCalculator
from .configuration import VERLET_LISTS, enumerate_configurations

TRIAL = "trial"


class BlowUpError(RuntimeError):
    """A particle left the domain by more than one domain length."""


class _StatusFlags(Exception):
    """Device status bits found by mdg_rebuild_checked (re-raised by
    Simulation._check_flags as BlowUpError / ValueError)."""

    def __init__(self, flags):
        super().__init__(flags)
        self.flags = flags


@dataclass
class IterationRecord:
    iteration: int
    configuration_id: str
    force_ns: int
    build_ns: int
    rebuilt: bool
    phase_index: int = 0


# MDG_STEP_TRACE=1: host wall time of each phase of a step() that reorders
# (diagnostics for host stalls: tools/spike_probe.sh)
_TRACE = bool(os.environ.get("MDG_STEP_TRACE"))
STEP_TRACE = []


@dataclass
class SimulationReport:
    name: str = "simulation"
    strategy_name: str = "fixed"
    records: list = field(default_factory=list)
    tuning_log: list = field(default_factory=list)
    phase_selections: list = field(default_factory=list)
    stats_snapshots: list = field(default_factory=list)
    trial_iterations: int = 0
    final_temperature: float | None = None
    error: str | None = None

    @property
    def total_force_ns(self) -> int:
        return sum(r.force_ns for r in self.records)

    @property
    def total_build_ns(self) -> int:
        return sum(r.build_ns for r in self.records)

    def configuration_sequence(self) -> list:
        return [r.configuration_id for r in self.records]


class _Fixed:
    """FixedStrategy as a controller: one configuration, never forced."""

    mode = "steady"

    def __init__(self, config):
        self.config = config

    def configuration_for_iteration(self, iteration):
        return self.config, False

    def record_timings(self, force_ns, build_ns):
        pass

    def record_failure(self, error=None):
        return False


class Simulation:
    """Stepper with persistent state (calculator, cadence, controller), so
    benchmarks can run warm-up and timed windows back to back on one
    trajectory.  ``config`` is a Configuration / FixedStrategy; ``controller``
    anything with the TuningController protocol (tuning.py:200-239)."""

    def __init__(self, particles, params, config=None, calculator=None, controller=None,
                 tuning_interval=None, graphs=False, fuse_kick_drift=False, reorder=0):
        if controller is None:
            if config is None:
                raise ValueError("need a configuration or a controller")
            controller = _Fixed(getattr(config, "config", config))
        self.p = particles
        self.params = params
        self.controller = controller
        self.tuning_interval = (tuning_interval or getattr(controller, "tuning_interval", None)
                                or 1000)
        self.calc = calculator or ForceCalculator(particles, params)
        self.active = None
        self.since = 0
        self.iteration = 0
        self._events = []
        self._records = []
        # steady-state iterations (no rebuild, not timed) from a cached CUDA
        # graph of drift + refresh + compute + kick (mdg_step_graph)
        self.graphs = graphs
        # defer an untimed step's kick into the next step's drift (one pass,
        # mdg_kick_drift, force / old_force swapped instead of copied); the
        # state is complete again after flush() (run(), check() and report()
        # flush; callers of step() who read particles in between call it)
        self.fuse_kick_drift = fuse_kick_drift
        self._kick_due = False
        # keep the particle arrays in the container's cell order: every
        # `reorder`-th rebuild outside tuning trials permutes them by the previous grid's
        # row order (mdg_owned_order), so the refresh gathers, the force
        # stores and the binning touch memory in order.  flush() restores
        # the caller's order; the next step re-applies it.  Verlet lists only:
        # their rows are z-ordered within a cell, so forces are unchanged bit
        # for bit, while the linked-cell rows follow the particle index (the
        # reference's stable order) and would sum in another order.  The
        # particle-order reductions (temperature) do sum in another order.
        # The ParticleSet's array tensors are replaced (spares are recycled):
        # hold the ParticleSet, not its tensors, across steps.  0 = off.
        self.reorder = int(reorder)
        self._perm = None          # current index -> caller's index
        self._permuted = False
        self._perm_gen = None
        self._rebuilds = 0
        self._active_cfg = None
        self._spare = {}           # array name -> spare arrays for _permute
        self._skip_reorder = False
        self._perm_spare = None
        self._iota = self._inv = None
        self._order_tmp = self._order_buf = None   # owned_order's buffers (no allocation per reorder)
        # untimed steady iterations of a fixed configuration run as one native
        # call (mdg_run) inside run(); False: every iteration through step()
        self.native = True

    @property
    def config(self):
        return getattr(self.controller, "current_config", None) or getattr(self.controller, "config", None)

    def _check_flags(self, flags=None):
        if flags is None:
            flags = self.calc.status_flags()
        if flags & FLAG_BLOWUP:
            # the reference raises inside the failing iteration's
            # apply_boundaries (integrator.py:108-116); the device flag is read
            # at rebuilds, so the loop may have run on: report the failing
            # iteration and keep only the records of the iterations before it
            it = self.calc.blowup_iteration() if hasattr(self.calc, "blowup_iteration") else -1
            where = ""
            if it >= 0:
                self._records = [r for r in self._records if r.iteration < it]
                self._events = [e for e in self._events if e[0] < it]
                self.iteration = it
                where = f" at iteration {it}"
            raise BlowUpError("particle left the domain by more than one domain length "
                              f"(or position is not finite){where}")
        if flags & FLAG_THERMO_ZERO:
            raise ValueError("thermostat cannot scale zero velocities toward a positive "
                             "target temperature")

    def _trial(self):
        return getattr(self.controller, "mode", TRIAL) == TRIAL

    # -- cell-order permutation of the particle arrays (reorder) --------------
    def _permute(self, order):
        """All five particle arrays gathered by ``order`` in one libmdg pass
        (mdg_gather_rows) into spare arrays of the same shape (double
        buffering: no allocation once both sets exist, so no cudaMalloc inside
        a timed loop)."""
        import ctypes

        from ._lib import check, lib
        p = self.p
        names = ("pos", "vel", "force", "old_force", "type_id")
        outs = {}
        for name in names:
            src = getattr(p, name)
            pool = self._spare.setdefault(name, [])
            out = next((t for t in pool if t.shape == src.shape and t.device == src.device
                        and t.dtype == src.dtype and t is not src), None)
            if out is None:
                out = torch.empty_like(src)
            else:
                pool.remove(out)
            outs[name] = out
        order = order.to(torch.int64).contiguous()
        P4 = ctypes.c_void_p * 4
        srcs = P4(*(getattr(p, k).data_ptr() for k in names[:4]))
        dsts = P4(*(outs[k].data_ptr() for k in names[:4]))
        check(lib().mdg_gather_rows(self.calc.ctx.h, ctypes.c_void_p(order.data_ptr()), int(order.numel()),
                                    int(p.layout == "SoA"), srcs, dsts,
                                    ctypes.c_void_p(p.type_id.data_ptr()),
                                    ctypes.c_void_p(outs["type_id"].data_ptr())), "gather_rows")
        for name in names:
            self._spare[name].append(getattr(p, name))
            setattr(p, name, outs[name])

    def _reapply_order(self):
        if self._perm is None or self._permuted:
            return
        if self.calc.generation != self._perm_gen:
            self._perm = None      # a container was rebuilt on the caller's order
            return
        self._permute(self._perm)
        self._permuted = True

    def _restore_order(self):
        if self._perm is None or not self._permuted:
            return
        n = self._perm.numel()
        if self._inv is None or self._inv.numel() != n or self._inv.device != self._perm.device:
            self._inv = torch.empty_like(self._perm)
        self.calc.permutation(1, self._perm, None, self._inv)   # inv[perm[i]] = i, in libmdg
        self._permute(self._inv)
        self._permuted = False
        self._perm_gen = self.calc.generation

    def warm_reorder(self):
        """Take the first cell reorder outside a timed loop: permute the arrays
        by the current grid's order now (the next step then rebuilds on the
        new order) and run the flush path once, so the one-time costs -- the
        spare arrays, the scratch of the order export, the first use of each
        kernel involved (a first scatter took 12.7 ms) -- are paid here."""
        cfg = self._active_cfg
        if not self.reorder or cfg is None or cfg.container != VERLET_LISTS:
            return
        self.flush()
        self._reapply_order()
        n = self.p.n
        ident = torch.arange(n, device=self.p.pos.device)
        self._iota = ident
        self._inv = torch.empty_like(ident)
        self._reorder()                       # allocates the first spares
        self._perm_spare = torch.empty_like(self._perm)
        self.calc.permutation(0, self._perm, ident, self._perm_spare)   # (later compositions)
        self._restore_order()                 # the flush path ...
        self._reapply_order()                 # ... and the next step's re-apply
        self._permute(ident)                  # the second set of spares
        self.since = self.params.rebuild_interval   # the grid is on the old order: rebuild next,
        self._skip_reorder = True                   # and take no order from it
        torch.cuda.synchronize(self.p.pos.device)

    def _reorder(self):
        # the order lands in buffers this loop owns: nothing is allocated from
        # the second reorder on
        n = self.p.n
        dev = self.p.pos.device
        if self._order_tmp is None or self._order_tmp.numel() != n or self._order_tmp.device != dev:
            self._order_tmp = torch.empty(n, dtype=torch.int32, device=dev)
        if self._order_buf is None or self._order_buf.numel() != n or self._order_buf.device != dev:
            self._order_buf = torch.empty(n, dtype=torch.int64, device=dev)
        order = self.calc.owned_order(self._active_cfg, out=self._order_buf, tmp=self._order_tmp)
        self._permute(order)
        if self._perm is None:
            self._perm = order
            self._order_buf = torch.empty_like(order)   # (the first reorder keeps its buffer)
        else:   # compose into the spare permutation buffer (no allocation)
            out = self._perm_spare
            if out is None or out.shape != self._perm.shape or out.device != self._perm.device:
                out = torch.empty_like(self._perm)
            self.calc.permutation(0, self._perm, order, out)   # out = perm[order], in libmdg
            self._perm_spare, self._perm = self._perm, out
        self._permuted = True

    def step(self, record=False):
        # an untimed iteration of a fixed configuration: one native call
        # (mdg_run; a steady step replays its captured graph)
        if self._native_span(1, record):
            since = self.since
            self._run_native(1)
            return self.since < since + 1   # rebuilt
        p, params, calc, ctl = self.p, self.params, self.calc, self.controller
        it = self.iteration
        self._reapply_order()
        if self.graphs and not record and not self._kick_due and self._graph_step(it):
            return False
        if hasattr(calc, "set_iteration"):
            calc.set_iteration(it)   # tags this drift for the blow-up report
        if self._kick_due:
            calc.kick_drift(p, params.delta_t, params.gravity, copy_old_force=False)
            p.force, p.old_force = p.old_force, p.force
            self._kick_due = False
        else:
            calc.drift_wrap(p, params.delta_t)
        pending = getattr(self, "_pending", None)
        self._pending = None
        tr = None
        while True:
            if pending is not None:
                cfg, forced = pending
                pending = None
            else:
                cfg, forced = ctl.configuration_for_iteration(it)
            rebuild = forced or self.active != cfg.id or self.since >= params.rebuild_interval
            trial = self._trial()
            # the error check before a rebuild (simulation.py:158-166) rides on
            # the rebuild's own host synchronisation (mdg_rebuild_checked)
            checked = bool(rebuild and it and hasattr(calc, "rebuild_checked"))
            if rebuild and it and not checked:
                self._check_flags()
            timed = record or trial
            if (rebuild and self.reorder and not trial and self._active_cfg is not None
                    and self._active_cfg.container == VERLET_LISTS and cfg.container == VERLET_LISTS
                    and hasattr(calc, "owned_order") and (self._rebuilds - 1) % self.reorder == 0):
                if self._skip_reorder:
                    self._skip_reorder = False
                else:
                    if _TRACE:
                        tr = [time.perf_counter()]
                    self._reorder()
                    if _TRACE:
                        tr.append(time.perf_counter())
            if timed:
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                ev[0].record()
            try:
                if p.layout != cfg.layout:
                    p.convert_layout(cfg.layout)
                if rebuild:
                    if checked:
                        flags = calc.rebuild_checked(p, cfg)
                        if flags:
                            raise _StatusFlags(flags)
                    else:
                        calc.rebuild(p, cfg)
                if tr is not None:
                    tr.append(time.perf_counter())
                calc.refresh(p, cfg)
                if timed:
                    ev[1].record()
                thermo = params.thermostat
                defer = (self.fuse_kick_drift and not timed and not self.graphs
                         and (thermo is None or (it + 1) % thermo.interval_iterations != 0))
                if defer:   # the kick runs inside the next step's drift
                    calc.compute_async(p, cfg)
                    self._kick_due = True
                else:
                    # force + gravity + finish_kick; the kick is fused into the
                    # force walk where the configuration allows (mdg_compute_kick)
                    calc.compute_kick_async(p, cfg, params.delta_t, params.gravity)
                if timed:
                    ev[2].record()
                if tr is not None:   # (iteration, reorder, rebuild, refresh + compute) host ms
                    tr.append(time.perf_counter())
                    STEP_TRACE.append((it,) + tuple(round((b - a) * 1e3, 3) for a, b in zip(tr, tr[1:])))
                break
            except (BlowUpError, KeyboardInterrupt):
                raise
            except _StatusFlags as sf:   # raised as the reference raises them, outside the retry
                self._check_flags(sf.flags)
                raise
            except Exception as exc:
                if not ctl.record_failure(exc):
                    raise
                self.active = None
        self.active = cfg.id
        self._active_cfg = cfg
        self._rebuilds += int(bool(rebuild))
        self.since = 0 if rebuild else self.since + 1
        phase = it // self.tuning_interval
        if trial:
            ev[2].synchronize()
            build_ns = int(ev[0].elapsed_time(ev[1]) * 1e6)
            force_ns = int(ev[1].elapsed_time(ev[2]) * 1e6)
            ctl.record_timings(force_ns, build_ns)
            self._records.append(IterationRecord(it, cfg.id, force_ns, build_ns, rebuild, phase))
        elif timed:
            self._events.append((it, cfg.id, rebuild, phase, ev))
        thermo = params.thermostat
        if thermo is not None and (it + 1) % thermo.interval_iterations == 0:
            calc.thermostat(p, thermo.target_temperature, thermo.max_delta_t)
        self.iteration += 1
        return rebuild

    def _graph_step(self, it) -> bool:
        """Steady-state iteration from the step graph; False when this
        iteration needs the eager path (rebuild due, trial, layout change)."""
        p, params, ctl = self.p, self.params, self.controller
        if self.active is None or self.since >= params.rebuild_interval or self._trial():
            return False
        cfg, forced = ctl.configuration_for_iteration(it)
        if forced or cfg.id != self.active or p.layout != cfg.layout or self._trial():
            # hand the (already answered) query to the eager path
            self._pending = (cfg, forced)
            return False
        self.calc.step_graph(p, cfg, params.delta_t, params.gravity)
        thermo = params.thermostat
        if thermo is not None and (it + 1) % thermo.interval_iterations == 0:
            self.calc.thermostat(p, thermo.target_temperature, thermo.max_delta_t)
        self.since += 1
        self.iteration += 1
        return True

    def flush(self):
        """Run a deferred kick (fuse_kick_drift) and restore the caller's particle
        order (reorder), completing the state."""
        if self._kick_due:
            self.calc.finish_kick(self.p, self.params.delta_t, self.params.gravity)
            self._kick_due = False
        self._restore_order()

    def run(self, steps, record=True):
        k = 0
        while k < steps:
            span = self._native_span(steps - k, record)
            if span:
                k += self._run_native(span)
            else:
                self.step(record=record)
                k += 1
        self.flush()

    # -- the fixed-configuration loop in one native call (mdg_run) ------------
    def _native_span(self, left, record) -> int:
        """How many of the next `left` iterations mdg_run may take: untimed
        steady iterations of a fixed configuration whose container is built,
        up to the next thermostat iteration (0: the eager step() runs)."""
        if (not self.native or record or self.graphs or not self.fuse_kick_drift
                or not isinstance(self.controller, _Fixed)
                or not hasattr(self.calc, "run_fixed") or self._active_cfg is None):
            return 0
        cfg = self.controller.config
        if self.active != cfg.id or self.p.layout != cfg.layout:
            return 0
        span = left
        if self.reorder and cfg.container == VERLET_LISTS:
            # the cell reorder runs at rebuilds, in step(): native spans stop short of them
            span = min(span, max(0, self.params.rebuild_interval - self.since))
        thermo = self.params.thermostat
        if thermo is not None:
            # iterations it with (it + 1) % interval == 0 run eagerly (kick, then thermostat)
            span = min(span, (-(self.iteration + 1)) % thermo.interval_iterations)
        return span

    def _run_native(self, span) -> int:
        cfg, params = self.controller.config, self.params
        self._reapply_order()   # as step() does: the container indexes the permuted arrays
        done, since, kick_due, flags = self.calc.run_fixed(
            self.p, cfg, span, params.delta_t, params.gravity, params.rebuild_interval,
            self.iteration, self.since, self._kick_due)
        self.iteration += done
        self.since, self._kick_due = since, kick_due
        if flags:
            self._check_flags(flags)   # raises (BlowUpError / ValueError), as step() does
        return done

    def check(self):
        self.flush()
        self._check_flags()

    def report(self, rep=None) -> SimulationReport:
        self.flush()
        torch.cuda.synchronize(self.p.device)
        rep = rep or SimulationReport()
        for it, cid, rebuilt, phase, ev in self._events:
            build_ns = int(ev[0].elapsed_time(ev[1]) * 1e6)
            force_ns = int(ev[1].elapsed_time(ev[2]) * 1e6)
            self._records.append(IterationRecord(it, cid, force_ns, build_ns, rebuilt, phase))
        self._events.clear()
        self._records.sort(key=lambda r: r.iteration)
        rep.records.extend(self._records)
        self._records = []
        ctl = self.controller
        rep.tuning_log = list(getattr(ctl, "log", rep.tuning_log))
        rep.phase_selections = list(getattr(ctl, "phase_selections", rep.phase_selections))
        rep.stats_snapshots = list(getattr(ctl, "stats_snapshots", rep.stats_snapshots))
        rep.trial_iterations = int(getattr(ctl, "trial_iterations", rep.trial_iterations))
        return rep


def _is_configuration(obj) -> bool:
    return hasattr(obj, "container") and hasattr(obj, "layout")


def simulate(particles, params, strategy, *, tuning_interval=1000, samples_per_config=3,
             space=None, name="simulation", raise_errors=False, steps=None, record=True,
             controller=None, controller_cls=None, graphs=False) -> SimulationReport:
    """simulation.py:126-197 on the device.

    ``strategy`` is a Configuration, a FixedStrategy (anything with
    ``.config``), or a tuning strategy; a tuning strategy is driven by
    ``controller_cls`` (default: the reference's ``mdtune.tuning.
    TuningController`` when importable), constructed exactly as the
    reference does (simulation.py:132-137) with the live statistics computed
    on the device.  ``controller`` passes a ready controller object instead.
    Returns the report, partial with ``error`` set if an error interrupted
    the run (re-raised when ``raise_errors``)."""
    steps = params.total_iterations if steps is None else steps
    calc = ForceCalculator(particles, params)
    fixed = None
    if controller is None:
        if _is_configuration(strategy):
            fixed = strategy
        elif hasattr(strategy, "config") and not hasattr(strategy, "candidates"):
            fixed = strategy.config
        else:
            if controller_cls is None:
                try:
                    from mdtune.tuning import TuningController as controller_cls
                except ImportError:
                    calc.close()
                    raise RuntimeError("a tuning strategy needs a controller: pass controller_cls= "
                                       "(mdtune.tuning.TuningController) or controller=") from None
            controller = controller_cls(
                space if space is not None else enumerate_configurations(), strategy,
                samples_per_config=samples_per_config, tuning_interval=tuning_interval,
                rebuild_interval=params.rebuild_interval,
                total_iterations=params.total_iterations,
                stats_provider=lambda: calc.live_stats(particles))
    strategy_name = getattr(strategy, "name", None) or ("fixed" if fixed is not None else "tuned")
    rep = SimulationReport(name=name, strategy_name=str(strategy_name))
    sim = Simulation(particles, params, fixed, calculator=calc, controller=controller,
                     tuning_interval=tuning_interval, graphs=graphs)
    try:
        sim.run(steps, record=record)
        sim.check()
        sim.report(rep)
        if particles.n:
            rep.final_temperature = calc.temperature(particles)
    except Exception as exc:
        try:
            sim.report(rep)
        except Exception:   # the device error that stopped the run
            pass
        rep.error = f"{type(exc).__name__}: {exc}"
        if raise_errors:
            raise
    finally:
        calc.close()
    return rep
