"""Device-resident simulation loop (mirror of mdtune.simulation.simulate,
simulation.py:126-197, for a fixed configuration).

Per iteration, in the reference's order: drift with the previous forces,
boundaries, F -> F_old (one fused kernel, integrator.py:31-37/98-128,
simulation.py:151-153); layout conversion + rebuild when due + refresh (timed as
build); compute (timed as force); gravity + finish_kick (one kernel).  The
rebuild cadence is the reference's: rebuild when the configuration changed or
``since_rebuild >= R`` (so every R+1 iterations, simulation.py:158-159,179);
forces start at zero, so iteration 0 drifts ballistically.

Timings come from CUDA events on the context stream and are read once at the
end, so steady-state iterations never synchronise with the host.  A blow-up
(integrator.py:108-116) is detected on the device and raised at the next
rebuild (which synchronises anyway) or at the end of the run.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .calculator import ForceCalculator


class BlowUpError(RuntimeError):
    """A particle left the domain by more than one domain length."""


@dataclass
class IterationRecord:
    iteration: int
    configuration_id: str
    force_ns: int
    build_ns: int
    rebuilt: bool


@dataclass
class SimulationReport:
    records: list = field(default_factory=list)
    error: str | None = None

    @property
    def total_force_ns(self) -> int:
        return sum(r.force_ns for r in self.records)

    @property
    def total_build_ns(self) -> int:
        return sum(r.build_ns for r in self.records)


class Simulation:
    """Stepper with persistent state (calculator, cadence), so benchmarks can
    run warm-up and timed windows back to back on one trajectory."""

    def __init__(self, particles, params, config, calculator=None):
        if params.thermostat is not None:
            raise NotImplementedError("thermostat is not on the device path yet")
        self.p = particles
        self.params = params
        self.config = getattr(config, "config", config)   # FixedStrategy or Configuration
        self.calc = calculator or ForceCalculator(particles, params)
        self.active = None
        self.since = 0
        self.iteration = 0
        self._events = []

    def step(self, record=False):
        p, params, cfg, calc = self.p, self.params, self.config, self.calc
        calc.drift_wrap(p, params.delta_t)
        rebuild = self.active != cfg.id or self.since >= params.rebuild_interval
        if record:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
        if p.layout != cfg.layout:
            p.convert_layout(cfg.layout)
        if rebuild:
            if self.iteration and calc.blowup():
                raise BlowUpError("particle left the domain by more than one domain length "
                                  "(or position is not finite)")
            calc.rebuild(p, cfg)
        calc.refresh(p, cfg)
        if record:
            ev[1].record()
        calc.compute_async(p, cfg)
        if record:
            ev[2].record()
            self._events.append((self.iteration, cfg.id, rebuild, ev))
        calc.finish_kick(p, params.delta_t, params.gravity)
        self.active = cfg.id
        self.since = 0 if rebuild else self.since + 1
        self.iteration += 1
        return rebuild

    def run(self, steps, record=True):
        for _ in range(steps):
            self.step(record=record)

    def check(self):
        if self.calc.blowup():
            raise BlowUpError("particle left the domain by more than one domain length "
                              "(or position is not finite)")

    def report(self) -> SimulationReport:
        torch.cuda.synchronize(self.p.device)
        rep = SimulationReport()
        for it, cid, rebuilt, ev in self._events:
            build_ns = int(ev[0].elapsed_time(ev[1]) * 1e6)
            force_ns = int(ev[1].elapsed_time(ev[2]) * 1e6)
            rep.records.append(IterationRecord(it, cid, force_ns, build_ns, rebuilt))
        self._events.clear()
        return rep


def simulate(particles, params, config, *, steps=None, record=True, raise_errors=True):
    """Run ``params.total_iterations`` (or ``steps``) iterations under a fixed
    configuration; returns the per-iteration device timings."""
    steps = params.total_iterations if steps is None else steps
    sim = Simulation(particles, params, config)
    try:
        sim.run(steps, record=record)
        sim.check()
        rep = sim.report()
    except BlowUpError as exc:
        rep = sim.report()
        rep.error = f"BlowUpError: {exc}"
        if raise_errors:
            raise
    finally:
        sim.calc.close()
    return rep
