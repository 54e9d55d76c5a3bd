"""Host-resident simulation with the GPU force path (the reference-facing
drop-in, end to end).

State lives in host memory the way the reference keeps it (numpy arrays of a
ParticleSet, particles.py:31-98); every step the reference loop
(simulation.py:150-188) runs with the GPU ``HostForceCalculator`` as its force
backend: positions go host->device, forces come back device->host, and the
Verlet update runs on the host with libmdg's native multithreaded integrator
(same rounding as the reference's numpy sequence, integrator.py:31-128).

``HostParticleSet`` allocates its arrays in pinned host memory so the copies run
at DMA speed; any object with the reference ParticleSet's attributes works.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .calculator import HostForceCalculator
from ._lib import check, lib


def _pinned(shape):
    """Page-locked host array (DMA-speed copies); plain pages when no CUDA
    driver is present (host-only use, e.g. the CPU test suite)."""
    if torch.cuda.is_available():
        return torch.zeros(shape, dtype=torch.float64).pin_memory().numpy()
    return np.zeros(shape)


class HostParticleSet:
    """Reference-shaped ParticleSet on pinned host memory."""

    def __init__(self, positions, velocities=None, type_ids=None, sigma=(1.0,), epsilon=(1.0,),
                 mass=(1.0,), layout="AoS"):
        pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
        n = pos.shape[0]
        self.layout = "AoS"
        self.pos, self.vel, self.force, self.old_force = (_pinned((n, 3)) for _ in range(4))
        self.pos[:] = pos
        if velocities is not None:
            self.vel[:] = np.asarray(velocities, dtype=np.float64).reshape(n, 3)
        self.type_id = (np.zeros(n, dtype=np.int64) if type_ids is None
                        else np.asarray(type_ids, dtype=np.int64).copy())
        self.sigma = np.asarray(sigma, dtype=np.float64)
        self.epsilon = np.asarray(epsilon, dtype=np.float64)
        self.mass = np.asarray(mass, dtype=np.float64)
        self._tid32 = self.type_id.astype(np.int32)
        if layout == "SoA":
            self.convert_layout("SoA")

    @property
    def n(self):
        return self.type_id.shape[0]

    def convert_layout(self, target):
        if target == self.layout:
            return self
        for name in ("pos", "vel", "force", "old_force"):
            a = getattr(self, name)
            b = _pinned(a.T.shape)
            b[:] = a.T
            setattr(self, name, b)
        self.layout = target
        return self

    def view(self, name):
        a = getattr(self, name)
        return a if self.layout == "AoS" else a.T

    positions = property(lambda s: s.view("pos"))
    velocities = property(lambda s: s.view("vel"))
    forces = property(lambda s: s.view("force"))
    old_forces = property(lambda s: s.view("old_force"))


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def host_drift_wrap(p, params, dt):
    """drift_with_force + apply_boundaries + F -> F_old (integrator.py)."""
    L = np.ascontiguousarray(params.domain_size, dtype=np.float64)
    per = np.ascontiguousarray(params.periodic_flags().astype(np.int32))
    mass = np.ascontiguousarray(p.mass, dtype=np.float64)
    tid = getattr(p, "_tid32", None)
    if tid is None:
        tid = np.asarray(p.type_id, dtype=np.int32)
    bad = ctypes.c_int()
    check(lib().mdg_host_drift_wrap(p.n, _lib.AOS if p.layout == "AoS" else _lib.SOA,
                                    _ptr(p.pos), _ptr(p.vel), _ptr(p.force), _ptr(p.old_force),
                                    _ptr(tid) if len(mass) > 1 else None, _ptr(mass),
                                    _ptr(L), _ptr(per), float(dt), ctypes.byref(bad)), "host drift")
    return bool(bad.value)


def host_drift_wrap_range(p, params, dt, a, b):
    """host_drift_wrap on particles [a, b)."""
    L = np.ascontiguousarray(params.domain_size, dtype=np.float64)
    per = np.ascontiguousarray(params.periodic_flags().astype(np.int32))
    mass = np.ascontiguousarray(p.mass, dtype=np.float64)
    tid = getattr(p, "_tid32", None)
    if tid is None:
        tid = np.asarray(p.type_id, dtype=np.int32)
    bad = ctypes.c_int()
    check(lib().mdg_host_drift_wrap_range(p.n, int(a), int(b), _lib.AOS if p.layout == "AoS" else _lib.SOA,
                                          _ptr(p.pos), _ptr(p.vel), _ptr(p.force), _ptr(p.old_force),
                                          _ptr(tid) if len(mass) > 1 else None, _ptr(mass),
                                          _ptr(L), _ptr(per), float(dt), ctypes.byref(bad)), "host drift")
    return bool(bad.value)


def host_finish_kick_range(p, dt, gravity, a, b):
    mass = np.ascontiguousarray(p.mass, dtype=np.float64)
    tid = getattr(p, "_tid32", None)
    if tid is None:
        tid = np.asarray(p.type_id, dtype=np.int32)
    check(lib().mdg_host_finish_kick_range(p.n, int(a), int(b), _lib.AOS if p.layout == "AoS" else _lib.SOA,
                                           _ptr(p.vel), _ptr(p.force), _ptr(p.old_force),
                                           _ptr(tid) if len(mass) > 1 else None, _ptr(mass), float(dt),
                                           int(gravity is not None), float(gravity or 0.0)),
          "host finish_kick")


def host_finish_kick(p, dt, gravity=None):
    mass = np.ascontiguousarray(p.mass, dtype=np.float64)
    tid = getattr(p, "_tid32", None)
    if tid is None:
        tid = np.asarray(p.type_id, dtype=np.int32)
    check(lib().mdg_host_finish_kick(p.n, _lib.AOS if p.layout == "AoS" else _lib.SOA,
                                     _ptr(p.vel), _ptr(p.force), _ptr(p.old_force),
                                     _ptr(tid) if len(mass) > 1 else None, _ptr(mass), float(dt),
                                     int(gravity is not None), float(gravity or 0.0)),
          "host finish_kick")


class HostSimulation:
    """The reference loop (simulation.py:150-188, fixed configuration) on host
    state with the GPU force backend.  Create once, then ``run(steps)``.

    With ``chunks > 1`` (default 16) a step is one native call
    (``mdg_host_step``) in which the host work overlaps the copies: the drift
    of chunk k runs while chunk k-1's positions are in flight to the device,
    and the kick of chunk k starts as soon as its forces have landed.  The
    arithmetic and its order per particle are unchanged (same results, bit
    for bit); only the copies are split."""

    def __init__(self, particles, params, config, calculator=None, chunks=16):
        self.p, self.params, self.config = particles, params, config
        self.calc = calculator or HostForceCalculator(particles, params)
        self.active, self.since, self.iteration = None, 0, 0
        self.chunks = max(1, int(chunks))

    def _bounds(self):
        n = self.p.n
        k = min(self.chunks, max(1, n))
        return [(n * i // k, n * (i + 1) // k) for i in range(k)]

    def step(self):
        p, params, cfg, calc = self.p, self.params, self.config, self.calc
        from .simulation import BlowUpError
        if p.layout != cfg.layout:
            p.convert_layout(cfg.layout)
        pipelined = self.chunks > 1 and p.n > 0 and isinstance(calc, HostForceCalculator) \
            and p.pos.flags.c_contiguous and p.force.flags.c_contiguous
        if not pipelined:
            if host_drift_wrap(p, params, params.delta_t):
                raise BlowUpError("particle left the domain by more than one domain length "
                                  "(or position is not finite)")
            rebuild = self.active != cfg.id or self.since >= params.rebuild_interval
            if rebuild:
                calc.rebuild(p, cfg)
            calc.refresh(p, cfg)
            calc.compute(p, cfg)
            host_finish_kick(p, params.delta_t, params.gravity)
        else:
            # one native call: chunked host drift / H2D overlap, device force
            # path, chunked D2H / host kick overlap (mdg_host_step)
            rebuild = self.active != cfg.id or self.since >= params.rebuild_interval
            calc._bind(p)
            mass = np.ascontiguousarray(p.mass, dtype=np.float64)
            tid = getattr(p, "_tid32", None)
            if tid is None:
                tid = np.asarray(p.type_id, dtype=np.int32)
            bad = ctypes.c_int()
            # F -> F_old by swapping the two buffers instead of copying (the
            # state after the step is the same, MDG_HOST_STEP_SWAPPED)
            p.force, p.old_force = p.old_force, p.force
            check(lib().mdg_host_step_ex(calc.ctx.h, ctypes.byref(_lib.config_struct(cfg)), _ptr(p.pos),
                                         _ptr(p.vel), _ptr(p.force), _ptr(p.old_force),
                                         _ptr(tid) if len(mass) > 1 else None, _ptr(mass),
                                         float(params.delta_t), int(params.gravity is not None),
                                         float(params.gravity or 0.0), int(rebuild), self.chunks,
                                         1, ctypes.byref(bad)), "host step")
            if bad.value:
                raise BlowUpError("particle left the domain by more than one domain length "
                                  "(or position is not finite)")
        self.active = cfg.id
        self.since = 0 if rebuild else self.since + 1
        self.iteration += 1

    def _pipelined(self):
        p, calc = self.p, self.calc
        return (self.chunks > 1 and p.n > 0 and isinstance(calc, HostForceCalculator)
                and p.pos.flags.c_contiguous and p.force.flags.c_contiguous)

    def run(self, steps):
        """``steps`` iterations.  Pipelined, they are ONE native call
        (``mdg_host_run``) that also overlaps consecutive steps: as each force
        chunk lands, its kick and the next step's drift run in one host pass
        and its positions go straight back up, while the rest of the forces
        are still coming down.  Same state after the run, bit for bit, as
        ``steps`` calls of ``step()``."""
        steps = int(steps)
        if steps <= 0:
            return
        p, params, cfg, calc = self.p, self.params, self.config, self.calc
        if p.layout != cfg.layout:
            p.convert_layout(cfg.layout)
        if not self._pipelined():
            for _ in range(steps):
                self.step()
            return
        from .simulation import BlowUpError
        calc._bind(p)
        mass = np.ascontiguousarray(p.mass, dtype=np.float64)
        tid = getattr(p, "_tid32", None)
        if tid is None:
            tid = np.asarray(p.type_id, dtype=np.int32)
        rebuild_first = self.active != cfg.id
        bad, done = ctypes.c_int(), ctypes.c_int()
        p.force, p.old_force = p.old_force, p.force   # MDG_HOST_STEP_SWAPPED on entry
        check(lib().mdg_host_run(calc.ctx.h, ctypes.byref(_lib.config_struct(cfg)), _ptr(p.pos),
                                 _ptr(p.vel), _ptr(p.force), _ptr(p.old_force),
                                 _ptr(tid) if len(mass) > 1 else None, _ptr(mass),
                                 float(params.delta_t), int(params.gravity is not None),
                                 float(params.gravity or 0.0), steps, int(params.rebuild_interval),
                                 int(self.since), int(rebuild_first), self.chunks,
                                 ctypes.byref(bad), ctypes.byref(done)), "host run")
        k = done.value
        if k % 2 == 0:   # the buffers alternate per step; put the latest forces in p.force
            p.force, p.old_force = p.old_force, p.force
        for s in range(k):
            rebuild = (s == 0 and rebuild_first) or self.since >= params.rebuild_interval
            self.since = 0 if rebuild else self.since + 1
        if k:
            self.active = cfg.id
        self.iteration += k
        if bad.value:
            raise BlowUpError("particle left the domain by more than one domain length "
                              "(or position is not finite)")
