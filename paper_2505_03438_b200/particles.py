"""Device-resident particle storage (mirror of mdtune.particles, particles.py:31-139).

AoS keeps every attribute as an (N, 3) C-contiguous fp64 tensor, SoA as a
(3, N) one; conversion is an exact transpose copy and converting to the current
layout is a no-op (particles.py:88-98).  Tensors live on a CUDA device (torch is
only the allocator); type ids are int32 on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

AOS = "AoS"
SOA = "SoA"
_ATTRS = ("pos", "vel", "force", "old_force")


@dataclass(frozen=True)
class ParticleTypeInfo:
    type_id: int
    epsilon: float
    sigma: float
    mass: float

    def __post_init__(self):
        if self.epsilon <= 0:
            raise ValueError("epsilon must be > 0")
        if self.sigma <= 0:
            raise ValueError("sigma must be > 0")
        if self.mass <= 0:
            raise ValueError("mass must be > 0")


def _as_f64(a, n, device, name):
    if a is None:
        return torch.zeros((n, 3), dtype=torch.float64, device=device)
    t = torch.as_tensor(np.asarray(a, dtype=np.float64) if not torch.is_tensor(a) else a,
                        dtype=torch.float64)
    if t.shape != (n, 3):
        raise ValueError(f"{name} must be ({n}, 3)")
    return t.to(device).contiguous().clone()


class ParticleSet:
    def __init__(self, positions, velocities=None, type_ids=None, types=None, layout=AOS,
                 device="cuda"):
        if torch.is_tensor(positions):
            n = positions.shape[0] if positions.ndim == 2 else -1
        else:
            positions = np.asarray(positions, dtype=np.float64)
            n = positions.shape[0] if positions.ndim == 2 else -1
        if n < 0 or (positions.shape[1] if positions.ndim == 2 else 0) != 3:
            raise ValueError("positions must be (N, 3)")
        self.device = torch.device(device)
        self.types = list(types) if types is not None else [ParticleTypeInfo(0, 1.0, 1.0, 1.0)]
        by_id = {t.type_id: t for t in self.types}
        if len(by_id) != len(self.types):
            raise ValueError("duplicate type ids")
        ntypes = max(by_id) + 1 if by_id else 1
        self.epsilon = np.zeros(ntypes)
        self.sigma = np.zeros(ntypes)
        self.mass = np.ones(ntypes)
        for t in self.types:
            self.epsilon[t.type_id] = t.epsilon
            self.sigma[t.type_id] = t.sigma
            self.mass[t.type_id] = t.mass
        tid = (np.zeros(n, dtype=np.int64) if type_ids is None
               else np.asarray(type_ids.cpu() if torch.is_tensor(type_ids) else type_ids,
                               dtype=np.int64))
        if tid.shape != (n,):
            raise ValueError("type ids must be (N,)")
        if n and not set(np.unique(tid).tolist()).issubset(by_id):
            raise ValueError("particle references unknown type id")
        self.layout = AOS
        self.pos = _as_f64(positions, n, self.device, "positions")
        self.vel = _as_f64(velocities, n, self.device, "velocities")
        self.force = torch.zeros((n, 3), dtype=torch.float64, device=self.device)
        self.old_force = torch.zeros((n, 3), dtype=torch.float64, device=self.device)
        self.type_id = torch.as_tensor(tid.astype(np.int32)).to(self.device)
        if layout == SOA:
            self.convert_layout(SOA)
        elif layout != AOS:
            raise ValueError(f"unknown layout {layout!r}")

    @classmethod
    def from_reference(cls, p, device="cuda"):
        """Device copy of an mdtune.particles.ParticleSet (or any duck-alike)."""
        types = [ParticleTypeInfo(t.type_id, t.epsilon, t.sigma, t.mass) for t in p.types]
        out = cls(np.asarray(p.positions), np.asarray(p.velocities), np.asarray(p.type_id),
                  types, device=device)
        out.force.copy_(torch.as_tensor(np.ascontiguousarray(p.forces)))
        out.old_force.copy_(torch.as_tensor(np.ascontiguousarray(p.old_forces)))
        out.convert_layout(p.layout)
        return out

    @property
    def n(self) -> int:
        return int(self.type_id.shape[0])

    @property
    def ntypes(self) -> int:
        return len(self.mass)

    def convert_layout(self, target: str) -> "ParticleSet":
        if target not in (AOS, SOA):
            raise ValueError(f"unknown layout {target!r}")
        if target == self.layout:
            return self
        for name in _ATTRS:
            setattr(self, name, getattr(self, name).t().contiguous())
        self.layout = target
        return self

    def view(self, name: str) -> torch.Tensor:
        a = getattr(self, name)
        return a if self.layout == AOS else a.t()

    positions = property(lambda self: self.view("pos"))
    velocities = property(lambda self: self.view("vel"))
    forces = property(lambda self: self.view("force"))
    old_forces = property(lambda self: self.view("old_force"))

    @property
    def masses(self) -> torch.Tensor:
        m = torch.as_tensor(self.mass, dtype=torch.float64, device=self.device)
        return m[self.type_id.long()]

    def numpy(self, name: str) -> np.ndarray:
        """(N, 3) host copy of an attribute."""
        return self.view(name).detach().cpu().numpy().copy()

    def copy(self) -> "ParticleSet":
        out = ParticleSet.__new__(ParticleSet)
        out.device = self.device
        out.types = list(self.types)
        out.epsilon, out.sigma, out.mass = self.epsilon.copy(), self.sigma.copy(), self.mass.copy()
        out.layout = self.layout
        for name in _ATTRS + ("type_id",):
            setattr(out, name, getattr(self, name).clone())
        return out
