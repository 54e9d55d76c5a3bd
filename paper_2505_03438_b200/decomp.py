"""Spatial domain decomposition across ranks.

One process per GPU.  The box is cut into slabs along one axis; each rank owns
the particles whose coordinate lies in its slab ``[lo, hi)`` and, every step,
receives *ghost* copies of the neighbours' particles that lie within
ℓ = rc + skin of its faces (positions only, with the global periodic shift
applied across the box boundary).  Ghost sets are chosen at each rebuild and
refreshed every step (the decomposed analogue of the reference's periodic
images, which are also fixed between rebuilds, containers.py:93-118); particles
that left their slab migrate to the neighbour at each rebuild with their full
state.  Forces are evaluated on ``owned + ghost`` particles as an open box along
the slab axis (no images on that axis, the ghosts stand in for them) and kept
for owned particles only, so there is no reverse force exchange.

The exchange is point-to-point through ``torch.distributed`` (NCCL between GPUs
over NVLink/NVSwitch, gloo on CPU for tests): counts first, then payloads, to the
left and right neighbours.  The force backend is pluggable (``force_fn``): on
GPUs it is libmdg (``gpu_force_backend``); tests pass the CPU oracle.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .params import PERIODIC, REFLECTIVE, SimulationParams


class SlabDecomposition:
    def __init__(self, params: SimulationParams, rank: int, world: int, axis: int = 2):
        self.params = params
        self.rank, self.world, self.axis = rank, world, axis
        L = float(params.domain_size[axis])
        self.L = L
        self.width = L / world
        self.lo = rank * self.width
        self.hi = L if rank == world - 1 else (rank + 1) * self.width
        self.ell = params.interaction_length
        self.periodic = bool(params.periodic_flags()[axis])
        if world > 1 and self.width < self.ell:
            raise ValueError(f"slab width {self.width} < interaction length {self.ell}")
        self.left = (rank - 1) % world
        self.right = (rank + 1) % world
        self.has_left = world > 1 and (self.periodic or rank > 0)
        self.has_right = world > 1 and (self.periodic or rank < world - 1)

    def owner_of(self, coord: np.ndarray) -> np.ndarray:
        r = np.floor(np.asarray(coord) / self.width).astype(np.int64)
        return np.clip(r, 0, self.world - 1)

    def local_params(self) -> SimulationParams:
        """Open box [lo - ell, hi + ell) along the slab axis (coordinates shifted
        by -(lo - ell)), the other axes unchanged."""
        p = self.params
        if self.world == 1:
            return p
        dom = np.array(p.domain_size, dtype=np.float64)
        dom[self.axis] = (self.hi - self.lo) + 2.0 * self.ell
        bnd = list(p.boundary)
        bnd[self.axis] = REFLECTIVE
        return SimulationParams(domain_size=dom, cutoff=p.cutoff, skin=p.skin,
                                rebuild_interval=p.rebuild_interval, delta_t=p.delta_t,
                                boundary=tuple(bnd), gravity=p.gravity)

    @property
    def origin(self) -> float:
        return self.lo - self.ell if self.world > 1 else 0.0

    def near(self, z):
        """Periodic image of z nearest to the slab centre (continuous local frame
        for particles that wrapped across the box face since the last rebuild)."""
        if not self.periodic or self.world == 1:
            return z
        c = 0.5 * (self.lo + self.hi)
        return z - self.L * torch.round((z - c) / self.L)


def _exchange(tensor_left, tensor_right, dec: SlabDecomposition, width: int, dtype,
              comm_device=None):
    """Send rows to the left/right neighbours, receive theirs.  Returns
    (from_left, from_right) on the device of the inputs.  ``comm_device``
    stages the messages elsewhere (e.g. "cpu" for gloo with device tensors)."""
    home = tensor_left.device
    if comm_device is not None:
        tensor_left, tensor_right = tensor_left.to(comm_device), tensor_right.to(comm_device)
    dev = tensor_left.device
    counts_out = [torch.tensor([tensor_left.shape[0]], device=dev),
                  torch.tensor([tensor_right.shape[0]], device=dev)]
    counts_in = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(2)]
    ops = []
    if dec.has_left:
        ops += [dist.P2POp(dist.isend, counts_out[0], dec.left),
                dist.P2POp(dist.irecv, counts_in[0], dec.left)]
    if dec.has_right:
        ops += [dist.P2POp(dist.isend, counts_out[1], dec.right),
                dist.P2POp(dist.irecv, counts_in[1], dec.right)]
    for req in dist.batch_isend_irecv(ops) if ops else []:
        req.wait()
    recv = [torch.empty((int(c.item()), width), dtype=dtype, device=dev) for c in counts_in]
    ops = []
    if dec.has_left:
        ops += [dist.P2POp(dist.isend, tensor_left.contiguous(), dec.left),
                dist.P2POp(dist.irecv, recv[0], dec.left)]
    if dec.has_right:
        ops += [dist.P2POp(dist.isend, tensor_right.contiguous(), dec.right),
                dist.P2POp(dist.irecv, recv[1], dec.right)]
    for req in dist.batch_isend_irecv(ops) if ops else []:
        req.wait()
    return recv[0].to(home), recv[1].to(home)


class DecomposedSimulation:
    """The reference loop (simulation.py:150-188) on one rank of a slab
    decomposition.  State arrays are (n_local, 3) fp64 torch tensors on the
    rank's device; ``force_fn(pos_all, type_all, n_owned, local_params)`` returns
    the forces on the first ``n_owned`` rows of ``pos_all`` (local coordinates).
    """

    def __init__(self, dec: SlabDecomposition, pos, vel, type_id, mass, params, force_fn, ids=None,
                 comm_device=None):
        self.dec, self.params, self.force_fn = dec, params, force_fn
        self.comm_device = comm_device
        self.ids = (torch.arange(pos.shape[0], device=pos.device) if ids is None else ids.clone())
        self.pos = pos.clone()
        self.vel = vel.clone()
        self.type_id = type_id.clone()
        self.mass = torch.as_tensor(np.asarray(mass, dtype=np.float64), device=pos.device)
        self.force = torch.zeros_like(pos)
        self.old_force = torch.zeros_like(pos)
        self.local_params = dec.local_params()
        self.since = 0
        self.iteration = 0
        self.ghost_idx = (None, None)

    # -- exchange ------------------------------------------------------------
    def _ghost_plan(self):
        """Owned particles within ell of the left / right face (rebuild time)."""
        d, ax = self.dec, self.dec.axis
        z = d.near(self.pos[:, ax])
        none = z.new_zeros(0, dtype=torch.long)
        left = torch.nonzero(z < d.lo + d.ell).flatten() if d.has_left else none
        right = torch.nonzero(z >= d.hi - d.ell).flatten() if d.has_right else none
        self.ghost_idx = (left, right)

    def _ghosts(self):
        left, right = self.ghost_idx
        pl, pr = self.pos[left], self.pos[right]
        tl = self.type_id[left].to(pl.dtype).unsqueeze(1)
        tr = self.type_id[right].to(pr.dtype).unsqueeze(1)
        gl, gr = _exchange(torch.cat([pl, tl], 1), torch.cat([pr, tr], 1), self.dec, 4, pl.dtype,
                           self.comm_device)
        g = torch.cat([gl, gr], 0)
        return g[:, :3].clone(), g[:, 3].to(self.type_id.dtype)

    def _migrate(self):
        """Particles that left [lo, hi) go to the neighbour with their state."""
        d, ax = self.dec, self.dec.axis
        if d.world == 1:
            return
        z = d.near(self.pos[:, ax])
        go_left = z < d.lo
        go_right = z >= d.hi
        if d.rank == 0 and not d.periodic:
            go_left = torch.zeros_like(go_left)
        if d.rank == d.world - 1 and not d.periodic:
            go_right = torch.zeros_like(go_right)
        stay = ~(go_left | go_right)
        pack = lambda m: torch.cat([self.pos[m], self.vel[m], self.force[m], self.old_force[m],
                                    self.type_id[m].to(self.pos.dtype).unsqueeze(1),
                                    self.ids[m].to(self.pos.dtype).unsqueeze(1)], 1)
        fl, fr = _exchange(pack(go_left), pack(go_right), d, 14, self.pos.dtype, self.comm_device)
        inc = torch.cat([fl, fr], 0)
        self.pos = torch.cat([self.pos[stay], inc[:, 0:3]], 0)
        self.vel = torch.cat([self.vel[stay], inc[:, 3:6]], 0)
        self.force = torch.cat([self.force[stay], inc[:, 6:9]], 0)
        self.old_force = torch.cat([self.old_force[stay], inc[:, 9:12]], 0)
        self.type_id = torch.cat([self.type_id[stay], inc[:, 12].to(self.type_id.dtype)], 0)
        self.ids = torch.cat([self.ids[stay], inc[:, 13].to(self.ids.dtype)], 0)

    # -- the loop ------------------------------------------------------------
    def step(self):
        p, dt = self.params, self.params.delta_t
        m = self.mass[self.type_id.long()].unsqueeze(1)
        # drift_with_force + boundaries + F -> F_old (integrator.py:31-37, 98-128)
        self.pos = self.pos + self.vel * dt
        self.pos = self.pos + self.force * (0.5 * dt * dt / m)
        L = torch.as_tensor(p.domain_size, dtype=self.pos.dtype, device=self.pos.device)
        for k in range(3):
            x = self.pos[:, k]
            if p.boundary[k] == PERIODIC:
                self.pos[:, k] = torch.remainder(x, L[k])
            else:
                lo, hi = x < 0, x > L[k]
                self.pos[:, k] = torch.where(lo, -x, torch.where(hi, 2 * L[k] - x, x))
                self.vel[:, k] = torch.where(lo | hi, -self.vel[:, k], self.vel[:, k])
        self.old_force = self.force.clone()
        rebuild = self.iteration == 0 or self.since >= p.rebuild_interval
        if rebuild:
            self._migrate()
            self._ghost_plan()
            m = self.mass[self.type_id.long()].unsqueeze(1)
        gpos, gtype = self._ghosts()
        n = self.pos.shape[0]
        pos_all = torch.cat([self.pos, gpos], 0)
        ax = self.dec.axis
        pos_all[:, ax] = self.dec.near(pos_all[:, ax]) - self.dec.origin
        type_all = torch.cat([self.type_id, gtype], 0)
        self.force = self.force_fn(pos_all, type_all, n, self.local_params, rebuild)
        if p.gravity is not None:
            self.force[:, 2] += m[:, 0] * p.gravity
        self.vel = self.vel + (self.force + self.old_force) * (0.5 * dt / m)
        self.since = 0 if rebuild else self.since + 1
        self.iteration += 1

    def run(self, steps):
        for _ in range(steps):
            self.step()


def gpu_force_backend(config, sigma, epsilon, mass):
    """libmdg as the per-rank force backend (owned + ghost rows, open slab box).

    The row set (owned + ghosts) is fixed between rebuilds, so the device
    ParticleSet and its neighbour structure are rebuilt only at rebuild steps;
    other steps copy the refreshed positions in and re-evaluate."""
    from .calculator import ForceCalculator
    from .particles import ParticleSet, ParticleTypeInfo
    types = [ParticleTypeInfo(t, float(epsilon[t]), float(sigma[t]), float(mass[t]))
             for t in range(len(mass))]
    state = {}

    def force_fn(pos_all, type_all, n_owned, local_params, rebuild):
        parts = state.get("parts")
        if rebuild or parts is None or parts.n != pos_all.shape[0]:
            parts = ParticleSet(pos_all, type_ids=type_all.cpu().numpy(), types=types,
                                device=pos_all.device)
            parts.convert_layout(config.layout)
            if "calc" in state:
                state["calc"].close()
            state["parts"], state["calc"] = parts, ForceCalculator(parts, local_params)
            state["calc"].rebuild(parts, config)
        else:
            parts.view("pos").copy_(pos_all)
        calc = state["calc"]
        calc.refresh(parts, config)
        calc.compute_async(parts, config)
        return parts.forces[:n_owned].clone()

    return force_fn
