"""Spatial domain decomposition across ranks.

One process per GPU.  The box is cut into a ``px x py x pz`` grid of
subdomains (z-slabs for BASELINE configs 3 and 4, 3-D grids for config 5);
each rank owns the particles whose coordinates lie in its subdomain
``[lo, hi)`` and, every step, receives *ghost* copies of the particles within
ℓ = rc + skin of its faces.  Ghosts travel axis by axis (x, then y, then z),
each axis forwarding the ghosts received on the previous ones, so edge and
corner neighbours arrive without diagonal messages.  Ghost sets are chosen at
each rebuild and refreshed every step (the decomposed analogue of the
reference's periodic images, which are also fixed between rebuilds,
containers.py:93-118); particles that left their subdomain migrate, again axis
by axis, at each rebuild with their full state.  Forces are evaluated on
``owned + ghost`` particles as an open box along every decomposed axis (no
images on those axes, the ghosts stand in for them) and kept for owned
particles only, so there is no reverse force exchange.  The thermostat's
temperature is an all-reduce of the ranks' kinetic energies and counts.

The exchange is point-to-point through ``torch.distributed`` (NCCL between GPUs
over NVLink/NVSwitch, gloo on CPU for tests): counts first, then payloads, to
the two neighbours of each decomposed axis.  The force backend is pluggable
(``force_fn``): on GPUs it is libmdg (``gpu_force_backend``); tests pass the
CPU oracle.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .params import PERIODIC, REFLECTIVE, SimulationParams


class GridDecomposition:
    """A ``dims = (px, py, pz)`` process grid over the box; rank r sits at
    ``(r // (py*pz), (r // pz) % py, r % pz)``."""

    def __init__(self, params: SimulationParams, rank: int, world: int, dims=None):
        dims = tuple(int(d) for d in (dims or (1, 1, world)))
        if len(dims) != 3 or int(np.prod(dims)) != world:
            raise ValueError(f"process grid {dims} does not have {world} ranks")
        self.params, self.rank, self.world, self.dims = params, rank, world, dims
        self.coords = (rank // (dims[1] * dims[2]), (rank // dims[2]) % dims[1], rank % dims[2])
        self.ell = params.interaction_length
        per = params.periodic_flags()
        self.L = [float(x) for x in params.domain_size]
        self.periodic = [bool(per[a]) for a in range(3)]
        self.width = [self.L[a] / dims[a] for a in range(3)]
        self.lo = [self.coords[a] * self.width[a] for a in range(3)]
        self.hi = [self.L[a] if self.coords[a] == dims[a] - 1 else self.lo[a] + self.width[a]
                   for a in range(3)]
        self.active = [dims[a] > 1 for a in range(3)]
        self.left, self.right, self.has_left, self.has_right = [], [], [], []
        for a in range(3):
            c = list(self.coords)
            c[a] = (self.coords[a] - 1) % dims[a]
            self.left.append(self.rank_of(c))
            c[a] = (self.coords[a] + 1) % dims[a]
            self.right.append(self.rank_of(c))
            self.has_left.append(self.active[a] and (self.periodic[a] or self.coords[a] > 0))
            self.has_right.append(self.active[a] and (self.periodic[a] or self.coords[a] < dims[a] - 1))
            if self.active[a]:
                if self.width[a] < self.ell:
                    raise ValueError(f"subdomain width {self.width[a]} < interaction length {self.ell}")
                if self.periodic[a] and self.width[a] + 2.0 * self.ell >= self.L[a]:
                    raise ValueError("periodic axis too short for this process grid "
                                     "(width + 2 ell must stay below the box length)")

    def rank_of(self, c) -> int:
        return (int(c[0]) * self.dims[1] + int(c[1])) * self.dims[2] + int(c[2])

    def owner_of_positions(self, pos: np.ndarray) -> np.ndarray:
        pos = np.asarray(pos, dtype=np.float64)
        c = [np.clip(np.floor(pos[:, a] / self.width[a]).astype(np.int64), 0, self.dims[a] - 1)
             for a in range(3)]
        return (c[0] * self.dims[1] + c[1]) * self.dims[2] + c[2]

    def local_params(self) -> SimulationParams:
        """Open box [lo - ell, hi + ell) along every decomposed axis (coordinates
        shifted by -(lo - ell)), the other axes unchanged."""
        p = self.params
        if self.world == 1:
            return p
        dom = np.array(p.domain_size, dtype=np.float64)
        bnd = list(p.boundary)
        for a in range(3):
            if self.active[a]:
                dom[a] = (self.hi[a] - self.lo[a]) + 2.0 * self.ell
                bnd[a] = REFLECTIVE
        return SimulationParams(domain_size=dom, cutoff=p.cutoff, skin=p.skin,
                                rebuild_interval=p.rebuild_interval, delta_t=p.delta_t,
                                boundary=tuple(bnd), gravity=p.gravity)

    def origin(self, a: int) -> float:
        return self.lo[a] - self.ell if self.active[a] else 0.0

    def near(self, x, a: int):
        """Periodic image of coordinate(s) ``x`` along axis ``a`` nearest to the
        subdomain centre (continuous local frame for particles that wrapped
        across the box face since the last rebuild)."""
        if not self.periodic[a] or not self.active[a]:
            return x
        c = 0.5 * (self.lo[a] + self.hi[a])
        return x - self.L[a] * torch.round((x - c) / self.L[a])


class SlabDecomposition(GridDecomposition):
    """Slabs along one axis (BASELINE configs 3 and 4)."""

    def __init__(self, params: SimulationParams, rank: int, world: int, axis: int = 2):
        dims = [1, 1, 1]
        dims[axis] = world
        super().__init__(params, rank, world, dims)
        self.axis = axis

    def owner_of(self, coord: np.ndarray) -> np.ndarray:
        r = np.floor(np.asarray(coord) / self.width[self.axis]).astype(np.int64)
        return np.clip(r, 0, self.world - 1)


def _exchange(tensor_left, tensor_right, dec: GridDecomposition, a: int, width: int, dtype,
              comm_device=None):
    """Send rows to the two neighbours along axis ``a``, receive theirs.
    Returns (from_left, from_right) on the device of the inputs.
    ``comm_device`` stages the messages elsewhere (e.g. "cpu" for gloo with
    device tensors)."""
    home = tensor_left.device
    if comm_device is not None:
        tensor_left, tensor_right = tensor_left.to(comm_device), tensor_right.to(comm_device)
    dev = tensor_left.device
    counts_out = [torch.tensor([tensor_left.shape[0]], device=dev),
                  torch.tensor([tensor_right.shape[0]], device=dev)]
    counts_in = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(2)]
    ops = []
    if dec.has_left[a]:
        ops += [dist.P2POp(dist.isend, counts_out[0], dec.left[a]),
                dist.P2POp(dist.irecv, counts_in[0], dec.left[a])]
    if dec.has_right[a]:
        ops += [dist.P2POp(dist.isend, counts_out[1], dec.right[a]),
                dist.P2POp(dist.irecv, counts_in[1], dec.right[a])]
    for req in dist.batch_isend_irecv(ops) if ops else []:
        req.wait()
    recv = [torch.empty((int(c.item()), width), dtype=dtype, device=dev) for c in counts_in]
    ops = []
    if dec.has_left[a]:
        ops += [dist.P2POp(dist.isend, tensor_left.contiguous(), dec.left[a]),
                dist.P2POp(dist.irecv, recv[0], dec.left[a])]
    if dec.has_right[a]:
        ops += [dist.P2POp(dist.isend, tensor_right.contiguous(), dec.right[a]),
                dist.P2POp(dist.irecv, recv[1], dec.right[a])]
    for req in dist.batch_isend_irecv(ops) if ops else []:
        req.wait()
    return recv[0].to(home), recv[1].to(home)


class DecomposedSimulation:
    """The reference loop (simulation.py:150-188) on one rank of a grid
    decomposition.  State arrays are (n_local, 3) fp64 torch tensors on the
    rank's device; ``force_fn(pos_all, type_all, n_owned, local_params,
    rebuild)`` returns the forces on the first ``n_owned`` rows of ``pos_all``
    (local coordinates)."""

    def __init__(self, dec: GridDecomposition, pos, vel, type_id, mass, params, force_fn, ids=None,
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
        self.plan = []   # per decomposed axis: (axis, left rows, right rows) of the combined set

    # -- exchange ------------------------------------------------------------
    def _ghosts(self, replan: bool):
        """Owned + ghost positions and types, axis by axis.  ``replan`` (rebuild
        time) selects the rows within ell of each face; otherwise the stored
        selection is re-sent with current positions."""
        d = self.dec
        cpos, ctype = self.pos, self.type_id
        plan = [] if replan else self.plan
        for k, a in enumerate(x for x in range(3) if d.active[x]):
            if replan:
                z = d.near(cpos[:, a], a)
                none = z.new_zeros(0, dtype=torch.long)
                left = torch.nonzero(z < d.lo[a] + d.ell).flatten() if d.has_left[a] else none
                right = torch.nonzero(z >= d.hi[a] - d.ell).flatten() if d.has_right[a] else none
                plan.append((a, left, right))
            else:
                _, left, right = plan[k]
            pl, pr = cpos[left], cpos[right]
            tl = ctype[left].to(pl.dtype).unsqueeze(1)
            tr = ctype[right].to(pr.dtype).unsqueeze(1)
            gl, gr = _exchange(torch.cat([pl, tl], 1), torch.cat([pr, tr], 1), d, a, 4, pl.dtype,
                               self.comm_device)
            g = torch.cat([gl, gr], 0)
            cpos = torch.cat([cpos, g[:, :3]], 0)
            ctype = torch.cat([ctype, g[:, 3].to(ctype.dtype)], 0)
        if replan:
            self.plan = plan
        return cpos, ctype

    def _migrate(self):
        """Particles that left [lo, hi) go to the neighbours, axis by axis, with
        their full state."""
        d = self.dec
        for a in range(3):
            if not d.active[a]:
                continue
            z = d.near(self.pos[:, a], a)
            go_left = z < d.lo[a]
            go_right = z >= d.hi[a]
            if d.coords[a] == 0 and not d.periodic[a]:
                go_left = torch.zeros_like(go_left)
            if d.coords[a] == d.dims[a] - 1 and not d.periodic[a]:
                go_right = torch.zeros_like(go_right)
            stay = ~(go_left | go_right)
            pack = lambda m: torch.cat([self.pos[m], self.vel[m], self.force[m], self.old_force[m],
                                        self.type_id[m].to(self.pos.dtype).unsqueeze(1),
                                        self.ids[m].to(self.pos.dtype).unsqueeze(1)], 1)
            fl, fr = _exchange(pack(go_left), pack(go_right), d, a, 14, self.pos.dtype,
                               self.comm_device)
            inc = torch.cat([fl, fr], 0)
            self.pos = torch.cat([self.pos[stay], inc[:, 0:3]], 0)
            self.vel = torch.cat([self.vel[stay], inc[:, 3:6]], 0)
            self.force = torch.cat([self.force[stay], inc[:, 6:9]], 0)
            self.old_force = torch.cat([self.old_force[stay], inc[:, 9:12]], 0)
            self.type_id = torch.cat([self.type_id[stay], inc[:, 12].to(self.type_id.dtype)], 0)
            self.ids = torch.cat([self.ids[stay], inc[:, 13].to(self.ids.dtype)], 0)

    def _thermostat(self, target, max_delta_t):
        """apply_thermostat (integrator.py:81-95) with the temperature reduced
        over all ranks (sum of m|v|^2 and of the particle counts)."""
        m = self.mass[self.type_id.long()]
        ke = torch.sum(m * torch.sum(self.vel * self.vel, dim=1)).to(torch.float64)
        red = torch.stack([ke, torch.tensor(float(self.pos.shape[0]), dtype=torch.float64,
                                            device=ke.device)])
        if self.dec.world > 1:
            home = red.device
            red = red.to(self.comm_device) if self.comm_device is not None else red
            dist.all_reduce(red)
            red = red.to(home)
        ke, n = float(red[0]), float(red[1])
        if n == 0:
            raise ValueError("temperature of an empty particle set is undefined")
        t_cur = ke / (3.0 * n)
        if t_cur == 0.0:
            if target > 0.0:
                raise ValueError("thermostat cannot scale zero velocities toward a positive "
                                 "target temperature")
            return
        delta = min(max(target - t_cur, -max_delta_t), max_delta_t)
        self.vel = self.vel * float(np.sqrt((t_cur + delta) / t_cur))

    # -- the loop ------------------------------------------------------------
    def step(self):
        p, dt = self.params, self.params.delta_t
        d = self.dec
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
            m = self.mass[self.type_id.long()].unsqueeze(1)
        pos_all, type_all = self._ghosts(replan=rebuild)
        n = self.pos.shape[0]
        pos_all = pos_all.clone()
        for a in range(3):
            if d.active[a]:
                pos_all[:, a] = d.near(pos_all[:, a], a) - d.origin(a)
        self.force = self.force_fn(pos_all, type_all, n, self.local_params, rebuild)
        if p.gravity is not None:
            self.force[:, 2] += m[:, 0] * p.gravity
        self.vel = self.vel + (self.force + self.old_force) * (0.5 * dt / m)
        thermo = getattr(p, "thermostat", None)
        if thermo is not None and (self.iteration + 1) % thermo.interval_iterations == 0:
            self._thermostat(thermo.target_temperature, thermo.max_delta_t)
        self.since = 0 if rebuild else self.since + 1
        self.iteration += 1

    def run(self, steps):
        for _ in range(steps):
            self.step()


def gpu_force_backend(config, sigma, epsilon, mass):
    """libmdg as the per-rank force backend (owned + ghost rows, open box along
    the decomposed axes).

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


# ---------------------------------------------------------------------------
# Device-resident decomposition (the bench's N > 1 path)
# ---------------------------------------------------------------------------

def _device_set(template, pos, vel, force, old_force, type_id, layout):
    """ParticleSet over the given (n, 3) device tensors without a host round
    trip (types, masses and parameters from ``template``)."""
    from .particles import AOS, ParticleSet
    out = ParticleSet.__new__(ParticleSet)
    out.device = pos.device
    out.types = list(template.types)
    out.epsilon, out.sigma, out.mass = template.epsilon, template.sigma, template.mass
    out.layout = AOS
    out.pos, out.vel = pos.contiguous(), vel.contiguous()
    out.force, out.old_force = force.contiguous(), old_force.contiguous()
    out.type_id = type_id.to(torch.int32).contiguous()
    out.convert_layout(layout)
    return out


class DeviceDecomposedSimulation:
    """The reference loop (simulation.py:150-188, fixed configuration) on one
    rank of a grid decomposition with everything on the device: libmdg's
    drift / force / kick kernels and ``torch.distributed`` point-to-point
    (NCCL over NVLink between GPUs) for the ghosts.

    Each rank keeps ONE device ParticleSet in its LOCAL frame (origin
    ``lo - ell`` along every decomposed axis; the local box is open there and
    periodic along the others): rows ``[0, n_owned)`` are its particles, the
    rows after them the ghosts of the current rebuild interval, in exchange
    order.  A step is

      drift (all rows) -> [rebuild: migrate, new ghost plan] -> ghost
      positions (gather, shift by the slab width, send/recv straight into
      the ghost rows; sizes fixed between rebuilds, so no count exchange and
      no host synchronisation) -> refresh + compute -> kick,

    forces of owned rows kept, no reverse exchange.  Ghost
    rows are drifted and kicked with the rest (their positions are replaced
    by the exchange before every force pass; their velocities are unused).
    All axes must be periodic (BASELINE configs 2-5)."""

    def __init__(self, dec: GridDecomposition, particles, params: SimulationParams, config,
                 comm_device=None, ids=None, controller=None):
        from .calculator import ForceCalculator
        per = params.periodic_flags()
        if not all(bool(x) for x in per):
            raise ValueError("the device decomposition needs periodic boundaries on every axis")
        self.dec, self.params, self.config = dec, params, config
        self.comm_device = comm_device
        self.local_params = dec.local_params()
        self.template = particles
        d = particles.device
        pos = particles.view("pos").clone()
        for a in range(3):
            if dec.active[a]:
                pos[:, a] = dec.near(pos[:, a], a) - dec.origin(a)
        self.n_owned = pos.shape[0]
        self.ids = (torch.arange(self.n_owned, device=pos.device) if ids is None
                    else torch.as_tensor(ids, device=pos.device).clone())
        self.ps = _device_set(particles, pos, particles.view("vel").clone(),
                              particles.view("force").clone(), particles.view("old_force").clone(),
                              particles.type_id.clone(), config.layout)
        self.calc = ForceCalculator(self.ps, self.local_params)
        self.axes = [a for a in range(3) if dec.active[a]]
        self.plan = []          # per active axis: (axis, left idx, right idx, recv_l, recv_r, row0)
        self.iteration, self.since = 0, 0
        self._kick_due = False
        self.dev = d
        # per-rank tuning (the paper's setup: one tuner per rank):
        # any TuningController-protocol object; its trials rebuild this rank's
        # container locally, the decomposition (migration, ghost plan) keeps
        # the global R+1 cadence every rank shares
        self.controller = controller
        self.active = None
        self.trial_log = []     # (iteration, configuration id, force_ns, build_ns)

    # -- point-to-point -----------------------------------------------------
    def _p2p(self, a, send_l, send_r, recv_l, recv_r):
        d = self.dec
        cd = self.comm_device
        if cd is not None:
            send_l, send_r = send_l.to(cd), send_r.to(cd)
            bl, br = recv_l.to(cd), recv_r.to(cd)
        else:
            bl, br = recv_l, recv_r
        ops = []
        if d.has_left[a]:
            ops += [dist.P2POp(dist.isend, send_l.contiguous(), d.left[a]),
                    dist.P2POp(dist.irecv, bl, d.left[a])]
        if d.has_right[a]:
            ops += [dist.P2POp(dist.isend, send_r.contiguous(), d.right[a]),
                    dist.P2POp(dist.irecv, br, d.right[a])]
        for req in dist.batch_isend_irecv(ops) if ops else []:
            req.wait()
        if cd is not None:
            recv_l.copy_(bl)
            recv_r.copy_(br)

    def _counts(self, a, nl, nr):
        t_out_l = torch.tensor([nl], dtype=torch.int64, device=self.dev)
        t_out_r = torch.tensor([nr], dtype=torch.int64, device=self.dev)
        t_in_l = torch.zeros(1, dtype=torch.int64, device=self.dev)
        t_in_r = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self._p2p(a, t_out_l, t_out_r, t_in_l, t_in_r)
        return int(t_in_l.item()), int(t_in_r.item())

    # -- rebuild-time work --------------------------------------------------
    def _owned_state(self):
        n, ps = self.n_owned, self.ps
        return [ps.view("pos")[:n].clone(), ps.view("vel")[:n].clone(),
                ps.view("force")[:n].clone(), ps.view("old_force")[:n].clone(),
                ps.type_id[:n].to(torch.float64).unsqueeze(1),
                self.ids.to(torch.float64).unsqueeze(1)]

    def _migrate(self, st):
        """Owned rows outside [ell, ell + w) along a decomposed axis go to that
        neighbour with their full state, axis by axis (frame shift +-w)."""
        d, ell = self.dec, self.dec.ell
        for a in self.axes:
            w = d.width[a]
            z = st[0][:, a]
            go_l = (z < ell) if d.has_left[a] else torch.zeros_like(z, dtype=torch.bool)
            go_r = (z >= ell + w) if d.has_right[a] else torch.zeros_like(z, dtype=torch.bool)
            stay = ~(go_l | go_r)
            pack = lambda m: torch.cat([s[m] for s in st], 1)
            pl, pr = pack(go_l), pack(go_r)
            pl[:, a] += w      # into the left neighbour's frame
            pr[:, a] -= w
            nl, nr = self._counts(a, pl.shape[0], pr.shape[0])
            rl = torch.empty((nl, 14), dtype=torch.float64, device=self.dev)
            rr = torch.empty((nr, 14), dtype=torch.float64, device=self.dev)
            self._p2p(a, pl, pr, rl, rr)
            inc = torch.cat([rl, rr], 0)
            cols = [(0, 3), (3, 6), (6, 9), (9, 12), (12, 13), (13, 14)]
            st = [torch.cat([s[stay], inc[:, c0:c1]], 0) for s, (c0, c1) in zip(st, cols)]
        return st

    def _replan(self, st):
        """Ghost selection, axis by axis over owned + the ghosts of the earlier
        axes: rows within ell of the low face go left, of the high face right."""
        d, ell = self.dec, self.dec.ell
        pos = st[0]
        tcol = st[4]
        plan = []
        for a in self.axes:
            w = d.width[a]
            z = pos[:, a]
            none = torch.zeros(0, dtype=torch.long, device=self.dev)
            li = torch.nonzero(z < 2.0 * ell).flatten() if d.has_left[a] else none
            ri = torch.nonzero(z >= w).flatten() if d.has_right[a] else none
            nl, nr = self._counts(a, li.numel(), ri.numel())
            row0 = pos.shape[0]
            # the types travel once per rebuild; positions every step (_ghosts)
            sl = torch.cat([pos[li], tcol[li]], 1)
            sr = torch.cat([pos[ri], tcol[ri]], 1)
            sl[:, a] += w
            sr[:, a] -= w
            rl = torch.empty((nl, 4), dtype=torch.float64, device=self.dev)
            rr = torch.empty((nr, 4), dtype=torch.float64, device=self.dev)
            self._p2p(a, sl, sr, rl, rr)
            g = torch.cat([rl, rr], 0)
            pos = torch.cat([pos, g[:, :3]], 0)
            tcol = torch.cat([tcol, g[:, 3:4]], 0)
            plan.append((a, torch.cat([li, ri]).to(torch.int64).contiguous(), li.numel(), nl, nr, row0))
        return plan, pos, tcol

    def _rebuild(self, cfg=None):
        cfg = cfg or self.config
        st = self._migrate(self._owned_state())
        n = st[0].shape[0]
        plan, pos, tcol = self._replan(st)
        m = pos.shape[0]
        z = torch.zeros((m - n, 3), dtype=torch.float64, device=self.dev)
        self.n_owned, self.plan = n, plan
        self.ids = st[5][:, 0].to(torch.int64)
        self.ps = _device_set(self.template, pos, torch.cat([st[1], z], 0),
                              torch.cat([st[2], z], 0), torch.cat([st[3], z], 0),
                              tcol[:, 0].to(torch.int32), cfg.layout)
        # per axis: one AoS send buffer (left part, right part) packed by
        # libmdg, one receive buffer (unused for AoS rows: received in place)
        self._bufs = [(torch.empty((idx.numel(), 3), dtype=torch.float64, device=self.dev),
                       torch.empty((nl + nr, 3), dtype=torch.float64, device=self.dev))
                      for a, idx, nsl, nl, nr, row0 in self.plan]
        # ghost rows (particle index >= n_owned) need no forces of their own
        self.calc.set_force_rows(n)
        self.calc.rebuild(self.ps, cfg)

    # -- per step -----------------------------------------------------------
    def _ghosts(self):
        """Ghost positions of the fixed plan, axis by axis: libmdg packs the
        left and right rows (shifted into the neighbours' frames) into one
        send buffer; the receive lands in the ghost rows (AoS: in place;
        SoA: a staging buffer + one unpack launch)."""
        aos = self.ps.layout == "AoS"
        for (a, idx, nsl, nl, nr, row0), (sbuf, rbuf) in zip(self.plan, self._bufs):
            w = self.dec.width[a]
            self.calc.ghost_pack(self.ps, idx, nsl, a, w, -w, sbuf)
            dst = self.ps.pos[row0:row0 + nl + nr] if aos else rbuf
            self._p2p(a, sbuf[:nsl], sbuf[nsl:], dst[:nl], dst[nl:])
            if not aos:
                self.calc.ghost_unpack(self.ps, rbuf, row0)

    def step(self):
        """One iteration; its kick is deferred into the next step's drift
        (mdg_kick_drift, force / old_force swapped) -- flush() completes it.
        With a controller, its configuration for this iteration is used; a
        trial's first sample or a configuration change rebuilds this rank's
        container (locally), and trial iterations hand device-event build /
        force nanoseconds to ``record_timings`` (simulation.py:155-181)."""
        p, calc = self.params, self.calc
        it, ctl = self.iteration, self.controller
        if ctl is not None:
            cfg, forced = ctl.configuration_for_iteration(it)
            trial = getattr(ctl, "mode", "steady") == "trial"
        else:
            cfg, forced, trial = self.config, False, False
        if self._kick_due:
            calc.kick_drift(self.ps, p.delta_t, p.gravity, copy_old_force=False)
            self.ps.force, self.ps.old_force = self.ps.old_force, self.ps.force
            self._kick_due = False
        else:
            calc.drift_wrap(self.ps, p.delta_t)
        if trial:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
        if self.ps.layout != cfg.layout:
            self.ps.convert_layout(cfg.layout)
        rebuild = self.iteration == 0 or self.since >= p.rebuild_interval
        if rebuild:
            self._rebuild(cfg)
        else:
            self._ghosts()
            if forced or cfg.id != self.active:
                calc.rebuild(self.ps, cfg)
        calc.refresh(self.ps, cfg)
        if trial:
            ev[1].record()
        calc.compute_async(self.ps, cfg)
        if trial:
            ev[2].record()
            ev[2].synchronize()
            build_ns = int(ev[0].elapsed_time(ev[1]) * 1e6)
            force_ns = int(ev[1].elapsed_time(ev[2]) * 1e6)
            ctl.record_timings(force_ns, build_ns)
            self.trial_log.append((it, cfg.id, force_ns, build_ns))
        self.active = cfg.id
        thermo = getattr(p, "thermostat", None)
        if thermo is not None and (self.iteration + 1) % thermo.interval_iterations == 0:
            calc.finish_kick(self.ps, p.delta_t, p.gravity)   # the thermostat needs the kicked state
            self._thermostat(thermo.target_temperature, thermo.max_delta_t)
        else:
            self._kick_due = True
        self.since = 0 if rebuild else self.since + 1
        self.iteration += 1

    def run(self, steps):
        for _ in range(steps):
            self.step()
        self.flush()

    def _thermostat(self, target, max_delta_t):
        """apply_thermostat (integrator.py:81-95) over the owned rows of every
        rank: the kinetic energy and the particle count are all-reduced."""
        n = self.n_owned
        v = self.ps.view("vel")[:n]
        mass = torch.as_tensor(np.asarray(self.template.mass, dtype=np.float64), device=self.dev)
        m = mass[self.ps.type_id[:n].long()]
        red = torch.stack([torch.sum(m * torch.sum(v * v, dim=1)),
                           torch.tensor(float(n), dtype=torch.float64, device=self.dev)])
        if self.dec.world > 1:
            buf = red.to(self.comm_device) if self.comm_device is not None else red
            dist.all_reduce(buf)
            red = buf.to(self.dev)
        ke, cnt = float(red[0]), float(red[1])
        if cnt == 0:
            raise ValueError("temperature of an empty particle set is undefined")
        t_cur = ke / (3.0 * cnt)
        if t_cur == 0.0:
            if target > 0.0:
                raise ValueError("thermostat cannot scale zero velocities toward a positive "
                                 "target temperature")
            return
        delta = min(max(target - t_cur, -max_delta_t), max_delta_t)
        v.mul_(float(np.sqrt((t_cur + delta) / t_cur)))

    def flush(self):
        """Run the deferred kick of the last step (state complete again)."""
        if self._kick_due:
            self.calc.finish_kick(self.ps, self.params.delta_t, self.params.gravity)
            self._kick_due = False

    def check(self):
        from .simulation import BlowUpError
        self.flush()
        if self.calc.blowup():
            raise BlowUpError("particle left the domain by more than one domain length "
                              "(or position is not finite)")

    def owned(self, name):
        """(n_owned, 3) of pos (GLOBAL frame, wrapped), vel, force, old_force."""
        self.flush()
        v = self.ps.view(name)[:self.n_owned].clone()
        if name == "pos":
            for a in self.axes:
                v[:, a] = torch.remainder(v[:, a] + self.dec.origin(a), self.dec.L[a])
        return v
