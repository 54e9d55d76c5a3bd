"""Worker for the multi-process domain-decomposition tests (gloo, CPU).

Every rank builds the same global seeded system, keeps the particles of its
slab, runs the decomposed reference loop with the oracle's brute-force forces
as the backend, and rank 0 gathers (id, position, velocity) into ``out_path``.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import port  # noqa: E402

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200.decomp import DecomposedSimulation, GridDecomposition  # noqa: E402

SIZES = {"small": (6, 6, 9), "cube10": (10, 10, 10)}


def system(seed=3, vscale=0.8, size="small"):
    """Jittered lattice with spacing 1.4 in a periodic box: "small" 6x6x9
    (8.4 x 8.4 x 12.6), "cube10" 10x10x10 (14^3, room for a 2x2x2 grid)."""
    rng = np.random.default_rng(seed)
    a = 1.4
    nx, ny, nz = SIZES[size]
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    pos = (g + 0.5) * a + rng.uniform(-0.1, 0.1, g.shape)
    vel = rng.normal(0.0, vscale, pos.shape)
    vel -= vel.mean(0)
    L = np.array([nx * a, ny * a, nz * a])
    return pos, vel, L


def thermostat():
    return P.ThermostatParams(0.9, 0.05, 3)


def oracle_force_fn(pos_all, type_all, n_owned, local_params, rebuild):
    f, _ = port.brute_forces(pos_all.numpy(), type_all.numpy().astype(np.int64), [1.0], [1.0],
                             local_params.cutoff, local_params.domain_size,
                             local_params.periodic_flags())
    return torch.as_tensor(f[:n_owned])


TUNED_SPACE = ["VL-List_Iter-NoN3L-SoA", "LC-C08-N3L-AoS-CSF1", "LC-SLI-N3L-SoA-CSF0.5",
               "VCL-ClusterIter-NoN3L-AoS", "LC-C01-NoN3L-SoA-CSF1"]


class RankScript:
    """A per-rank controller (TuningController protocol, tuning.py:200-239):
    a trial phase over five configurations rotated by rank (two samples
    each, the first forcing a rebuild, layouts switching), then the rank's
    own steady choice -- so the ranks run different configurations at the
    same iteration, as per-rank tuners do."""

    def __init__(self, rank):
        ids = TUNED_SPACE[rank % 5:] + TUNED_SPACE[:rank % 5]
        self.seq = [(c, s == 0, "trial") for c in ids for s in range(2)]
        self.steady = ids[-1]
        self.mode = "steady"
        self.timings = []

    def configuration_for_iteration(self, it):
        cid, forced, self.mode = self.seq[it] if it < len(self.seq) else (self.steady, False, "steady")
        return P.parse_configuration(cid), forced

    def record_timings(self, force_ns, build_ns):
        assert self.mode == "trial" and force_ns > 0 and build_ns > 0
        self.timings.append((force_ns, build_ns))

    def record_failure(self, error=None):
        return False


def run(rank, world, port_no, steps, out_path, vscale=0.8, dt=2e-3, backend="oracle",
        dims=None, size="small", thermo=False):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, vel, L = system(vscale=vscale, size=size)
    params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4,
                                delta_t=dt, boundary=(P.PERIODIC,) * 3,
                                thermostat=thermostat() if thermo else None)
    dec = GridDecomposition(params, rank, world, dims or (1, 1, world))
    mine = np.flatnonzero(dec.owner_of_positions(pos) == rank)
    if backend in ("gpudev", "gpudev_tuned"):   # the device-resident decomposition (bench's N > 1 path)
        from paper_2505_03438_b200.decomp import DeviceDecomposedSimulation
        cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA" if world % 2 == 0 else
                                    "VL-List_Iter-NoN3L-AoS")
        parts = P.ParticleSet(pos[mine], vel[mine], device="cuda:0")
        ctl = RankScript(rank) if backend == "gpudev_tuned" else None
        sim = DeviceDecomposedSimulation(dec, parts, params, cfg, comm_device="cpu",
                                         ids=torch.as_tensor(mine), controller=ctl)
        sim.run(steps)
        sim.check()
        if ctl is not None:
            assert len(ctl.timings) == len(ctl.seq) == len(sim.trial_log)
        sim.pos, sim.vel, sim.ids = sim.owned("pos").cpu(), sim.owned("vel").cpu(), sim.ids.cpu()
    elif backend == "gpu":   # libmdg on the (single) GPU, messages staged on the host for gloo
        from paper_2505_03438_b200.decomp import gpu_force_backend
        dev = torch.device("cuda", 0)
        fn = gpu_force_backend(P.parse_configuration("VL-List_Iter-NoN3L-AoS"), [1.0], [1.0], [1.0])
        comm = "cpu"
    else:
        dev, fn, comm = torch.device("cpu"), oracle_force_fn, None
    if backend not in ("gpudev", "gpudev_tuned"):
        sim = DecomposedSimulation(dec, torch.as_tensor(pos[mine]).to(dev), torch.as_tensor(vel[mine]).to(dev),
                                   torch.zeros(len(mine), dtype=torch.int64, device=dev), [1.0], params,
                                   fn, ids=torch.as_tensor(mine).to(dev), comm_device=comm)
        sim.run(steps)
        sim.pos, sim.vel, sim.ids = sim.pos.cpu(), sim.vel.cpu(), sim.ids.cpu()
    payload = torch.cat([sim.ids.to(torch.float64).unsqueeze(1), sim.pos, sim.vel,
                         torch.full((sim.pos.shape[0], 1), float(rank), dtype=torch.float64)], 1)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([payload.shape[0]]))
    mx = int(max(s.item() for s in sizes))
    padded = torch.zeros((mx, 8), dtype=torch.float64)
    padded[:payload.shape[0]] = payload
    bufs = [torch.zeros((mx, 8), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(bufs, padded)
    if rank == 0:
        rows = torch.cat([b[:int(s.item())] for b, s in zip(bufs, sizes)], 0).numpy()
        rows = rows[np.argsort(rows[:, 0])]
        np.save(out_path, rows)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    r, w, pn, st, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    vs = float(sys.argv[6]) if len(sys.argv) > 6 else 0.8
    dt = float(sys.argv[7]) if len(sys.argv) > 7 else 2e-3
    be = sys.argv[8] if len(sys.argv) > 8 else "oracle"
    dims = tuple(int(x) for x in sys.argv[9].split("x")) if len(sys.argv) > 9 and sys.argv[9] != "-" else None
    size = sys.argv[10] if len(sys.argv) > 10 else "small"
    th = len(sys.argv) > 11 and sys.argv[11] == "1"
    run(r, w, pn, st, out, vs, dt, be, dims, size, th)
