"""Domain decomposition on CPU over gloo: z-slabs with 2
ranks (configs 3 / 4) and 2x2x1 / 2x2x2 process grids (config 5).

The decomposed loop (per-step ghost exchange axis by axis, migration at
rebuilds, the thermostat's all-reduced temperature) must reproduce the
single-rank run and the reference loop (oracle restatement of
simulation.py:126-197) on the same seeded system.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

WORKER = os.path.join(ROOT, "tests", "decomp_worker.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, steps, tmp_path, vscale=0.8, dt=2e-3, tag="", backend="oracle", dims=None,
         size="small", thermo=False):
    out = str(tmp_path / f"decomp_{world}{tag}{backend}{size}{int(thermo)}.npy")
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    if not backend.startswith("gpu"):
        env["CUDA_VISIBLE_DEVICES"] = ""
    dim_arg = "x".join(str(d) for d in dims) if dims else "-"
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(world), str(port), str(steps), out,
                               str(vscale), str(dt), backend, dim_arg, size, "1" if thermo else "0"],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    logs = [p.communicate(timeout=600)[0].decode() for p in procs]
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return np.load(out)


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("decomp")
    return {w: _run(w, 20, tmp) for w in (1, 2)}


def test_two_ranks_match_one_rank(runs):
    one, two = runs[1], runs[2]
    assert one.shape == two.shape
    assert np.array_equal(one[:, 0], two[:, 0])          # every particle owned exactly once
    L = np.array([8.4, 8.4, 12.6])
    d = two[:, 1:4] - one[:, 1:4]
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-10
    assert np.abs(two[:, 4:7] - one[:, 4:7]).max() <= 1e-10


def test_hot_system_migrates_and_wraps(tmp_path):
    """Fast particles: some change owner and some cross the periodic z face;
    the decomposed result still equals the single-rank run."""
    one = _run(1, 40, tmp_path, vscale=4.0, dt=4e-3, tag="hot")
    two = _run(2, 40, tmp_path, vscale=4.0, dt=4e-3, tag="hot")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from decomp_worker import system
    pos0, _, L = system(vscale=4.0)
    start_owner = (pos0[two[:, 0].astype(int), 2] >= L[2] / 2).astype(int)
    assert np.count_nonzero(start_owner != two[:, 7]) > 0          # migrations happened
    dz = two[:, 3] - pos0[two[:, 0].astype(int), 2]
    assert np.count_nonzero(np.abs(dz) > L[2] / 2) > 0             # periodic crossings
    d = two[:, 1:4] - one[:, 1:4]
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-9
    assert np.abs(two[:, 4:7] - one[:, 4:7]).max() <= 1e-9


def test_decomposed_loop_matches_reference_loop(runs):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from decomp_worker import system
    from oracle import port
    pos, vel, L = system()
    params = port.Params(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4, delta_t=2e-3,
                         boundary=(port.PERIODIC,) * 3)
    p = port.Particles(pos, vel)
    port.simulate_fixed(p, params, port.parse("VL-List_Iter-NoN3L-AoS"), steps=20)
    two = runs[2]
    d = two[:, 1:4] - np.asarray(p.positions)
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-10
    assert np.abs(two[:, 4:7] - np.asarray(p.velocities)).max() <= 1e-10


@pytest.mark.gpu
def test_decomposed_gpu_backend_matches_reference_loop(tmp_path):
    """Two gloo ranks sharing the one GPU, each computing its slab + ghosts with
    libmdg (VL), reproduce the reference loop (no rank waits on another inside
    a kernel: the exchange is host-side)."""
    two = _run(2, 40, tmp_path, vscale=4.0, dt=4e-3, tag="hot", backend="gpu")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from decomp_worker import system
    from oracle import port
    pos, vel, L = system(vscale=4.0)
    params = port.Params(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4, delta_t=4e-3,
                         boundary=(port.PERIODIC,) * 3)
    p = port.Particles(pos, vel)
    port.simulate_fixed(p, params, port.parse("VL-List_Iter-NoN3L-AoS"), steps=40)
    d = two[:, 1:4] - np.asarray(p.positions)
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-9
    assert np.abs(two[:, 4:7] - np.asarray(p.velocities)).max() <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("world,dims,size,steps", [(2, None, "small", 40), (8, (2, 2, 2), "cube10", 24),
                                                   (3, (1, 1, 3), "cube10", 24)])
def test_device_decomposition_matches_reference_loop(tmp_path, world, dims, size, steps):
    """DeviceDecomposedSimulation (everything on the GPU: libmdg drift / force /
    kick, ghosts gathered and scattered on the device, sizes fixed between
    rebuilds) with gloo ranks sharing the one GPU (messages staged on the
    host; no rank waits on another inside a kernel) reproduces the reference
    loop: z-slabs (VL-SoA), a 2x2x2 grid (VL-SoA) and 3 slabs (VL-AoS)."""
    vs, dt = (4.0, 4e-3) if size == "small" else (2.0, 3e-3)
    many = _run(world, steps, tmp_path, vscale=vs, dt=dt, tag="dev", backend="gpudev", dims=dims,
                size=size)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from decomp_worker import system
    from oracle import port
    pos, vel, L = system(vscale=vs, size=size)
    assert np.array_equal(many[:, 0], np.arange(len(pos)))   # every particle owned once
    assert len(np.unique(many[:, 7])) == world
    params = port.Params(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4, delta_t=dt,
                         boundary=(port.PERIODIC,) * 3)
    p = port.Particles(pos, vel)
    port.simulate_fixed(p, params, port.parse("VL-List_Iter-NoN3L-AoS"), steps=steps)
    d = many[:, 1:4] - np.asarray(p.positions)
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-9
    assert np.abs(many[:, 4:7] - np.asarray(p.velocities)).max() <= 1e-9


@pytest.mark.gpu
def test_device_decomposition_with_per_rank_tuners_matches_reference_loop(tmp_path):
    """One controller per rank (the paper's setup): on a 2x2x2 grid every rank
    trials five configurations in its own order (LC C08 / SLI / C01 at both
    CSFs, VCL, VL; AoS and SoA; forced local rebuilds, device-event timings
    to record_timings) and then settles on its own choice, while migration
    and the ghost plan keep the shared R+1 cadence.  The trajectory equals
    the reference loop's (every axis is decomposed, so no rank has a local
    periodic face and the linked-cell traversals see what Verlet lists see)."""
    steps, vs, dt = 24, 2.0, 3e-3
    many = _run(8, steps, tmp_path, vscale=vs, dt=dt, tag="tuned", backend="gpudev_tuned",
                dims=(2, 2, 2), size="cube10")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from decomp_worker import system
    from oracle import port
    pos, vel, L = system(vscale=vs, size="cube10")
    assert np.array_equal(many[:, 0], np.arange(len(pos)))
    params = port.Params(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4, delta_t=dt,
                         boundary=(port.PERIODIC,) * 3)
    p = port.Particles(pos, vel)
    port.simulate_fixed(p, params, port.parse("VL-List_Iter-NoN3L-AoS"), steps=steps)
    d = many[:, 1:4] - np.asarray(p.positions)
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-9
    assert np.abs(many[:, 4:7] - np.asarray(p.velocities)).max() <= 1e-9


@pytest.fixture(scope="module")
def grid_runs(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("grid")
    kw = dict(vscale=2.0, dt=3e-3, size="cube10")
    return {"1": _run(1, 24, tmp, tag="g1", **kw),
            "2x2x1": _run(4, 24, tmp, tag="g4", dims=(2, 2, 1), **kw),
            "2x2x2": _run(8, 24, tmp, tag="g8", dims=(2, 2, 2), **kw)}


@pytest.mark.parametrize("grid", ["2x2x1", "2x2x2"])
def test_process_grids_match_one_rank(grid_runs, grid):
    """Config-5 style 3-D grids: edge and corner ghosts arrive through the
    axis-by-axis exchange; every particle owned once; same trajectory."""
    one, many = grid_runs["1"], grid_runs[grid]
    assert np.array_equal(one[:, 0], many[:, 0])
    L = np.array([14.0, 14.0, 14.0])
    d = many[:, 1:4] - one[:, 1:4]
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-10
    assert np.abs(many[:, 4:7] - one[:, 4:7]).max() <= 1e-10
    assert len(np.unique(many[:, 7])) == int(np.prod([int(x) for x in grid.split("x")]))


def test_grid_with_thermostat_matches_reference_loop(tmp_path):
    """2x2x2 ranks with the thermostat (all-reduced temperature, config 4's
    quench mechanism) against the reference loop with the same thermostat."""
    from conftest import ScriptedController  # noqa: F401  (fixture module import)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from decomp_worker import system, thermostat
    from oracle import port
    many = _run(8, 18, tmp_path, vscale=2.0, dt=3e-3, tag="th", dims=(2, 2, 2), size="cube10",
                thermo=True)
    pos, vel, L = system(vscale=2.0, size="cube10")
    params = port.Params(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4, delta_t=3e-3,
                         boundary=(port.PERIODIC,) * 3, thermostat=thermostat())

    class Fixed:
        mode = "steady"

        def configuration_for_iteration(self, it):
            return port.parse("VL-List_Iter-NoN3L-AoS"), False

        def record_timings(self, f, b):
            pass

        def record_failure(self, e=None):
            return False

    p = port.Particles(pos, vel)
    port.simulate_controlled(p, params, Fixed(), steps=18)
    d = many[:, 1:4] - np.asarray(p.positions)
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-9
    assert np.abs(many[:, 4:7] - np.asarray(p.velocities)).max() <= 1e-9



@pytest.mark.gpu
def test_device_decomposition_with_thermostat_matches_reference_loop(tmp_path):
    """DeviceDecomposedSimulation on a 2x2x2 grid with the thermostat (kinetic
    energy and counts all-reduced over the owned rows; the thermostat's steps
    kick eagerly) against the reference loop with the same thermostat."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from decomp_worker import system, thermostat
    from oracle import port
    many = _run(8, 18, tmp_path, vscale=2.0, dt=3e-3, tag="devth", backend="gpudev", dims=(2, 2, 2),
                size="cube10", thermo=True)
    pos, vel, L = system(vscale=2.0, size="cube10")
    params = port.Params(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4, delta_t=3e-3,
                         boundary=(port.PERIODIC,) * 3, thermostat=thermostat())

    class Fixed:
        mode = "steady"

        def configuration_for_iteration(self, it):
            return port.parse("VL-List_Iter-NoN3L-AoS"), False

        def record_timings(self, f, b):
            pass

        def record_failure(self, e=None):
            return False

    p = port.Particles(pos, vel)
    port.simulate_controlled(p, params, Fixed(), steps=18)
    d = many[:, 1:4] - np.asarray(p.positions)
    d -= L * np.rint(d / L)
    assert np.abs(d).max() <= 1e-9
    assert np.abs(many[:, 4:7] - np.asarray(p.velocities)).max() <= 1e-9
