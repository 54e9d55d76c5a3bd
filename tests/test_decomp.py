"""Domain decomposition on CPU: world_size 2 over gloo.

The decomposed loop (slabs along z, per-step ghost exchange, migration at
rebuilds) must reproduce the single-rank run and the reference loop (oracle
restatement of simulation.py:126-197) on the same seeded system.
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


def _run(world, steps, tmp_path, vscale=0.8, dt=2e-3, tag="", backend="oracle"):
    out = str(tmp_path / f"decomp_{world}{tag}{backend}.npy")
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    if backend != "gpu":
        env["CUDA_VISIBLE_DEVICES"] = ""
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(world), str(port), str(steps), out,
                               str(vscale), str(dt), backend],
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
