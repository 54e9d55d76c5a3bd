"""bench.py's JSON contract on reduced sizes: the reference arm (CPU), the
single-GPU line and the N > 1 decomposed path (two gloo ranks sharing the
one GPU -- a smoke run of the code path, never a performance number)."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _line(out):
    lines = [x for x in out.strip().splitlines() if x.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


def test_reference_arm_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--n", "32768", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "MUPS"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    # the other ranks of a torchrun launch exit 0 without output
    r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--n", "32768"],
                       capture_output=True, text=True, timeout=600,
                       env=dict(env, RANK="1", WORLD_SIZE="2"))
    assert r.returncode == 0 and not r.stdout.strip()


@pytest.mark.gpu
def test_gpu_line_contract():
    r = subprocess.run([sys.executable, BENCH, "--n", "65536", "--steps", "11", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 11 and d["value"] > 0 and d["gpu_launches"] > 0
    assert 0 < d["roofline"]["frac"] < 1 and d["roofline"]["unit"] == "TFLOP/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 24 * 65536 and d["e2e"]["value"] > 0


def _torchrun(n, *args, timeout=1200):
    return subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
                           str(n), "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), BENCH,
                           "--gpus", str(n), "--steps", "11", "--warmup", "3", "--dist-backend", "gloo",
                           *args], capture_output=True, text=True, timeout=timeout)


@pytest.mark.gpu
@pytest.mark.parametrize("n,extra,grid", [(2, ("--n5-side", "48"), "2x1x1"),
                                          (4, ("--n5-side", "48"), "2x2x1"),
                                          (2, ("--workload", "config2", "--particles", "65536"), "1x1x2")])
def test_decomposed_bench_path(n, extra, grid):
    """torchrun with --dist-backend gloo (ranks sharing the one GPU; a smoke
    run of the code path, never a performance number): the default N > 1
    workload is config 5 strong-scaled over the 3-D process grid (a reduced
    48^3-cell lattice here); config 2 runs as z-slabs of a system relaxed on
    rank 0 and broadcast.  One JSON line naming the workload and the split."""
    r = _torchrun(n, *extra)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == n and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["decomposition"] == grid and d["comm"]["ranks"] == n
    if "--n5-side" in extra:
        assert d["config"]["workload"].startswith("config5") and d["config"]["n_particles"] == 4 * 48 ** 3
    else:
        assert d["config"]["n_particles"] == 65536


@pytest.mark.gpu
def test_decomposed_bench_with_per_rank_predictive_tuners():
    """--tune predictive: one reference TuningController per rank (needs the
    staged reference under baseline/_ref) selecting from device timings."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "mdtune")):
        pytest.skip("reference not staged under baseline/_ref")
    r = _torchrun(2, "--n5-side", "48", "--tune", "predictive", "--steps", "90")
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["config"]["tuning"] == "predictive" and d["tuning_trials"] > 0
    assert d["phase_selections"]


def test_process_grids_and_workload_names():
    """bench.py's decomposition choice: config 5 as 2x1x1 /
    2x2x1 / 2x2x2 at 2 / 4 / 8 ranks (a 3-factor split otherwise), configs
    2-4 as z-slabs; the default workload is config 2 at N = 1 and config 5 at
    N > 1."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", BENCH)
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert [b.grid_dims("config5", n) for n in (1, 2, 4, 8)] == [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2)]
    for n in (3, 6, 12, 16):
        d = b.grid_dims("config5", n)
        assert d[0] * d[1] * d[2] == n
    assert b.grid_dims("config3", 4) == (1, 1, 4) and b.grid_dims("config4", 8) == (1, 1, 8)
    assert b.default_workload(1) == "config2" and b.default_workload(8) == "config5"
    assert set(b.WORKLOADS) == {"config2", "config3", "config4", "config5"}
