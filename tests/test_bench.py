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


@pytest.mark.gpu
def test_decomposed_bench_path_two_ranks():
    """torchrun --nproc-per-node 2 with --dist-backend gloo: two z-slabs of
    65,536 particles each, ghosts exchanged every step, one JSON line."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), BENCH,
                        "--gpus", "2", "--particles", "65536", "--steps", "11", "--warmup", "3",
                        "--dist-backend", "gloo"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["n_particles"] == 2 * 65536
    assert d["config"]["parallelism"].startswith("zslab2") and d["value"] > 0
