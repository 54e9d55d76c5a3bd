"""Shared test plumbing.

Markers: ``gpu`` = needs a B200 (runs through the C-ABI library); everything
else runs on CPU in the build container.  The oracle (oracle/port.py + the C
restatement in oracle/ljport.c) is the checker for every parity test.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    lib = os.path.join(ROOT, "oracle", "_build", "libljport.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


@pytest.fixture(scope="session")
def config2_snapshot():
    """BASELINE config 2 (1,048,576 particles, rho = 0.75) after its 50
    steepest-descent steps on the device: the identical seeded input both
    the GPU path and the oracle consume at full size."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA")
    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200 import systems
    pos, vel, params = systems.config2_inputs()
    parts = P.ParticleSet(pos, vel)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    return parts.numpy("pos"), parts.numpy("vel"), params


def golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def system_names():
    return sorted(f[4:-4] for f in os.listdir(GOLDEN) if f.startswith("sys_"))


class ScriptedController:
    """Replays a TuningController run recorded from the reference
    (tests/golden/traj_tuned.npz: per iteration the configuration, the forced
    flag and the controller mode, tuning.py:200-210), through the same
    protocol: configuration_for_iteration / record_timings / record_failure."""

    def __init__(self, z, parse):
        self.seq = {int(i): (parse(str(c)), bool(f), str(m))
                    for i, c, f, m in zip(z["seq_it"], z["seq_cfg"], z["seq_forced"], z["seq_mode"])}
        self.mode = "steady"
        self.timings = []
        self.trial_iterations = 0
        self.tuning_interval = int(z["tuning"][0])

    def configuration_for_iteration(self, iteration):
        cfg, forced, self.mode = self.seq[iteration]
        return cfg, forced

    def record_timings(self, force_ns, build_ns):
        if self.mode == "trial":           # tuning.py:213: no-op outside trials
            self.timings.append((force_ns, build_ns))
            self.trial_iterations += 1

    def record_failure(self, error=None):
        return False


class Thermostat:
    def __init__(self, target, max_delta_t, interval):
        self.target_temperature = target
        self.max_delta_t = max_delta_t
        self.interval_iterations = interval
