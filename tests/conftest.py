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


def golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def system_names():
    return sorted(f[4:-4] for f in os.listdir(GOLDEN) if f.startswith("sys_"))
