"""Device-side bounds checks in place of compute-sanitizer (closed on the GPU
pool): the checked build of libmdg (``make CHECKS=1`` ->
paper_2505_03438_b200/_build_checks/libmdg.so, MDG_DCHECK in mdg.cuh) traps
on any out-of-range shared-memory gather index, list slot, window range or
atomic-claimed cell slot.  tools/sanitize_cases.py drives every kernel family
built on mbarrier / bulk-copy rings, shared-memory windows and atomics (tiled
walk + prune walk + fp32 walk + tile build, LC C08/C18/SLI/C01, VCL N3L, the
fused loop with cell reorder and a prune every step) through it; the run must
finish cleanly and give the product library's eval counts."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
CHECKED = os.path.join(ROOT, "paper_2505_03438_b200", "_build_checks", "libmdg.so")
CASES = os.path.join(ROOT, "tools", "sanitize_cases.py")


def _run(lib=None):
    env = dict(os.environ)
    if lib:
        env["MDG_LIB_PATH"] = lib
    r = subprocess.run([sys.executable, CASES], capture_output=True, text=True, env=env, timeout=900)
    return r


def test_checked_build_runs_every_kernel_family_clean():
    if not os.path.exists(CHECKED):
        pytest.fail("checked build missing: make -C paper_2505_03438_b200/csrc CHECKS=1")
    plain, checked = _run(), _run(CHECKED)
    assert plain.returncode == 0, plain.stderr[-2000:]
    assert checked.returncode == 0 and "MDG_DCHECK failed" not in checked.stdout + checked.stderr, \
        (checked.stdout + checked.stderr)[-3000:]
    counts = lambda out: [ln for ln in out.splitlines() if " count " in ln]
    assert counts(checked.stdout) == counts(plain.stdout) and len(counts(plain.stdout)) >= 10
    assert "sanitize cases done" in checked.stdout
