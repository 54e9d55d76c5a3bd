"""GPU training-data sweep (mirror of mdtune.dataset,
dataset.py:104-202, on-disk format unchanged).

The reference labels each sweep point with the measured-cheapest
configuration of a static-snapshot trial (dataset.py:104-140) and writes
the eight live-statistics features, one ``cost:<configId>`` column per
configuration and the winning id in ``label`` (dataset.py:143-146, 193-197).
Here every piece runs on the device:

* the trial of each configuration (one rebuild, ``trial_iterations``
  refresh + compute) is timed with CUDA events on the calculator's stream,
  not host wall clock;
* the features come from ``mdg_live_stats`` (bit-identical to
  livestats.py:46-77);
* the cost is the reference's ``evidence_cost`` (tuning.py:24-30): median
  force + slowest build / rebuild interval.

The CSV is readable by the reference's ``load_training_csv`` /
``train_forest_from_csv`` (dataset.py:205-235) and rule tooling, so the
reference's own trainers can be retrained on GPU labels -- including the
GPU-only configurations when ``space=extended_configurations()``.
Scenario generation stays with the caller (the reference's scenarios.py is
out of scope): pass ``(particles, params)`` sweep points.
"""

from __future__ import annotations

import csv
import logging
import math
import statistics

import torch

from .calculator import ForceCalculator
from .configuration import enumerate_configurations
from .livestats import FEATURE_NAMES

log = logging.getLogger(__name__)

TRIAL_ITERATIONS = 10   # dataset.py:36


def evidence_cost(force_ns: float, build_ns: float, rebuild_interval: int) -> float:
    """tuning.py:24-30."""
    if rebuild_interval < 1:
        raise ValueError("rebuild interval must be >= 1")
    return float(force_ns) + float(build_ns) / rebuild_interval


def measure_configuration_costs(particles, params, *, trial_iterations=TRIAL_ITERATIONS,
                                space=None, calculator=None) -> dict:
    """dataset.py:104-140 on the device: per configuration one rebuild and
    ``trial_iterations`` refresh + compute, device-timed; failures cost inf."""
    space = space if space is not None else enumerate_configurations()
    calc = calculator or ForceCalculator(particles, params)
    costs = {}
    try:
        for config in space:
            try:
                forces, builds = [], []
                for i in range(trial_iterations):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                    ev[0].record(calc.ctx.stream)
                    if particles.layout != config.layout:
                        particles.convert_layout(config.layout)
                    if i == 0:
                        calc.rebuild(particles, config)
                    calc.refresh(particles, config)
                    ev[1].record(calc.ctx.stream)
                    calc.compute_async(particles, config)
                    ev[2].record(calc.ctx.stream)
                    ev[2].synchronize()
                    builds.append(ev[0].elapsed_time(ev[1]) * 1e6)
                    forces.append(ev[1].elapsed_time(ev[2]) * 1e6)
                costs[config.id] = evidence_cost(statistics.median(forces), max(builds),
                                                 params.rebuild_interval)
            except Exception as exc:   # the reference's trial-failure rule
                log.warning("configuration %s failed during trial: %s", config.id, exc)
                costs[config.id] = float("inf")
    finally:
        if calculator is None:
            calc.close()
    return costs


def dataset_columns(space=None) -> list:
    """dataset.py:143-146."""
    space = space if space is not None else enumerate_configurations()
    return list(FEATURE_NAMES) + [f"cost:{c.id}" for c in space] + ["label"]


def sweep_row(particles, params, *, space=None, trial_iterations=TRIAL_ITERATIONS):
    """One labelled row (features, costs, label) of a sweep point, or None
    when every configuration failed (dataset.py:183-197)."""
    space = space if space is not None else enumerate_configurations()
    calc = ForceCalculator(particles, params)
    try:
        stats = calc.live_stats(particles)
        costs = measure_configuration_costs(particles, params, trial_iterations=trial_iterations,
                                            space=space, calculator=calc)
    finally:
        calc.close()
    if not math.isfinite(min(costs.values())):
        return None
    label = min(space, key=lambda c: costs[c.id]).id   # ties: earliest in the space
    return ([f"{v!r}" for v in stats.feature_vector().tolist()]
            + [repr(costs[c.id]) for c in space] + [label])


def generate_training_dataset(out_path, points, *, space=None,
                              trial_iterations=TRIAL_ITERATIONS, progress=None) -> int:
    """Write the training CSV for ``points`` = iterable of (particles, params)
    (dataset.py:149-202 with the scenario roster left to the caller);
    returns the number of rows.  Failing points are logged and skipped."""
    space = list(space) if space is not None else enumerate_configurations()
    rows = 0
    with open(out_path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(dataset_columns(space))
        for k, (particles, params) in enumerate(points):
            try:
                row = sweep_row(particles, params, space=space, trial_iterations=trial_iterations)
            except Exception as exc:
                log.warning("sweep point %d failed: %s", k, exc)
                continue
            if row is None:
                log.warning("sweep point %d: every configuration failed", k)
                continue
            writer.writerow(row)
            rows += 1
            if progress:
                progress(k, row[-1])
    return rows


# -- GPU-labelled tuning artefacts (tools/gpu_training.py) ----------------------

import os as _os

DATA_DIR = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "data")
GPU_TRAINING_CSV = _os.path.join(DATA_DIR, "gpu_training.csv")
GPU_FOREST = _os.path.join(DATA_DIR, "gpu_forest.json")
GPU_RULES = _os.path.join(DATA_DIR, "gpu_rules.txt")


def gpu_rules_text() -> str:
    """The rule file distilled from the device-timed sweep of the reference's
    roster, in the reference's grammar: pass it to mdtune's
    ``parse_rule_file(text, tuning_space())`` and ``ExpertStrategy``."""
    with open(GPU_RULES) as fh:
        return fh.read()


def load_gpu_forest():
    """The forest the reference's trainer built from GPU labels
    (``mdtune.forest.load_forest``; needs the reference package)."""
    from mdtune.forest import load_forest
    return load_forest(GPU_FOREST)
