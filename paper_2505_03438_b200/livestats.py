"""Live statistics (mirror of mdtune.livestats, livestats.py:1-77).

The eight runtime features the expert / forest selectors consume, in the
reference's order (livestats.py:17-19, the dataset/model contract).  On this
path they are computed on the device by ``mdg_live_stats`` (stats.cu), so a
tuning phase never copies positions to the host:
``ForceCalculator.live_stats(particles)`` or ``compute_live_stats``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

FEATURE_NAMES = ("meanParticlesPerBin", "relStdDevParticlesPerBin",
                 "medianParticlesPerBin", "maxParticlesPerBin",
                 "numBins", "numEmptyBins", "threadCount", "skin")


@dataclass(frozen=True)
class LiveStatistics:
    mean_particles_per_bin: float
    rel_std_dev_particles_per_bin: float
    median_particles_per_bin: float
    max_particles_per_bin: float
    num_bins: int
    num_empty_bins: int
    thread_count: int
    skin: float

    def feature_vector(self) -> np.ndarray:
        return np.array([
            self.mean_particles_per_bin, self.rel_std_dev_particles_per_bin,
            self.median_particles_per_bin, self.max_particles_per_bin,
            float(self.num_bins), float(self.num_empty_bins),
            float(self.thread_count), self.skin,
        ])


def compute_live_stats(particles, params, calculator=None) -> LiveStatistics:
    """livestats.py:46-77 on the device.  Pass the simulation's
    ForceCalculator to reuse its context; otherwise a temporary one is made."""
    from .calculator import ForceCalculator
    if calculator is not None:
        return calculator.live_stats(particles)
    calc = ForceCalculator(particles, params)
    try:
        return calc.live_stats(particles)
    finally:
        calc.close()
