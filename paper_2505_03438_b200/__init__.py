"""B200-native (sm_100a) Lennard-Jones force + neighbour-identification path of
the mdtune reference (arXiv 2505.03438 re-creation).

Public surface mirrors the reference's names on this path:
``Configuration / enumerate_configurations / parse_configuration``
(configuration.py), ``SimulationParams`` (params.py), ``ParticleSet``
(particles.py, device-resident), ``ForceCalculator / compute_forces``
(containers.py:378-511) and ``simulate`` (simulation.py:126-197).
``HostForceCalculator`` is the drop-in for the reference's own host-side loop
(see plugin.py).  All compute runs in libmdg (include/mdg.h).
"""

from .configuration import (C01, C08, C18, CELL_TRAVERSALS, CLUSTER_ITER, CSF_VALUES, LINKED_CELLS,
                            LIST_ITER, SLI, VERLET_CLUSTER_LISTS, VERLET_LISTS, Configuration,
                            configuration_index,
                            enumerate_configurations, extended_configurations, tuning_space,
                            parse_configuration)
from .params import PERIODIC, REFLECTIVE, SimulationParams, ThermostatParams
from .particles import AOS, SOA, ParticleSet, ParticleTypeInfo

__all__ = [
    "AOS", "SOA", "C01", "C08", "C18", "SLI", "LIST_ITER", "CLUSTER_ITER", "LINKED_CELLS",
    "VERLET_LISTS", "VERLET_CLUSTER_LISTS",
    "CELL_TRAVERSALS", "CSF_VALUES", "PERIODIC", "REFLECTIVE", "Configuration",
    "enumerate_configurations", "extended_configurations", "tuning_space", "parse_configuration", "configuration_index",
    "SimulationParams", "ThermostatParams", "ParticleSet", "ParticleTypeInfo",
    "ForceCalculator", "HostForceCalculator", "compute_forces", "Timings", "simulate",
    "Simulation", "BlowUpError",
]


def __getattr__(name):
    # GPU-facing pieces load lazily so host-only imports work without CUDA
    if name in ("ForceCalculator", "HostForceCalculator", "compute_forces", "Timings"):
        from . import calculator
        return getattr(calculator, name)
    if name in ("simulate", "Simulation", "BlowUpError"):
        from . import simulation
        return getattr(simulation, name)
    raise AttributeError(name)
