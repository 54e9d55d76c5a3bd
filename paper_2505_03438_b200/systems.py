"""Seeded synthetic inputs of BASELINE.json's configurations.

The reference's scenario generators (scenarios.py:79-201) do not cover these
systems; they are built here with numpy's seeded Generator so the GPU arm and
the CPU baseline (oracle/) consume identical inputs.

* config 1: simple-cubic sites (i + 0.5) * 1.1 sigma, i < 20 per axis, jitter
  U(-0.05, 0.05) sigma, periodic cube of 22 sigma, T = 0.7.
* config 2: N uniform points at rho = 0.75 in a periodic cube, overlaps relaxed
  by 50 capped steepest-descent steps on the GPU, T = 0.7.
"""

from __future__ import annotations

import math

import numpy as np

from .params import PERIODIC, SimulationParams


def thermal_velocities(rng, masses, temperature):
    """Maxwell-Boltzmann draw, zero net momentum, rescaled onto T exactly
    (scenarios.py:192-201)."""
    n = len(masses)
    v = rng.normal(0.0, 1.0, size=(n, 3))
    v *= np.sqrt(temperature / masses)[:, None]
    v -= np.average(v, axis=0, weights=masses)
    t_now = float(np.sum(masses * np.sum(v * v, axis=1)) / (3.0 * n))
    if t_now > 0.0:
        v *= math.sqrt(temperature / t_now)
    return v


def sc_lattice(n_side=20, spacing=1.1, jitter=0.05, seed=0, temperature=0.7, offset=0.5):
    """BASELINE config 1 (and its scaled-down variants)."""
    rng = np.random.default_rng(seed)
    i = (np.arange(n_side) + offset) * spacing
    sites = np.stack(np.meshgrid(i, i, i, indexing="ij"), axis=-1).reshape(-1, 3)
    pos = sites + rng.uniform(-jitter, jitter, sites.shape)
    vel = thermal_velocities(rng, np.ones(len(pos)), temperature)
    L = n_side * spacing
    return pos, vel, np.array([L, L, L])


def config1_params(steps=100, rebuild_interval=10):
    pos, vel, L = sc_lattice()
    params = SimulationParams(domain_size=L, cutoff=2.5, skin=0.3,
                              rebuild_interval=rebuild_interval, delta_t=1e-3,
                              total_iterations=steps, boundary=(PERIODIC,) * 3)
    return pos, vel, params


def uniform_box(n, density, seed=0):
    L = (n / density) ** (1.0 / 3.0)
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, L, (n, 3))
    return pos, np.array([L, L, L]), rng


SD_STEPS = 50
SD_GAMMA = 1e-3      # displacement per unit force
SD_MAX_DISP = 0.05   # sigma per step


def relax_on_device(particles, params, config, steps=SD_STEPS, gamma=SD_GAMMA,
                    max_disp=SD_MAX_DISP):
    """Capped steepest descent x += F/|F| min(gamma |F|, max_disp) with the GPU
    force path (fresh neighbour structures every step)."""
    from .calculator import ForceCalculator
    calc = ForceCalculator(particles, params)
    particles.convert_layout(config.layout)
    for _ in range(steps):
        calc.rebuild(particles, config)
        calc.refresh(particles, config)
        calc.compute_async(particles, config)
        calc.sd_step(particles, gamma, max_disp)
    if calc.blowup():
        raise RuntimeError("steepest descent left the domain")
    calc.close()
    particles.force.zero_()
    particles.old_force.zero_()


def config2_inputs(n=1_048_576, density=0.75, seed=0, temperature=0.7):
    """Unrelaxed config-2 positions, velocities and params (relax separately)."""
    pos, L, rng = uniform_box(n, density, seed)
    vel = thermal_velocities(rng, np.ones(n), temperature)
    params = SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                              delta_t=2e-3, total_iterations=1000, boundary=(PERIODIC,) * 3)
    return pos, vel, params


def fcc_sites(n_cells, a, offset=0.25):
    """FCC sites of an n_cells[0] x n_cells[1] x n_cells[2] block, lattice constant a."""
    basis = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]]) + offset
    g = np.stack(np.meshgrid(*[np.arange(k) for k in n_cells], indexing="ij"), -1).reshape(-1, 1, 3)
    return ((g + basis[None]) * a).reshape(-1, 3)


def config3_inputs(n=2_097_152, box=(128.0, 128.0, 640.0), density=0.8, seed=0,
                   temperature=2.0, ramp=1.0):
    """BASELINE config 3: dense FCC slab centred in z with vacuum around it.

    As stated the config is inconsistent (the central 20% of 640 sigma at
    rho = 0.8 holds 1,677,721 particles, not 2,097,152); N is kept
    and the slab is as thick as rho = 0.8 requires (about 160 sigma).  Sites:
    FCC with a = (4/rho)^(1/3), the N sites closest to the mid-plane.
    Velocities: Maxwell-Boltzmann at T plus v_z += ramp * (z - zc)/(h/2)."""
    rng = np.random.default_rng(seed)
    a = (4.0 / density) ** (1.0 / 3.0)
    L = np.asarray(box, dtype=np.float64)
    h = n / (density * L[0] * L[1])
    nx, ny = int(L[0] // a), int(L[1] // a)
    nc = (nx, ny, int(np.ceil(n / (4.0 * nx * ny))) + 1)
    sites = fcc_sites(nc, a)
    zc = 0.5 * L[2]
    sites[:, 2] += zc - 0.5 * nc[2] * a
    keep = np.argsort(np.abs(sites[:, 2] - zc), kind="stable")[:n]
    pos = sites[np.sort(keep)]
    pos += rng.uniform(-0.05, 0.05, pos.shape)
    vel = thermal_velocities(rng, np.ones(n), temperature)
    vel[:, 2] += ramp * (pos[:, 2] - zc) / (0.5 * h)
    params = SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                              delta_t=1e-3, total_iterations=5000, boundary=(PERIODIC,) * 3)
    return pos, vel, params


def config4_inputs(n=4_194_304, density=0.4, seed=0, temperature=1.4):
    """BASELINE config 4 before relaxation/equilibration: uniform at rho = 0.4
    (relax with relax_on_device; equilibrate at T = 1.4, then rescale to 0.7)."""
    pos, L, rng = uniform_box(n, density, seed)
    vel = thermal_velocities(rng, np.ones(n), temperature)
    params = SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                              delta_t=2e-3, total_iterations=10000, boundary=(PERIODIC,) * 3)
    return pos, vel, params


def config5_inputs(n_side=256, density=0.8, seed=0, temperature=0.9, jitter=0.05):
    """BASELINE config 5: FCC 256^3 cells (67,108,864 particles), a = (4/rho)^(1/3),
    jittered, Maxwell-Boltzmann at T = 0.9."""
    rng = np.random.default_rng(seed)
    a = (4.0 / density) ** (1.0 / 3.0)
    pos = fcc_sites((n_side,) * 3, a)
    pos += rng.uniform(-jitter, jitter, pos.shape)
    vel = thermal_velocities(rng, np.ones(len(pos)), temperature)
    L = np.full(3, n_side * a)
    params = SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                              delta_t=2e-3, total_iterations=1000, boundary=(PERIODIC,) * 3)
    return pos, vel, params


def config4_state(equil_steps=1000, quench_steps=4000, seed=0, config="VL-List_Iter-NoN3L-SoA",
                  interval=10, stats=None):
    """BASELINE config 4's quench, run on the device: uniform rho = 0.4 ->
    50 steepest-descent steps -> ``equil_steps`` at T = 1.4 (thermostat every
    ``interval`` steps, integrator.py:81-95 on the device) -> velocities
    rescaled to T = 0.7 in one application -> ``quench_steps`` held at
    T = 0.7.  At rho = 0.4, T = 0.7 the fluid sits inside the LJ liquid-vapour
    coexistence region (truncated LJ: T_c ~ 1.19, rho_c ~ 0.32), so droplets
    nucleate and the cell occupancy turns strongly non-uniform (see
    ``stats``: a list that receives the live statistics (livestats.py:46-77)
    before and after the quench).  Returns numpy (pos, vel, params)."""
    from dataclasses import replace

    from .configuration import parse_configuration
    from .params import ThermostatParams
    from .particles import ParticleSet
    from .simulation import Simulation
    pos, vel, params = config4_inputs(seed=seed)
    cfg = parse_configuration(config)
    parts = ParticleSet(pos, vel)
    del pos, vel
    relax_on_device(parts, params, parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    parts.convert_layout(cfg.layout)
    eq = replace(params, thermostat=ThermostatParams(1.4, 1e9, interval))
    sim = Simulation(parts, eq, cfg, fuse_kick_drift=True, reorder=8)
    if stats is not None:
        stats.append(sim.calc.live_stats(parts))
    sim.run(equil_steps, record=False)
    sim.check()
    sim.calc.thermostat(parts, 0.7, 1e9)            # the quench: one rescale to T = 0.7
    q = replace(params, thermostat=ThermostatParams(0.7, 1e9, interval))
    sim = Simulation(parts, q, cfg, fuse_kick_drift=True, reorder=8)
    sim.run(quench_steps, record=False)
    sim.check()
    if stats is not None:
        stats.append(sim.calc.live_stats(parts))
    parts.convert_layout("AoS")
    return parts.numpy("pos"), parts.numpy("vel"), params
