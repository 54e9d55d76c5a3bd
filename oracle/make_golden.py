"""ORACLE / TEST INFRASTRUCTURE: regenerate tests/golden/*.npz from the REAL
reference package (mdtune, numba kernels) imported from /root/reference.

Run in the build container only (the reference does not exist on GPU boxes):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/make_golden.py

Every array written here is produced by the reference's own public API:
``make_geometry / pruned_stencil / forward_stencil`` (cells.py:55-111),
``GridState.rebuild`` (containers.py:93-118), ``VerletListState.rebuild``
(containers.py:352-375), ``compute_forces`` (containers.py:494-511) and
``simulate`` with ``FixedStrategy`` (simulation.py:126-197).  The inputs are
seeded and stored next to the outputs, so the fixtures are self-contained.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from mdtune.cells import forward_stencil, make_geometry, pruned_stencil  # noqa: E402
from mdtune.configuration import enumerate_configurations, parse_configuration  # noqa: E402
from mdtune.containers import GridState, VerletListState, compute_forces  # noqa: E402
from mdtune.integrator import apply_thermostat, current_temperature  # noqa: E402
from mdtune.livestats import compute_live_stats  # noqa: E402
from mdtune.params import PERIODIC, REFLECTIVE, SimulationParams, ThermostatParams  # noqa: E402
from mdtune.particles import ParticleSet, ParticleTypeInfo  # noqa: E402
from mdtune.simulation import simulate  # noqa: E402
import mdtune.simulation as _msim  # noqa: E402
from mdtune.tuning import FixedStrategy, FullSearchStrategy, TuningController  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
P, R = PERIODIC, REFLECTIVE


def _types(n_types):
    return [ParticleTypeInfo(t, epsilon=1.0 + 0.5 * t, sigma=1.0 - 0.2 * t,
                             mass=1.0 + t) for t in range(n_types)]


def _random(rng, n, domain, n_types):
    pos = rng.uniform(0.0, 1.0, (n, 3)) * np.asarray(domain, float)
    tid = (np.arange(n) % n_types).astype(np.int64)
    return pos, tid


def geometry_cases():
    cases = [((9.0, 9.0, 9.0), 3.0, 1.0, (1, 1, 1)), ((10.0, 10.0, 10.0), 3.0, 1.0, (1, 1, 1)),
             ((9.0, 9.0, 9.0), 3.0, 0.5, (1, 1, 1)), ((2.5, 2.5, 2.5), 3.0, 1.0, (0, 0, 0)),
             ((23.7, 11.0, 8.1), 3.5, 1.0, (1, 1, 1)), ((23.7, 11.0, 8.1), 3.5, 0.5, (1, 1, 1)),
             ((12.0, 12.0, 12.0), 3.0, 1.0, (1, 0, 1)), ((22.0, 22.0, 22.0), 2.8, 1.0, (1, 1, 1)),
             ((22.0, 22.0, 22.0), 2.8, 0.5, (1, 1, 1)), ((111.8183, 111.8183, 111.8183), 2.8, 1.0, (1, 1, 1)),
             ((111.8183, 111.8183, 111.8183), 2.8, 0.5, (1, 1, 1)), ((128.0, 128.0, 800.0), 2.8, 0.5, (1, 1, 1))]
    out = {}
    for k, (dom, ell, csf, per) in enumerate(cases):
        g = make_geometry(dom, ell, csf, tuple(bool(p) for p in per))
        out[f"g{k}_in_domain"] = np.array(dom)
        out[f"g{k}_in_scalars"] = np.array([ell, csf])
        out[f"g{k}_in_periodic"] = np.array(per, dtype=np.int64)
        out[f"g{k}_dims_owned"] = np.array(g.dims_owned)
        out[f"g{k}_cell_length"] = np.array(g.cell_length)
        out[f"g{k}_overlap"] = np.array(g.overlap)
        out[f"g{k}_halo"] = np.array(g.halo)
        out[f"g{k}_dims"] = np.array(g.dims)
        out[f"g{k}_pruned"] = pruned_stencil(g).reshape(-1, 3)
        for major in range(3):
            out[f"g{k}_forward{major}"] = forward_stencil(g, major).reshape(-1, 3)
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "geometry.npz"), **out)


def systems():
    """The reference test-suite systems (tests/conftest.py:73-99,
    tests/test_containers.py:40-55, tests/test_acceptance.py:57-141) plus two
    edge cases (a domain at the 2*ell periodic minimum; an empty set)."""
    out = []
    rng = np.random.default_rng(1234)
    pos, tid = _random(rng, 120, (9.0, 9.0, 9.0), 2)
    out.append(("small_periodic", pos, tid, 2, dict(domain_size=(9.0, 9.0, 9.0), cutoff=2.5, skin=0.3,
                                                     boundary=(P, P, P))))
    rng = np.random.default_rng(1234)
    pos, tid = _random(rng, 100, (9.0, 11.0, 10.0), 2)
    out.append(("reflective", pos, tid, 2, dict(domain_size=(9.0, 11.0, 10.0), cutoff=2.5, skin=0.2,
                                                 boundary=(R, R, R))))
    rng = np.random.default_rng(1234)
    pos, tid = _random(rng, 110, (9.0, 11.0, 10.0), 2)
    out.append(("mixed", pos, tid, 2, dict(domain_size=(9.0, 11.0, 10.0), cutoff=2.5, skin=0.3,
                                            boundary=(P, R, P))))
    # acceptance criterion 1 generator (tests/test_acceptance.py:59-72), first 3 cases
    rng = np.random.default_rng(20260823)
    for case in range(3):
        domain = tuple(np.round(rng.uniform(8.0, 13.0, 3), 2))
        boundary = tuple(str(b) for b in rng.choice([P, R], 3))
        cutoff = float(rng.uniform(2.5, 3.0))
        skin = float(rng.uniform(0.0, 0.5))
        nt = int(rng.integers(1, 4))
        pos, tid = _random(rng, 500, domain, nt)
        out.append((f"crit1_{case}", pos, tid, nt, dict(domain_size=domain, cutoff=cutoff, skin=skin,
                                                         boundary=boundary)))
    # criterion 3 tight blob (most cells empty)
    rng = np.random.default_rng(88)
    pos = rng.uniform(3.0, 6.0, (120, 3))
    out.append(("blob", pos, np.zeros(120, dtype=np.int64), 1,
                dict(domain_size=(10.0, 12.0, 9.0), cutoff=3.0, skin=0.0, boundary=(R, R, R))))
    # periodic domain at exactly 2*ell on one axis, small cells on others
    rng = np.random.default_rng(7)
    pos, tid = _random(rng, 60, (5.6, 6.0, 7.3), 3)
    out.append(("tight", pos, tid, 3, dict(domain_size=(5.6, 6.0, 7.3), cutoff=2.5, skin=0.3,
                                            boundary=(P, P, P))))
    # particles sitting exactly on the faces / at L (binning clip, image rules)
    rng = np.random.default_rng(11)
    pos, tid = _random(rng, 90, (9.0, 9.0, 9.0), 1)
    pos[:10, 0] = 0.0
    pos[10:20, 1] = 9.0
    pos[20:30, 2] = np.nextafter(9.0, 0.0)
    pos[30:35] = [9.0, 0.0, 9.0]
    pos[30:35, 0] -= np.arange(5) * 1.3
    out.append(("faces", pos, tid, 1, dict(domain_size=(9.0, 9.0, 9.0), cutoff=2.5, skin=0.3,
                                            boundary=(P, P, P))))
    return out


def containers():
    space = enumerate_configurations()
    for name, pos, tid, nt, kw in systems():
        params = SimulationParams(rebuild_interval=5, **kw)
        doc = {"pos": pos, "tid": tid, "n_types": np.array(nt),
               "domain": np.asarray(params.domain_size), "cutoff": np.array(params.cutoff),
               "skin": np.array(params.skin),
               "periodic": params.periodic_flags().astype(np.int64)}
        types = _types(nt)
        for csf, tag in ((1.0, "csf1"), (0.5, "csf05")):
            g = make_geometry(params.domain_size, params.interaction_length, csf,
                              params.periodic_flags())
            gs = GridState(g)
            gs.rebuild(ParticleSet(pos.copy(), type_ids=tid, types=types))
            doc[f"{tag}_src"] = gs.src
            doc[f"{tag}_shift"] = gs.shift
            doc[f"{tag}_start"] = gs.start
            doc[f"{tag}_end"] = gs.end
        g = make_geometry(params.domain_size, params.interaction_length, 1.0,
                          params.periodic_flags())
        vl = VerletListState(g)
        vl.rebuild(ParticleSet(pos.copy(), type_ids=tid, types=types))
        doc["vl_nbr"] = vl.nbr
        doc["vl_noff"] = vl.noff
        forces = np.zeros((len(space), len(pos), 3))
        counts = np.zeros(len(space), dtype=np.int64)
        for k, cfg in enumerate(space):
            p = ParticleSet(pos.copy(), type_ids=tid, types=types)
            _, counts[k] = compute_forces(p, cfg, params, workers=1)
            forces[k] = p.forces
        doc["forces"] = forces
        doc["counts"] = counts
        doc["config_ids"] = np.array([c.id for c in space])
        np.savez_compressed(os.path.join(OUT, f"sys_{name}.npz"), **doc)
        print(name, len(pos), counts[:3])


def sc_lattice(n_side, spacing, jitter, seed, offset=0.5):
    """Config-1 style input: sites (i+offset)*spacing + U(-jitter, jitter)."""
    rng = np.random.default_rng(seed)
    i = (np.arange(n_side) + offset) * spacing
    g = np.stack(np.meshgrid(i, i, i, indexing="ij"), axis=-1).reshape(-1, 3)
    pos = g + rng.uniform(-jitter, jitter, g.shape)
    v = rng.normal(0.0, 1.0, pos.shape)
    v -= v.mean(axis=0)
    v *= np.sqrt(0.7 / (np.sum(v * v) / (3.0 * len(v))))
    return pos, v


def trajectories():
    runs = [
        # (name, n_side, offset, steps, config ids)
        ("traj_small", 6, 0.5, 40, ["LC-C08-N3L-SoA-CSF1", "LC-C01-NoN3L-AoS-CSF0.5",
                                    "LC-SLI-NoN3L-AoS-CSF1", "LC-C18-N3L-AoS-CSF0.5",
                                    "VL-List_Iter-NoN3L-SoA"]),
        # sites on the faces: the LC periodic-crossing drop
        ("traj_faces", 6, 0.0, 40, ["LC-C08-N3L-AoS-CSF1", "VL-List_Iter-NoN3L-AoS"]),
        # BASELINE config 1: 8,000 SC sites at (i+0.5)*1.1, jitter 0.05, 100 steps, R=10
        ("traj_config1", 20, 0.5, 100, ["LC-C08-N3L-SoA-CSF1"]),
    ]
    for name, ns, off, steps, ids in runs:
        pos0, vel0 = sc_lattice(ns, 1.1, 0.05, seed=0, offset=off)
        L = ns * 1.1
        doc = {"pos0": pos0, "vel0": vel0, "domain": np.array([L, L, L]), "steps": np.array(steps),
               "config_ids": np.array(ids)}
        for k, cid in enumerate(ids):
            params = SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3,
                                      rebuild_interval=10, delta_t=1e-3,
                                      total_iterations=steps, boundary=(P, P, P))
            p = ParticleSet(pos0.copy(), velocities=vel0.copy(), types=_types(1))  # ParticleSet aliases contiguous input
            rep = simulate(p, params, FixedStrategy(parse_configuration(cid)),
                           tuning_interval=10 ** 9, raise_errors=True)
            assert rep.error is None
            doc[f"pos_{k}"] = np.ascontiguousarray(p.positions)
            doc[f"vel_{k}"] = np.ascontiguousarray(p.velocities)
            doc[f"force_{k}"] = np.ascontiguousarray(p.forces)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **doc)
        print(name, "done")


def reflect_gravity_trajectory():
    """simulate() with reflective walls, gravity and two particle types
    (integrator.py:47-51 apply_gravity, :98-128 apply_boundaries; masses
    1 and 2 enter drift, kick and m*g).  Periodic x, reflective y and z; a
    strong downward g so the bottom layer bounces off the z = 0 wall and
    fast particles bounce off the y walls inside the run.  The number of
    reflections the reference applied is recorded (counted by wrapping its
    apply_boundaries), so the fixture is known to exercise the branch."""
    ns, steps = 7, 90
    rng = np.random.default_rng(11)
    i = (np.arange(ns) + 0.3) * 1.1
    g = np.stack(np.meshgrid(i, i, i, indexing="ij"), axis=-1).reshape(-1, 3)
    pos0 = g + rng.uniform(-0.05, 0.05, g.shape)
    tid = (np.arange(len(pos0)) % 2).astype(np.int64)
    vel0 = rng.normal(0.0, 1.6, pos0.shape)
    L = ns * 1.1
    ids = ["LC-C08-N3L-SoA-CSF1", "LC-C01-NoN3L-AoS-CSF0.5", "LC-SLI-N3L-AoS-CSF1",
           "LC-C18-NoN3L-SoA-CSF1", "VL-List_Iter-NoN3L-SoA", "VL-List_Iter-NoN3L-AoS"]
    doc = {"pos0": pos0, "vel0": vel0, "tid": tid, "domain": np.array([L, L, L]),
           "steps": np.array(steps), "gravity": np.array(-25.0), "dt": np.array(2e-3),
           "periodic": np.array([True, False, False]), "config_ids": np.array(ids)}
    saved = _msim.apply_boundaries
    for k, cid in enumerate(ids):
        hits = [0]

        def counting(p, params, _orig=saved, _hits=hits):
            x = p.positions   # (N, 3) view in either layout
            for ax in (1, 2):
                _hits[0] += int(np.sum((x[:, ax] < 0.0) | (x[:, ax] > L)))
            return _orig(p, params)

        params = SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3, rebuild_interval=6,
                                  delta_t=2e-3, total_iterations=steps, boundary=(P, R, R),
                                  gravity=-25.0)
        p = ParticleSet(pos0.copy(), velocities=vel0.copy(), type_ids=tid.copy(), types=_types(2))
        _msim.apply_boundaries = counting
        try:
            rep = simulate(p, params, FixedStrategy(parse_configuration(cid)),
                           tuning_interval=10 ** 9, raise_errors=True)
        finally:
            _msim.apply_boundaries = saved
        assert rep.error is None
        assert hits[0] > 0, "no reflection happened"
        p.convert_layout("AoS")
        doc[f"pos_{k}"] = np.ascontiguousarray(p.positions)
        doc[f"vel_{k}"] = np.ascontiguousarray(p.velocities)
        doc[f"force_{k}"] = np.ascontiguousarray(p.forces)
        doc[f"reflections_{k}"] = np.array(hits[0])
        print(cid, "reflections", hits[0])
    np.savez_compressed(os.path.join(OUT, "traj_reflect_gravity.npz"), **doc)
    print("traj_reflect_gravity done")


def thermo_and_stats():
    """current_temperature / apply_thermostat (integrator.py:72-95) and
    compute_live_stats (livestats.py:46-77) on seeded inputs."""
    rng = np.random.default_rng(7)
    doc = {}
    # live statistics: (name, positions, domain, cutoff, skin, boundary, threads)
    L = 20.0
    blob = np.clip(rng.normal(10.0, 1.5, (3000, 3)), 0.0, L)
    edges = np.array([[0.0, 0.0, 0.0], [L, L, L], [L, 0.0, 5.0], [19.999999999, 7.0, 0.0]])
    lattice = (np.stack(np.meshgrid(*(np.arange(7) + 0.5,) * 3, indexing="ij"), -1).reshape(-1, 3)
               * (L / 7))
    cases = [("uniform", rng.uniform(0.0, L, (5000, 3)), (L, L, L), 2.5, 0.3, P, 4),
             ("blob", blob, (L, L, L), 2.5, 0.3, R, 1),
             ("edges", edges, (L, L, L), 2.5, 0.3, R, 2),
             ("lattice", lattice, (L, L, L), 2.5, 0.35, P, 8),
             ("empty", np.zeros((0, 3)), (L, L, L), 2.5, 0.3, P, 1),
             ("slab", rng.uniform(0.0, 1.0, (4000, 3)) * (31.3, 9.1, 6.0), (31.3, 9.1, 6.0), 2.5, 0.0, R, 3),
             ("one_bin", rng.uniform(0.0, 3.0, (50, 3)), (3.0, 3.0, 3.0), 2.5, 0.3, R, 1)]
    names = []
    for name, pos, dom, rc, skin, bnd, thr in cases:
        params = SimulationParams(domain_size=dom, cutoff=rc, skin=skin, boundary=(bnd,) * 3,
                                  thread_count=thr)
        p = ParticleSet(pos.copy(), types=_types(1))
        doc[f"ls_{name}_pos"] = pos
        doc[f"ls_{name}_in"] = np.array([*dom, rc, skin, float(bnd == P), thr])
        doc[f"ls_{name}_out"] = compute_live_stats(p, params).feature_vector()
        names.append(name)
    doc["ls_names"] = np.array(names)
    # temperature + thermostat: (name, n, n_types, layout, target, max_dt, zero velocities)
    tcases = [("one", 1, 1, "AoS", 1.0, 0.1, False), ("seven", 7, 2, "SoA", 0.5, 0.2, False),
              ("eight", 8, 1, "AoS", 2.0, 5.0, False), ("odd", 129, 3, "AoS", 0.1, 0.05, False),
              ("mid", 1000, 2, "SoA", 1.3, 0.01, False), ("big", 100003, 2, "AoS", 0.7, 0.2, False),
              ("cold_zero_target", 64, 1, "AoS", 0.0, 0.1, True)]
    tnames = []
    for name, n, nt, layout, target, mdt, zero in tcases:
        vel = np.zeros((n, 3)) if zero else rng.normal(0.0, 1.1, (n, 3))
        tid = rng.integers(0, nt, n)
        p = ParticleSet(rng.uniform(0, 10, (n, 3)), velocities=vel.copy(), type_ids=tid,
                        types=_types(nt))
        p.convert_layout(layout)
        t = current_temperature(p)
        apply_thermostat(p, target, mdt)
        doc[f"th_{name}_vel0"] = vel
        doc[f"th_{name}_tid"] = tid
        doc[f"th_{name}_in"] = np.array([nt, float(layout == "SoA"), target, mdt])
        doc[f"th_{name}_t"] = np.array(t)
        doc[f"th_{name}_vel"] = np.ascontiguousarray(p.velocities)
        tnames.append(name)
    doc["th_names"] = np.array(tnames)
    np.savez_compressed(os.path.join(OUT, "thermo_stats.npz"), **doc)
    print("thermo_stats done")


def tuned_trajectory():
    """simulate() with the real TuningController + FullSearchStrategy over a
    3-configuration space, thermostat on.  The timer is a counter, so every
    candidate costs the same and the controller's tie rule (earliest in the
    space, tuning.py:288-291) decides: the run is deterministic.  The
    per-iteration (configuration, forced, mode) sequence is recorded by
    wrapping the controller."""
    seq = []

    class Recording(TuningController):
        def configuration_for_iteration(self, iteration):
            cfg, forced = super().configuration_for_iteration(iteration)
            seq.append((iteration, cfg.id, bool(forced), self.mode))
            return cfg, forced

    space_ids = ["VL-List_Iter-NoN3L-AoS", "LC-C08-N3L-SoA-CSF1", "LC-C01-NoN3L-AoS-CSF0.5"]
    ns, steps = 6, 40
    pos0, vel0 = sc_lattice(ns, 1.1, 0.05, seed=3, offset=0.5)
    L = ns * 1.1
    params = SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3, rebuild_interval=4,
                              delta_t=1e-3, total_iterations=steps, boundary=(P, P, P),
                              thermostat=ThermostatParams(0.9, 0.05, 7))
    p = ParticleSet(pos0.copy(), velocities=vel0.copy(), types=_types(1))
    counter = iter(range(10 ** 9))
    saved = _msim.TuningController
    _msim.TuningController = Recording
    try:
        rep = simulate(p, params, FullSearchStrategy(), tuning_interval=15, samples_per_config=2,
                       space=[parse_configuration(c) for c in space_ids],
                       timer=lambda: next(counter), raise_errors=True)
    finally:
        _msim.TuningController = saved
    assert rep.error is None
    doc = {"pos0": pos0, "vel0": vel0, "domain": np.array([L, L, L]), "steps": np.array(steps),
           "space": np.array(space_ids), "tuning": np.array([15, 2, 4, 7]),
           "thermo": np.array([0.9, 0.05]),
           "seq_it": np.array([s[0] for s in seq]), "seq_cfg": np.array([s[1] for s in seq]),
           "seq_forced": np.array([s[2] for s in seq]), "seq_mode": np.array([s[3] for s in seq]),
           "pos": np.ascontiguousarray(p.positions), "vel": np.ascontiguousarray(p.velocities),
           "force": np.ascontiguousarray(p.forces), "layout": np.array(p.layout),
           "final_temperature": np.array(rep.final_temperature),
           "trial_iterations": np.array(rep.trial_iterations)}
    np.savez_compressed(os.path.join(OUT, "traj_tuned.npz"), **doc)
    print("traj_tuned done", rep.phase_selections)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    only = sys.argv[1:]
    if not only or "geometry" in only:
        geometry_cases()
    if not only or "containers" in only:
        containers()
    if not only or "trajectories" in only:
        trajectories()
    if not only or "reflect_gravity" in only:
        reflect_gravity_trajectory()
    if not only or "thermo_stats" in only:
        thermo_and_stats()
    if not only or "tuned" in only:
        tuned_trajectory()
