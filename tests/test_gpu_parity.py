"""GPU parity: libmdg through its C ABI against the oracle and the reference's
golden outputs (tests/golden/, generated from the reference by
oracle/make_golden.py).

Bars (BASELINE north_star): cell assignments and Verlet pair sets bit-exact;
eval counts exact; fp64 forces and trajectories within 1e-10 relative
(Frobenius norm, tests/conftest.py:55-60 of the reference).
"""

import numpy as np
import pytest

from conftest import golden, system_names
from oracle import port
from test_gpu_scale import _band_pairs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FP64_TOL = 1e-10


def _ids():
    return [c.id for c in port.all_configs()]


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA")
    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200 import calculator
    return P, calculator


def _system(P, d, layout="AoS"):
    nt = int(d["n_types"])
    types = [P.ParticleTypeInfo(t, 1.0 + 0.5 * t, 1.0 - 0.2 * t, 1.0 + t) for t in range(nt)]
    per = tuple(P.PERIODIC if f else P.REFLECTIVE for f in d["periodic"])
    params = P.SimulationParams(domain_size=d["domain"], cutoff=float(d["cutoff"]),
                                skin=float(d["skin"]), rebuild_interval=5, boundary=per)
    parts = P.ParticleSet(d["pos"], type_ids=d["tid"], types=types, layout=layout)
    return parts, params


@pytest.mark.parametrize("name", system_names())
def test_all_30_configurations_match_reference(pkg, name):
    P, calc = pkg
    d = golden(f"sys_{name}.npz")
    assert [str(s) for s in d["config_ids"]] == _ids()
    for k, cfg in enumerate(P.enumerate_configurations()):
        parts, params = _system(P, d)
        _, count = calc.compute_forces(parts, cfg, params)
        assert count == int(d["counts"][k]), cfg.id
        err = port.force_rel_error(parts.numpy("force"), d["forces"][k])
        assert err <= FP64_TOL, f"{cfg.id}: {err:.3g}"


@pytest.mark.parametrize("name", system_names())
def test_cell_assignment_bit_exact(pkg, name):
    P, calc = pkg
    d = golden(f"sys_{name}.npz")
    for csf, tag in ((1.0, "csf1"), (0.5, "csf05")):
        for layout in ("AoS", "SoA"):
            parts, params = _system(P, d, layout)
            fc = calc.ForceCalculator(parts, params)
            cfg = P.Configuration("LC", "C08", True, layout, csf)
            fc.rebuild(parts, cfg)
            g = fc.grid_state(csf)
            assert np.array_equal(g["src"], d[f"{tag}_src"]), (tag, layout)
            assert np.array_equal(g["shift"], d[f"{tag}_shift"]), (tag, layout)
            assert np.array_equal(g["start"], d[f"{tag}_start"]), (tag, layout)
            assert np.array_equal(g["end"], d[f"{tag}_end"]), (tag, layout)
            fc.close()


@pytest.mark.parametrize("name", system_names())
def test_verlet_pair_sets_bit_exact(pkg, name):
    P, calc = pkg
    d = golden(f"sys_{name}.npz")
    for layout in ("AoS", "SoA"):
        parts, params = _system(P, d, layout)
        fc = calc.ForceCalculator(parts, params)
        fc.rebuild(parts, P.parse_configuration(f"VL-List_Iter-NoN3L-{layout}"))
        noff, nbr = fc.verlet_lists()
        assert np.array_equal(noff, d["vl_noff"])
        assert np.array_equal(nbr, d["vl_nbr"])
        fc.close()


@pytest.mark.parametrize("name", system_names())
def test_lc_pair_sets_bit_exact(pkg, name):
    """the pairs the LC traversals evaluate within rc
    (mdg_lc_pairs, owner pairs on pos[src] + shift) equal the reference's
    Verlet pairs filtered to minimum-image r^2 < rc^2 -- as sorted pair lists,
    at both cell-size factors."""
    P, calc = pkg
    d = golden(f"sys_{name}.npz")
    pos, L = d["pos"], np.asarray(d["domain"], dtype=np.float64)
    per = np.asarray(d["periodic"], dtype=bool)
    rc2 = float(d["cutoff"]) ** 2
    noff, nbr = d["vl_noff"], d["vl_nbr"]
    i = np.repeat(np.arange(len(noff) - 1), np.diff(noff))
    j = nbr.astype(np.int64)
    keep = i < j
    i, j = i[keep], j[keep]
    dd = pos[i] - pos[j]
    dd[:, per] -= L[per] * np.rint(dd[:, per] / L[per])   # kernels.py:739-757
    r2 = dd[:, 0] * dd[:, 0] + dd[:, 1] * dd[:, 1] + dd[:, 2] * dd[:, 2]
    ref = np.unique(np.stack([i[r2 < rc2], j[r2 < rc2]], 1), axis=0)
    for csf in (1.0, 0.5):
        parts, params = _system(P, d)
        fc = calc.ForceCalculator(parts, params)
        fc.rebuild(parts, P.Configuration("LC", "C01", False, "AoS", csf))
        got = fc.lc_pairs(csf)
        fc.close()
        assert np.array_equal(got, ref), (name, csf, len(got), len(ref))


def test_device_timings_export(pkg):
    """mdg_timings: device-event build (rebuild + refresh) and force (compute)
    intervals, the reference's timing hooks (simulation.py:155-181)."""
    P, calc = pkg
    d = golden("sys_blob.npz")
    parts, params = _system(P, d)
    fc = calc.ForceCalculator(parts, params)
    cfg = P.parse_configuration("LC-C08-N3L-AoS-CSF1")
    assert fc.timings() == (-1, -1)
    fc.timings(True)
    fc.rebuild(parts, cfg)
    fc.refresh(parts, cfg)
    fc.compute(parts, cfg)
    b, f = fc.timings()
    assert b > 0 and f > 0
    fc.timings(False)
    assert fc.timings() == (-1, -1)
    fc.close()


@pytest.mark.parametrize("traj", ["traj_small", "traj_faces", "traj_config1"])
def test_trajectories_match_reference(pkg, traj):
    P, calc = pkg
    from paper_2505_03438_b200.simulation import simulate
    z = golden(f"{traj}.npz")
    L = z["domain"]
    for k, cid in enumerate(str(s) for s in z["config_ids"]):
        params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                                    delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
        parts = P.ParticleSet(z["pos0"], z["vel0"])
        rep = simulate(parts, params, P.parse_configuration(cid), steps=int(z["steps"]))
        assert rep.error is None, rep.error
        dpos = parts.numpy("pos") - z[f"pos_{k}"]
        dpos -= L * np.rint(dpos / L)   # positions compared modulo the box
        assert np.linalg.norm(dpos) / np.linalg.norm(z[f"pos_{k}"]) <= FP64_TOL, cid
        assert port.force_rel_error(parts.numpy("vel"), z[f"vel_{k}"]) <= FP64_TOL, cid


def test_host_drop_in_drives_the_reference_loop(pkg):
    """HostForceCalculator inside the oracle's restatement of simulate()
    (the reference loop with numpy host arrays) reproduces the reference."""
    P, calc = pkg
    z = golden("traj_small.npz")
    L = float(z["domain"][0])
    for k, cid in enumerate(str(s) for s in z["config_ids"]):
        params = port.Params(domain_size=(L, L, L), cutoff=2.5, skin=0.3, rebuild_interval=10,
                             delta_t=1e-3, boundary=(port.PERIODIC,) * 3)
        p = port.Particles(z["pos0"], z["vel0"])
        port.simulate_fixed(p, params, port.parse(cid), steps=int(z["steps"]),
                            calculator_cls=calc.HostForceCalculator)
        assert port.force_rel_error(p.velocities, z[f"vel_{k}"]) <= FP64_TOL, cid


def test_lattice_32k_all_configs_vs_oracle(pkg):
    """Mid-size parity against the oracle (config-1 style lattice, 32,768)."""
    P, calc = pkg
    from paper_2505_03438_b200 import systems
    pos, _, L = systems.sc_lattice(n_side=32, seed=3)
    pp = port.Params(domain_size=L, cutoff=2.5, skin=0.3, boundary=(port.PERIODIC,) * 3)
    ref = port.Particles(pos)
    _, ref_count = port.compute_forces(ref, port.parse("LC-C08-N3L-AoS-CSF1"), pp, workers=4)
    ref_f = np.asarray(ref.forces)
    params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, boundary=(P.PERIODIC,) * 3)
    for cfg in P.enumerate_configurations():
        parts = P.ParticleSet(pos)
        _, count = calc.compute_forces(parts, cfg, params)
        assert count == ref_count * (1 if cfg.newton3 else 2), cfg.id
        assert port.force_rel_error(parts.numpy("force"), ref_f) <= FP64_TOL, cfg.id


def test_empty_set_and_layout_mismatch(pkg):
    P, calc = pkg
    params = P.SimulationParams(domain_size=(9.0, 9.0, 9.0), cutoff=2.5, skin=0.3,
                                boundary=(P.PERIODIC,) * 3)
    for cfg in P.enumerate_configurations():
        parts = P.ParticleSet(np.zeros((0, 3)))
        _, count = calc.compute_forces(parts, cfg, params)
        assert count == 0
    # the loop on an empty set, native spans included (mdg_run)
    from paper_2505_03438_b200.simulation import Simulation
    for cid in ("VL-List_Iter-NoN3L-SoA", "LC-C08-N3L-AoS-CSF1", "VCL-ClusterIter-NoN3L-SoA"):
        cfg = P.parse_configuration(cid)
        parts = P.ParticleSet(np.zeros((0, 3)), layout=cfg.layout)
        sim = Simulation(parts, params, cfg, fuse_kick_drift=True)
        sim.run(13, record=False)
        sim.check()
        assert sim.iteration == 13 and sim.calc.last_eval_count == 0
    parts = P.ParticleSet(np.random.default_rng(0).uniform(0, 9, (20, 3)))
    fc = calc.ForceCalculator(parts, params)
    cfg = P.parse_configuration("LC-C08-N3L-SoA-CSF1")
    fc.rebuild(parts, cfg)
    with pytest.raises(ValueError):
        fc.compute(parts, cfg)


def test_hand_cases(pkg):
    P, calc = pkg
    refl = P.SimulationParams(domain_size=(10.0, 10.0, 10.0), cutoff=2.5, skin=0.3,
                              boundary=(P.REFLECTIVE,) * 3)
    r_min = 2.0 ** (1.0 / 6.0)
    for cid in ("LC-C08-N3L-AoS-CSF1", "LC-C18-N3L-SoA-CSF0.5", "VL-List_Iter-NoN3L-SoA"):
        parts = P.ParticleSet(np.array([[4.0, 5.0, 5.0], [4.0 + r_min, 5.0, 5.0]]))
        calc.compute_forces(parts, P.parse_configuration(cid), refl)
        assert np.max(np.abs(parts.numpy("force"))) <= 1e-12
    box12 = P.SimulationParams(domain_size=(12.0, 12.0, 12.0), cutoff=2.5, skin=0.3,
                               boundary=(P.REFLECTIVE,) * 3)
    for cid in ("LC-SLI-N3L-AoS-CSF1", "LC-C01-NoN3L-SoA-CSF1", "VL-List_Iter-NoN3L-AoS"):
        parts = P.ParticleSet(np.array([[4.0, 6.0, 6.0], [5.5, 6.0, 6.0], [7.0, 6.0, 6.0]]))
        calc.compute_forces(parts, P.parse_configuration(cid), box12)
        f = parts.numpy("force")
        assert np.allclose(f[1], 0.0, atol=1e-12)
        assert np.allclose(f[0], -f[2], atol=1e-12)
        assert abs(f[0][0]) > 0.1
    per = P.SimulationParams(domain_size=(9.0, 9.0, 9.0), cutoff=2.5, skin=0.3,
                             boundary=(P.PERIODIC,) * 3)
    pos = np.array([[0.3, 4.5, 4.5], [8.7, 4.5, 4.5]])
    ref, _ = port.brute_forces(pos, np.zeros(2, dtype=np.int64), [1.0], [1.0], 2.5,
                               per.domain_size, per.periodic_flags())
    for cid in ("LC-C08-N3L-AoS-CSF1", "VL-List_Iter-NoN3L-AoS"):
        parts = P.ParticleSet(pos)
        calc.compute_forces(parts, P.parse_configuration(cid), per)
        assert np.allclose(parts.numpy("force"), ref, atol=1e-12)
    vlp = P.SimulationParams(domain_size=(14.0, 14.0, 14.0), cutoff=3.0, skin=0.5,
                             boundary=(P.REFLECTIVE,) * 3)
    parts = P.ParticleSet(np.array([[3.0, 7.0, 7.0], [6.4, 7.0, 7.0], [10.0, 7.0, 7.0]]))
    fc = calc.ForceCalculator(parts, vlp)
    fc.rebuild(parts, P.parse_configuration("VL-List_Iter-NoN3L-AoS"))
    noff, nbr = fc.verlet_lists()
    assert [set(nbr[noff[i]:noff[i + 1]].tolist()) for i in range(3)] == [{1}, {0}, set()]


@pytest.mark.parametrize("name", ["small_periodic", "mixed", "crit1_0", "tight", "blob"])
def test_potential_energy_matches_reference_helper(pkg, name):
    """Shifted LJ potential energy vs the reference's brute-force energy helper
    (tests/test_integrator.py:227-247), fp64 tolerance."""
    P, calc = pkg
    d = golden(f"sys_{name}.npz")
    parts, params = _system(P, d)
    fc = calc.ForceCalculator(parts, params)
    pe = fc.potential_energy(parts)
    nt = int(d["n_types"])
    ref = port.brute_potential(d["pos"], d["tid"], [1.0 + 0.5 * t for t in range(nt)],
                               [1.0 - 0.2 * t for t in range(nt)], params.cutoff,
                               params.domain_size, params.periodic_flags())
    assert abs(pe - ref) <= FP64_TOL * max(1.0, abs(ref)), (pe, ref)
    fc.close()


def test_energy_conserved_on_device(pkg):
    """Device loop + PE: total energy drift <= 1e-3 over 1000 small steps
    (the reference's criterion, tests/test_integrator.py:250-275)."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    rng = np.random.default_rng(11)
    side = np.arange(6) * 1.4 + 0.5
    pos = np.array(np.meshgrid(side, side, side)).reshape(3, -1).T[:120]
    pos = pos + rng.uniform(-0.05, 0.05, pos.shape)
    vel = rng.normal(0.0, 0.4, pos.shape)
    params = P.SimulationParams(domain_size=(9.0, 9.0, 9.0), cutoff=2.5, skin=0.3,
                                rebuild_interval=10, delta_t=1e-4, boundary=(P.PERIODIC,) * 3)
    parts = P.ParticleSet(pos, vel)
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-AoS")
    sim = Simulation(parts, params, cfg)

    def energy():
        kin = 0.5 * float((parts.numpy("vel") ** 2).sum())
        return kin + sim.calc.potential_energy(parts)

    sim.step()            # iteration 0 drifts with zero force (simulation.py:7-8)
    e0 = energy()
    sim.run(1000, record=False)
    assert abs(energy() - e0) / abs(e0) <= 1e-3


def test_host_resident_loop_matches_reference(pkg):
    """hostloop.HostSimulation (pinned host state, GPU forces, native host
    integrator) reproduces the reference trajectories."""
    P, calc = pkg
    from paper_2505_03438_b200.hostloop import HostParticleSet, HostSimulation
    z = golden("traj_small.npz")
    L = z["domain"]
    for k, cid in enumerate(str(s) for s in z["config_ids"]):
        params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                                    delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
        p = HostParticleSet(z["pos0"], z["vel0"])
        HostSimulation(p, params, P.parse_configuration(cid)).run(int(z["steps"]))
        assert port.force_rel_error(p.velocities, z[f"vel_{k}"]) <= FP64_TOL, cid


@pytest.mark.parametrize("name", ["small_periodic", "mixed", "crit1_0", "crit1_1", "blob", "faces"])
def test_fp32_variant_within_1e4(pkg, name):
    """fp32-compute / fp64-accumulate Verlet walk: forces within 1e-4 of the
    reference (north_star tolerance for the fp32 variant)."""
    P, calc = pkg
    d = golden(f"sys_{name}.npz")
    k = _ids().index("VL-List_Iter-NoN3L-AoS")
    for layout in ("AoS", "SoA"):
        parts, params = _system(P, d, layout)
        _, count = calc.compute_forces(parts, P.parse_configuration(f"VL-List_Iter-NoN3L-{layout}-FP32"),
                                       params)
        err = port.force_rel_error(parts.numpy("force"), d["forces"][k])
        assert err <= 1e-4, (layout, err)
        # only pairs within the fp32 rounding band of rc may flip (none here:
        # the count must then be exact)
        band = _band_pairs(d["pos"], d["vl_noff"], d["vl_nbr"], params)
        assert abs(count - int(d["counts"][k])) <= 2 * band, (layout, count, int(d["counts"][k]), band)


# -- §8(f): live statistics, temperature/thermostat, tuned loop on device ------

def test_live_stats_bit_exact(pkg):
    P, calc = pkg
    z = golden("thermo_stats.npz")
    for name in (str(s) for s in z["ls_names"]):
        a = z[f"ls_{name}_in"]
        per = P.PERIODIC if a[5] else P.REFLECTIVE
        params = P.SimulationParams(domain_size=a[:3], cutoff=float(a[3]), skin=float(a[4]),
                                    boundary=(per,) * 3, thread_count=int(a[6]))
        for layout in ("AoS", "SoA"):
            parts = P.ParticleSet(z[f"ls_{name}_pos"], layout=layout)
            fc = calc.ForceCalculator(parts, params)
            got = fc.live_stats(parts).feature_vector()
            again = fc.live_stats(parts).feature_vector()       # cached plan, re-zeroed buffers
            fc.close()
            assert np.array_equal(got, z[f"ls_{name}_out"]), (name, layout, got, z[f"ls_{name}_out"])
            assert np.array_equal(again, got)


def test_temperature_and_thermostat_bit_exact(pkg):
    P, calc = pkg
    z = golden("thermo_stats.npz")
    params = P.SimulationParams(domain_size=(10.0, 10.0, 10.0), cutoff=2.5, skin=0.3)
    for name in (str(s) for s in z["th_names"]):
        nt, soa, target, mdt = z[f"th_{name}_in"]
        nt = int(nt)
        vel0 = z[f"th_{name}_vel0"]
        types = [P.ParticleTypeInfo(t, 1.0 + 0.5 * t, 1.0 - 0.2 * t, 1.0 + t) for t in range(nt)]
        parts = P.ParticleSet(np.full_like(vel0, 5.0), vel0, type_ids=z[f"th_{name}_tid"], types=types,
                              layout="SoA" if soa else "AoS")
        fc = calc.ForceCalculator(parts, params)
        assert fc.temperature(parts) == float(z[f"th_{name}_t"]), name
        fc.thermostat(parts, float(target), float(mdt))
        assert fc.status_flags() == 0
        fc.close()
        assert np.array_equal(parts.numpy("vel"), z[f"th_{name}_vel"]), name


def test_thermostat_zero_velocity_error_and_empty(pkg):
    P, calc = pkg
    params = P.SimulationParams(domain_size=(10.0, 10.0, 10.0), cutoff=2.5, skin=0.3,
                                boundary=(P.PERIODIC,) * 3,
                                thermostat=P.ThermostatParams(1.0, 0.1, 1))
    g = np.array([2.0, 6.0])
    sites = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)   # 4 apart: no pair forces
    parts = P.ParticleSet(sites)
    rep = P.simulate(parts, params, P.parse_configuration("LC-C08-N3L-AoS-CSF1"), steps=3)
    # reference: apply_thermostat raises ValueError at iteration 0 (integrator.py:84-88)
    assert rep.error is not None and rep.error.startswith("ValueError"), rep.error
    empty = P.ParticleSet(np.zeros((0, 3)))
    fc = calc.ForceCalculator(empty, params)
    with pytest.raises(ValueError):
        fc.temperature(empty)
    fc.close()


def test_tuned_loop_replays_reference_controller(pkg):
    """The reference's TuningController run (FullSearch over VL / LC-C08-SoA /
    LC-C01-CSF0.5, thermostat every 7) replayed through the device loop:
    same configuration per iteration, device timings delivered for exactly
    the trial iterations, final state within the fp64 bar."""
    from conftest import ScriptedController
    P, calc = pkg
    z = golden("traj_tuned.npz")
    L = float(z["domain"][0])
    interval, spc, R, tint = (int(x) for x in z["tuning"])
    params = P.SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3, rebuild_interval=R,
                                delta_t=1e-3, total_iterations=int(z["steps"]),
                                boundary=(P.PERIODIC,) * 3,
                                thermostat=P.ThermostatParams(float(z["thermo"][0]),
                                                              float(z["thermo"][1]), tint))
    parts = P.ParticleSet(z["pos0"], z["vel0"])
    ctl = ScriptedController(z, P.parse_configuration)
    rep = P.simulate(parts, params, None, controller=ctl, tuning_interval=interval)
    assert rep.error is None, rep.error
    assert rep.configuration_sequence() == [str(s) for s in z["seq_cfg"]]
    assert ctl.trial_iterations == int(z["trial_iterations"])
    assert all(f > 0 for f, _ in ctl.timings)
    forced = [bool(f) for f in z["seq_forced"]]
    assert all(r.rebuilt for r, f in zip(rep.records, forced) if f)
    assert parts.layout == str(z["layout"])
    dpos = parts.numpy("pos") - z["pos"]
    dpos -= L * np.rint(dpos / L)
    assert np.linalg.norm(dpos) / np.linalg.norm(z["pos"]) <= FP64_TOL
    assert port.force_rel_error(parts.numpy("vel"), z["vel"]) <= FP64_TOL
    assert port.force_rel_error(parts.numpy("force"), z["force"]) <= FP64_TOL
    assert abs(rep.final_temperature - float(z["final_temperature"])) <= 1e-10 * float(z["final_temperature"])


# -- Verlet cluster lists (north_star container; no reference implementation:
#    the oracle is the reference's own Verlet-list forces and counts) ----------

VCL_IDS = ["VCL-ClusterIter-N3L-AoS", "VCL-ClusterIter-N3L-SoA",
           "VCL-ClusterIter-NoN3L-AoS", "VCL-ClusterIter-NoN3L-SoA"]


@pytest.mark.parametrize("name", system_names())
def test_vcl_matches_reference_forces_and_counts(pkg, name):
    P, calc = pkg
    d = golden(f"sys_{name}.npz")
    ids = [str(s) for s in d["config_ids"]]
    k_vl = ids.index("VL-List_Iter-NoN3L-AoS")
    for cid in VCL_IDS:
        cfg = P.parse_configuration(cid)
        parts, params = _system(P, d, layout=cfg.layout)
        _, count = calc.compute_forces(parts, cfg, params)
        want = int(d["counts"][k_vl]) // (2 if cfg.newton3 else 1)
        assert count == want, (cid, count, want)
        err = port.force_rel_error(parts.numpy("force"), d["forces"][k_vl])
        assert err <= FP64_TOL, f"{cid}: {err:.3g}"


def test_vcl_trajectory_matches_reference(pkg):
    P, calc = pkg
    from paper_2505_03438_b200.simulation import simulate
    z = golden("traj_small.npz")
    L = float(z["domain"][0])
    ids = [str(s) for s in z["config_ids"]]
    k = ids.index("VL-List_Iter-NoN3L-SoA")
    for cid in ("VCL-ClusterIter-N3L-SoA", "VCL-ClusterIter-NoN3L-AoS"):
        params = P.SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3, rebuild_interval=10,
                                    delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
        parts = P.ParticleSet(z["pos0"], z["vel0"])
        rep = simulate(parts, params, P.parse_configuration(cid), steps=int(z["steps"]))
        assert rep.error is None, rep.error
        dpos = parts.numpy("pos") - z[f"pos_{k}"]
        dpos -= L * np.rint(dpos / L)
        assert np.linalg.norm(dpos) / np.linalg.norm(z[f"pos_{k}"]) <= FP64_TOL, cid
        assert port.force_rel_error(parts.numpy("vel"), z[f"vel_{k}"]) <= FP64_TOL, cid


def test_device_wrap_matches_np_mod_on_edges(pkg):
    """drift_wrap_kernel's np.mod fast path vs numpy, bit for bit (zero
    velocity and force: the drift is the identity, only the wrap acts)."""
    P, calc = pkg
    L = 11.18183
    e = np.nextafter
    xs = np.array([0.0, -0.0, 1e-300, -1e-300, -5e-324, L, e(L, 0), e(L, 3 * L), 2 * L, e(2 * L, 0),
                   -L, e(-L, 0), -1e-17, -L / 3, 1.5 * L, 0.7 * L])
    xs = np.concatenate([xs, np.random.default_rng(3).uniform(-L, 2 * L, 5000)])
    pos = np.repeat(xs[:, None], 3, axis=1)
    params = P.SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3,
                                boundary=(P.PERIODIC,) * 3)
    for layout in ("AoS", "SoA"):
        parts = P.ParticleSet(pos, layout=layout)
        fc = calc.ForceCalculator(parts, params)
        fc.drift_wrap(parts, 0.001)
        assert not fc.blowup()
        fc.close()
        got = parts.numpy("pos")
        assert np.array_equal(got.view(np.uint64), np.mod(pos, L).view(np.uint64)), layout


def test_pipelined_host_loop_is_bit_identical(pkg):
    """Chunked host loop (drift/upload and download/kick overlapped) vs the
    one-shot loop: identical bits, LC / VL / VCL, AoS and SoA."""
    P, calc = pkg
    from paper_2505_03438_b200.hostloop import HostParticleSet, HostSimulation
    z = golden("traj_small.npz")
    L = z["domain"]
    for cid in ("LC-C08-N3L-SoA-CSF1", "VL-List_Iter-NoN3L-AoS", "VL-List_Iter-NoN3L-SoA",
                "VCL-ClusterIter-NoN3L-AoS"):
        out = []
        # one-shot steps; one cross-step pipelined run (odd); runs of uneven
        # lengths (even totals in between, rebuild cadence across calls)
        for chunks, runs in ((1, (25,)), (7, (25,)), (3, (4, 1, 20))):
            params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                                        delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
            p = HostParticleSet(z["pos0"], z["vel0"])
            sim = HostSimulation(p, params, P.parse_configuration(cid), chunks=chunks)
            for k in runs:
                sim.run(k)
            assert sim.iteration == 25 and sim.since == 25 % 11 - 1
            out.append((np.array(p.positions), np.array(p.velocities), np.array(p.forces),
                        np.array(p.old_forces)))
        for other in out[1:]:
            for a, b in zip(out[0], other):
                assert np.array_equal(a, b), cid


def test_pipelined_host_run_typed_gravity_reflective(pkg):
    """mdg_host_run with two types, gravity and reflective axes (the fused
    kick+drift pass falls back to its two-pass form there) vs one-shot steps."""
    P, calc = pkg
    from paper_2505_03438_b200.hostloop import HostParticleSet, HostSimulation
    z = golden("traj_small.npz")
    L = z["domain"]
    n = len(z["pos0"])
    tid = np.arange(n) % 2
    for boundary in ((P.PERIODIC,) * 3, (P.REFLECTIVE, P.PERIODIC, P.REFLECTIVE)):
        out = []
        for chunks in (1, 5):
            params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4,
                                        delta_t=1e-3, boundary=boundary, gravity=-0.5)
            p = HostParticleSet(z["pos0"], z["vel0"], tid, sigma=[1.0, 0.9], epsilon=[1.0, 1.2],
                                mass=[1.0, 1.5], layout="SoA")
            sim = HostSimulation(p, params, P.parse_configuration("VL-List_Iter-NoN3L-SoA"),
                                 chunks=chunks)
            sim.run(6)
            sim.run(7)
            out.append((np.array(p.positions), np.array(p.velocities), np.array(p.forces),
                        np.array(p.old_forces)))
        for a, b in zip(*out):
            assert np.array_equal(a, b), boundary


def test_fused_kick_matches_separate_kick(pkg):
    """mdg_compute_kick with the kick fused into the tiled walk (opt-in,
    MDG_FUSE_KICK=1) gives the same trajectory as compute + finish_kick."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, '.')\n"
        "from conftest import golden\n"
        "import paper_2505_03438_b200 as P\n"
        "from paper_2505_03438_b200.simulation import simulate\n"
        "z = golden('traj_small.npz'); L = z['domain']\n"
        "params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,"
        " delta_t=1e-3, boundary=(P.PERIODIC,) * 3, gravity=-0.5)\n"
        "parts = P.ParticleSet(z['pos0'], z['vel0'])\n"
        "rep = simulate(parts, params, P.parse_configuration('VL-List_Iter-NoN3L-AoS'), steps=30)\n"
        "assert rep.error is None\n"
        "np.save(sys.argv[1], np.concatenate([parts.numpy('pos').ravel(), parts.numpy('vel').ravel()]))\n")
    import os
    import tempfile
    here = os.path.dirname(os.path.abspath(__file__))
    out = []
    for fuse in ("0", "1"):
        f = os.path.join(tempfile.mkdtemp(), "state.npy")
        env = dict(os.environ, MDG_FUSE_KICK=fuse, PYTHONPATH=os.path.dirname(here))
        subprocess.run([sys.executable, "-c", code, f], cwd=here, env=env, check=True)
        out.append(np.load(f))
    assert np.array_equal(out[0], out[1])


def test_gpu_training_sweep_writes_reference_csv(pkg, tmp_path):
    """§8(f) row 3: device-timed static-snapshot trials labelled into the
    reference's dataset format; features equal the reference's live stats."""
    import csv as _csv
    P, calc = pkg
    from paper_2505_03438_b200 import dataset
    z = golden("thermo_stats.npz")
    points = []
    for name in ("uniform", "blob"):
        a = z[f"ls_{name}_in"]
        per = P.PERIODIC if a[5] else P.REFLECTIVE
        params = P.SimulationParams(domain_size=a[:3], cutoff=float(a[3]), skin=float(a[4]),
                                    rebuild_interval=10, boundary=(per,) * 3, thread_count=int(a[6]))
        points.append((P.ParticleSet(z[f"ls_{name}_pos"]), params))
    space = [P.parse_configuration(c) for c in ("LC-C08-N3L-AoS-CSF1", "VL-List_Iter-NoN3L-SoA",
                                                "VCL-ClusterIter-NoN3L-AoS")]
    out = tmp_path / "gpu.csv"
    assert dataset.generate_training_dataset(out, points, space=space, trial_iterations=3) == 2
    rows = list(_csv.reader(open(out)))
    assert rows[0] == dataset.dataset_columns(space)
    for (name, row) in zip(("uniform", "blob"), rows[1:]):
        feats = [float(x) for x in row[:8]]
        assert feats == list(z[f"ls_{name}_out"]), name
        costs = {c.id: float(x) for c, x in zip(space, row[8:-1])}
        assert all(0 < v < float("inf") for v in costs.values())
        assert row[-1] == min(space, key=lambda c: costs[c.id]).id


@pytest.mark.parametrize("env", [{"MDG_VLT_WIN": "64"}, {"MDG_VLT_WIN": "256"}, {"MDG_VLT_ORDER": "2"}, {"MDG_VL_TILED": "0"},
                                 {"MDG_VLT_STAGES": "3", "MDG_VLT_WIN": "1024"},
                                 {"MDG_LC_ROWS": "0", "_prefix": "LC-C18"},
                                 {"MDG_LC_C08": "0", "_prefix": "LC-C08"},
                                 {"MDG_LC_C08": "2", "_prefix": "LC-C08"},
                                 {"MDG_VL_CAP0": "8"}, {"MDG_VL_CAP0": "8", "MDG_VLT_SPECULATE": "0"},
                                 {"MDG_VLT_SPECULATE": "0", "MDG_VLT_WIN": "256"},
                                 {"MDG_LC_C08_ALL": "0", "_prefix": "LC-C08"},
                                 {"MDG_LC_C08_LISTS": "0", "_prefix": "LC-C08"},
                                 {"MDG_LC_C08_ALL": "3", "_prefix": "LC-C08"}])
def test_vl_walk_variants_match_reference(pkg, env):
    """The tunable paths of the Verlet walk against the reference forces and
    counts: a tiny window budget (most tiles overflow to the row-space walk),
    bank-aware list order, the untiled walk, a 3-stage window ring, a list
    capacity guessed far too small (the build's capacity retry, with the first
    walk queued before the build's check and without); and the alternative
    linked-cell realisations (C18 per-colour warp tiles, C08 warp tiles, C08
    in one launch with atomics, colour by colour, without per-unit lists, with
    the colour partials added in the fold)."""
    env = dict(env)
    prefix = env.pop("_prefix", "VL-")
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, '.')\n"
        "import numpy as np\n"
        "from conftest import golden, system_names\n"
        "from oracle import port\n"
        "import paper_2505_03438_b200 as P\n"
        "from paper_2505_03438_b200 import calculator as calc\n"
        "for name in system_names():\n"
        "    d = golden(f'sys_{name}.npz')\n"
        "    ids = [str(s) for s in d['config_ids']]\n"
        "    nt = int(d['n_types'])\n"
        "    types = [P.ParticleTypeInfo(t, 1.0 + 0.5 * t, 1.0 - 0.2 * t, 1.0 + t) for t in range(nt)]\n"
        "    per = tuple(P.PERIODIC if f else P.REFLECTIVE for f in d['periodic'])\n"
        "    params = P.SimulationParams(domain_size=d['domain'], cutoff=float(d['cutoff']),"
        " skin=float(d['skin']), rebuild_interval=5, boundary=per)\n"
        "    for cid in ids:\n"
        f"        if not cid.startswith({prefix!r}): continue\n"
        "        parts = P.ParticleSet(d['pos'], type_ids=d['tid'], types=types,"
        " layout=P.parse_configuration(cid).layout)\n"
        "        _, count = calc.compute_forces(parts, P.parse_configuration(cid), params)\n"
        "        k = ids.index(cid)\n"
        "        assert count == int(d['counts'][k]), (name, cid)\n"
        "        err = port.force_rel_error(parts.numpy('force'), d['forces'][k])\n"
        "        assert err <= 1e-10, (name, cid, err)\n"
        "print('ok')\n")
    here = os.path.dirname(os.path.abspath(__file__))
    e = dict(os.environ, PYTHONPATH=os.path.dirname(here), **env)
    r = subprocess.run([sys.executable, "-c", code], cwd=here, env=e, capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


# -- BASELINE full size (config 2: 1,048,576 particles) through size-independent
#    properties (the oracle would take minutes at this size) -------------------

def test_full_size_configurations_agree(pkg, config2_snapshot):
    """At 1,048,576 particles every container family gives the same forces
    (fp64 bar; fp32 variant 1e-4), N3L counts are half the NoN3L counts, and
    the total force vanishes (Newton's third law, momentum conservation)."""
    P, calc = pkg
    pos, vel, params = config2_snapshot
    ids = ["VL-List_Iter-NoN3L-SoA", "VL-List_Iter-NoN3L-AoS", "LC-SLI-N3L-SoA-CSF0.5",
           "LC-C08-N3L-AoS-CSF1", "LC-C01-NoN3L-SoA-CSF1", "VCL-ClusterIter-N3L-AoS",
           "VCL-ClusterIter-NoN3L-SoA", "VL-List_Iter-NoN3L-AoS-FP32"]
    ref, ref_count = None, None
    for cid in ids:
        cfg = P.parse_configuration(cid)
        parts = P.ParticleSet(pos, layout=cfg.layout)
        _, count = calc.compute_forces(parts, cfg, params)
        f = parts.numpy("force")
        directed = count if not cfg.newton3 else 2 * count
        if ref is None:
            ref, ref_count = f, directed
            total = np.abs(f.sum(axis=0)).max() / np.abs(f).sum(axis=0).max()
            assert total <= 1e-12, total
            continue
        if cfg.precision == "fp32":   # pairs within fp32 rounding of rc may flip
            assert abs(directed - ref_count) <= 1e-6 * ref_count, (cid, directed, ref_count)
        else:
            assert directed == ref_count, (cid, directed, ref_count)
        tol = 1e-4 if cfg.precision == "fp32" else FP64_TOL
        assert port.force_rel_error(f, ref) <= tol, cid


def test_full_size_energy_conservation(pkg, config2_snapshot):
    """200 NVE steps of config 2 on the tiled Verlet walk: total energy drift
    stays at the integrator's level (relative 1e-4)."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    pos, vel, params = config2_snapshot
    parts = P.ParticleSet(pos, vel, layout="SoA")
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    sim = Simulation(parts, params, cfg)

    def energy():
        v = parts.numpy("vel")
        return 0.5 * float(np.sum(v * v)) + sim.calc.potential_energy(parts, rebuild=True)

    e0 = energy()
    sim.run(200, record=False)
    sim.check()
    e1 = energy()
    assert abs(e1 - e0) / abs(e0) <= 1e-4, (e0, e1)


def test_step_graph_is_bit_identical(pkg):
    """§8(f) row 1, CUDA-graph steady state: the loop with steady-state
    iterations replayed from the captured step graph (re-captured after every
    rebuild) equals the eager loop bit for bit (LC, VL, VCL; thermostat and
    gravity on)."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import simulate
    z = golden("traj_small.npz")
    L = z["domain"]
    for cid in ("VL-List_Iter-NoN3L-AoS", "LC-C08-N3L-SoA-CSF1", "VCL-ClusterIter-NoN3L-AoS"):
        out = []
        for graphs in (False, True):
            params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4,
                                        delta_t=1e-3, boundary=(P.PERIODIC,) * 3, gravity=-0.3,
                                        thermostat=P.ThermostatParams(0.9, 0.05, 5))
            parts = P.ParticleSet(z["pos0"], z["vel0"], layout=P.parse_configuration(cid).layout)
            rep = simulate(parts, params, P.parse_configuration(cid), steps=23, record=False,
                           graphs=graphs, raise_errors=True)
            assert rep.error is None
            out.append((parts.numpy("pos"), parts.numpy("vel"), parts.numpy("force")))
        for a, b in zip(*out):
            assert np.array_equal(a, b), cid


def test_fused_kick_drift_loop_is_bit_identical(pkg):
    """Simulation(fuse_kick_drift=True): each untimed step's kick deferred into
    the next step's drift (mdg_kick_drift, force / old_force swapped instead
    of copied) equals the two-pass loop bit for bit -- LC / VL / VCL, two
    types, gravity, a reflective axis, a thermostat (whose steps kick
    eagerly), and state read back between partial runs."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    z = golden("traj_small.npz")
    L = z["domain"]
    n = len(z["pos0"])
    tid = np.arange(n) % 2
    types = [P.ParticleTypeInfo(0, 1.0, 1.0, 1.0), P.ParticleTypeInfo(1, 1.2, 0.9, 1.5)]
    for cid in ("VL-List_Iter-NoN3L-SoA", "LC-C08-N3L-AoS-CSF1", "VCL-ClusterIter-NoN3L-AoS"):
        for boundary in ((P.PERIODIC,) * 3, (P.PERIODIC, P.REFLECTIVE, P.PERIODIC)):
            out = []
            for fuse in (False, True):
                params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4,
                                            delta_t=1e-3, boundary=boundary, gravity=-0.3,
                                            thermostat=P.ThermostatParams(0.9, 0.05, 7))
                cfg = P.parse_configuration(cid)
                parts = P.ParticleSet(z["pos0"], z["vel0"], type_ids=tid, types=types,
                                      layout=cfg.layout)
                sim = Simulation(parts, params, cfg, fuse_kick_drift=fuse)
                snaps = []
                for k in (5, 1, 13):
                    sim.run(k, record=False)
                    snaps.append(parts.numpy("vel"))
                sim.check()
                out.append([parts.numpy("pos"), parts.numpy("vel"), parts.numpy("force"),
                            parts.numpy("old_force")] + snaps)
            for a, b in zip(*out):
                assert np.array_equal(a, b), (cid, boundary)


def test_permutation_ops_match_numpy(pkg):
    """mdg_permutation (the cell reorder's index work in libmdg): composition,
    inverse and the int32 -> int64 widening, against numpy."""
    P, calc_mod = pkg
    from paper_2505_03438_b200.calculator import ForceCalculator
    z = golden("traj_small.npz")
    params = P.SimulationParams(domain_size=z["domain"], cutoff=2.5, skin=0.3, rebuild_interval=10,
                                delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
    calc = ForceCalculator(P.ParticleSet(z["pos0"]), params)
    rng = np.random.default_rng(3)
    for n in (1, 1000, 100_003):
        a = rng.permutation(n)
        b = rng.permutation(n)
        ta, tb = torch.tensor(a, device="cuda"), torch.tensor(b, device="cuda")
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        calc.permutation(0, ta, tb, out)
        assert np.array_equal(out.cpu().numpy(), a[b])
        calc.permutation(1, ta, None, out)
        inv = np.empty(n, dtype=np.int64)
        inv[a] = np.arange(n)
        assert np.array_equal(out.cpu().numpy(), inv)
        calc.permutation(2, torch.tensor(a.astype(np.int32), device="cuda"), None, out)
        assert np.array_equal(out.cpu().numpy(), a)
    calc.close()


def test_native_fixed_loop_matches_step_loop(pkg):
    """Simulation.run's native spans (mdg_run: a fixed configuration's untimed
    iterations in one C call, steady steps replayed from captured graphs)
    equal the Python step() loop bit for bit -- every deterministic container
    family, two types, gravity, a reflective axis, a thermostat (its
    iterations run eagerly between native spans), the cell reorder (spans stop
    short of its rebuilds), runs split at arbitrary points -- and a blow-up is
    reported at the same iteration."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import BlowUpError, Simulation
    z = golden("traj_small.npz")
    L = z["domain"]
    n = len(z["pos0"])
    tid = np.arange(n) % 2
    types = [P.ParticleTypeInfo(0, 1.0, 1.0, 1.0), P.ParticleTypeInfo(1, 1.2, 0.9, 1.5)]
    # the deterministic traversals (C18 / SLI / VCL-N3L add reactions with fp64 atomics)
    for cid, reorder in (("LC-C08-N3L-SoA-CSF1", 0), ("LC-C08-N3L-AoS-CSF0.5", 0),
                         ("LC-C01-NoN3L-SoA-CSF1", 0), ("VL-List_Iter-NoN3L-AoS", 0),
                         ("VL-List_Iter-NoN3L-SoA", 1), ("VCL-ClusterIter-NoN3L-SoA", 0),
                         ("VL-List_Iter-NoN3L-SoA-FP32", 0)):
        out = []
        for native in (False, True):
            params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4,
                                        delta_t=1e-3, boundary=(P.PERIODIC, P.REFLECTIVE, P.PERIODIC),
                                        gravity=-0.3, thermostat=P.ThermostatParams(0.9, 0.05, 7))
            cfg = P.parse_configuration(cid)
            parts = P.ParticleSet(z["pos0"], z["vel0"], type_ids=tid, types=types, layout=cfg.layout)
            sim = Simulation(parts, params, cfg, fuse_kick_drift=True, reorder=reorder)
            sim.native = native
            snaps = []
            for k in (3, 11, 1, 17):
                sim.run(k, record=False)
                snaps.append(parts.numpy("pos"))
            sim.check()
            out.append([parts.numpy("pos"), parts.numpy("vel"), parts.numpy("force"),
                        parts.numpy("old_force"), np.array([sim.iteration, sim.since])] + snaps)
        for a, b in zip(*out):
            assert np.array_equal(a, b), cid
    # a particle thrown out of the box: same failing iteration either way
    pos = np.array(z["pos0"], copy=True)
    pos[1] = pos[0] + np.array([0.3, 0.0, 0.0])
    its = []
    for native in (False, True):
        params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=3,
                                    delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
        parts = P.ParticleSet(np.mod(pos, L), z["vel0"])
        sim = Simulation(parts, params, P.parse_configuration("LC-C08-N3L-AoS-CSF1"), fuse_kick_drift=True)
        sim.native = native
        with pytest.raises(BlowUpError):
            sim.run(12, record=False)
        its.append(sim.iteration)
    assert its[0] == its[1], its


def test_pipelined_host_run_blow_up_matches_step_path(pkg):
    """A particle thrown out of the box (two particles 0.3 sigma apart: the
    step-1 drift moves one by >> L) raises BlowUpError from HostSimulation.run
    at the same iteration as the one-step-per-call path."""
    P, calc = pkg
    from paper_2505_03438_b200.hostloop import HostParticleSet, HostSimulation
    from paper_2505_03438_b200.simulation import BlowUpError
    z = golden("traj_small.npz")
    L = z["domain"]
    pos = np.array(z["pos0"], copy=True)
    pos[1] = pos[0] + np.array([0.3, 0.0, 0.0])
    its = []
    for chunks in (1, 4):
        params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                                    delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
        p = HostParticleSet(np.mod(pos, L), z["vel0"])
        sim = HostSimulation(p, params, P.parse_configuration("VL-List_Iter-NoN3L-AoS"), chunks=chunks)
        with pytest.raises(BlowUpError):
            sim.run(5)
        its.append(sim.iteration)
    assert its[0] == its[1] == 1, its


def test_device_decomposition_single_rank_is_the_plain_loop(pkg):
    """DeviceDecomposedSimulation on one rank (no decomposed axis, no ghosts,
    no process group needed) is the plain device loop, bit for bit."""
    P, calc = pkg
    from paper_2505_03438_b200.decomp import DeviceDecomposedSimulation, GridDecomposition
    from paper_2505_03438_b200.simulation import Simulation
    z = golden("traj_small.npz")
    L = z["domain"]
    params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4,
                                delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    a = P.ParticleSet(z["pos0"], z["vel0"], layout="SoA")
    Simulation(a, params, cfg).run(17, record=False)
    dsim = DeviceDecomposedSimulation(GridDecomposition(params, 0, 1), P.ParticleSet(z["pos0"], z["vel0"]),
                                      params, cfg)
    dsim.run(17)
    dsim.check()
    assert np.array_equal(dsim.owned("pos").cpu().numpy(), a.numpy("pos"))
    assert np.array_equal(dsim.owned("vel").cpu().numpy(), a.numpy("vel"))
    assert np.array_equal(dsim.ids.cpu().numpy(), np.arange(len(z["pos0"])))


def test_config5_tiled_lists_past_32_bit_entries(pkg):
    """BASELINE config 5 (67,108,864 FCC particles) on one GPU: the tiled
    Verlet lists hold ~5.4 G entries (64-bit offsets; per-tile bases count
    32-bit slots).  Size-independent parity against an independent path on
    the same snapshot: the VL count (2 per pair) is exactly twice LC-SLI-N3L's
    (1 per pair), and the forces agree within the fp64 tolerance."""
    P, calc = pkg
    import torch
    from paper_2505_03438_b200 import systems
    pos, vel, params = systems.config5_inputs()
    parts = P.ParticleSet(pos, layout="SoA")
    del pos, vel
    fc = calc.ForceCalculator(parts, params)
    vl = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    fc.rebuild(parts, vl)
    fc.refresh(parts, vl)
    n_vl = fc.compute(parts, vl)
    f_vl = parts.view("force").clone()
    lc = P.parse_configuration("LC-SLI-N3L-SoA-CSF1")
    fc.rebuild(parts, lc)
    fc.refresh(parts, lc)
    n_lc = fc.compute(parts, lc)
    fc.close()
    assert n_vl == 2 * n_lc and n_lc > 1_700_000_000
    num = torch.linalg.vector_norm(parts.view("force") - f_vl)
    den = torch.linalg.vector_norm(f_vl)
    assert float(num / den) <= FP64_TOL


def test_stale_verlet_lists_between_rebuilds(pkg):
    """The reference's stale-list semantics (tests/test_containers.py:145-161,
    containers.py:435-436): a pair that enters the cutoff without a rebuild is
    missed by VL (its list is from the last rebuild) and seen by LC (refresh
    re-gathers positions); both as the oracle's ForceCalculator does."""
    P, calc = pkg
    params = P.SimulationParams(domain_size=(12.0, 12.0, 12.0), cutoff=2.5, skin=0.3,
                                boundary=(P.REFLECTIVE,) * 3)
    pp = port.Params(domain_size=(12.0, 12.0, 12.0), cutoff=2.5, skin=0.3,
                     boundary=(port.REFLECTIVE,) * 3)
    start = np.array([[4.0, 6.0, 6.0], [7.0, 6.0, 6.0]])       # 3.0 apart: beyond ell = 2.8
    moved = np.array([[4.0, 6.0, 6.0], [6.0, 6.0, 6.0]])       # 2.0 apart: inside rc
    for cid in ("VL-List_Iter-NoN3L-AoS", "LC-C08-N3L-AoS-CSF1", "LC-C01-NoN3L-SoA-CSF1"):
        cfg = P.parse_configuration(cid)
        parts = P.ParticleSet(start, layout=cfg.layout)
        fc = calc.ForceCalculator(parts, params)
        fc.rebuild(parts, cfg)
        parts.view("pos").copy_(torch.as_tensor(moved))
        fc.refresh(parts, cfg)
        n = fc.compute(parts, cfg)
        fc.close()
        ref = port.Particles(start, layout=cfg.layout)
        rfc = port.ForceCalculator(ref, pp)
        rfc.rebuild(ref, port.parse(cid))
        ref.view("pos")[:] = moved
        rfc.refresh(ref, port.parse(cid))
        rn = rfc.compute(ref, port.parse(cid))
        assert n == rn, (cid, n, rn)
        assert np.allclose(parts.numpy("force"), np.asarray(ref.forces), atol=1e-12), cid
        if cid.startswith("VL"):
            assert n == 0 and np.all(parts.numpy("force") == 0.0)
        else:
            assert n > 0


def _fuzz_system(seed):
    """Seeded random system: N, a non-cubic box, mixed periodic / reflective
    axes, 1-3 types, random density; positions by sequential rejection
    (>= 0.85 sigma apart, so the fp32 variant stays finite)."""
    rng = np.random.default_rng(1000 + seed)
    n_target = int(rng.choice([2, 7, 64, 500, 1500, 3000]))
    L = rng.uniform(6.0, 16.0, 3)
    per = rng.random(3) < 0.6
    nt = int(rng.integers(1, 4))
    pos = []
    tries = 0
    while len(pos) < n_target and tries < 40 * n_target:
        tries += 1
        x = rng.uniform(0.0, 1.0, 3) * L
        if pos:
            d = np.asarray(pos) - x
            d[:, per] -= L[per] * np.rint(d[:, per] / L[per])
            if np.min(np.einsum("ij,ij->i", d, d)) < 0.85 ** 2:
                continue
        pos.append(x)
    return np.asarray(pos), L, per, nt


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_every_configuration_vs_oracle(pkg, seed):
    """Random systems (size, box shape, boundaries, types, density) through
    every configuration -- the 30 reference ids, VCL and the fp32 variant --
    against the oracle: exact counts, fp64 forces within 1e-10, fp32 within
    1e-4."""
    P, calc = pkg
    pos, L, per, nt = _fuzz_system(seed)
    n = len(pos)
    tid = (np.arange(n) % nt).astype(np.int64)
    types = [P.ParticleTypeInfo(t, 1.0 + 0.5 * t, 1.0 - 0.2 * t, 1.0 + t) for t in range(nt)]
    bnd = tuple(P.PERIODIC if f else P.REFLECTIVE for f in per)
    params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, boundary=bnd)
    pp = port.Params(domain_size=L, cutoff=2.5, skin=0.3,
                     boundary=tuple(port.PERIODIC if f else port.REFLECTIVE for f in per))
    ref = {}
    for cfg in P.enumerate_configurations():
        rp = port.Particles(pos, type_id=tid, sigma=[t.sigma for t in types],
                            epsilon=[t.epsilon for t in types], mass=[t.mass for t in types])
        _, c = port.compute_forces(rp, port.parse(cfg.id), pp, workers=2)
        ref[cfg.id] = (c, np.asarray(rp.forces).copy())
    f_vl = ref["VL-List_Iter-NoN3L-AoS"][1]
    c_vl = ref["VL-List_Iter-NoN3L-AoS"][0]
    for cfg in P.extended_configurations():
        parts = P.ParticleSet(pos, type_ids=tid, types=types, layout=cfg.layout)
        _, count = calc.compute_forces(parts, cfg, params)
        got = parts.numpy("force")
        if cfg.id in ref:
            want_c, want_f = ref[cfg.id]
            assert count == want_c, (seed, cfg.id, count, want_c)
            assert port.force_rel_error(got, want_f) <= FP64_TOL, (seed, cfg.id)
        elif cfg.id.startswith("VCL"):
            assert count == c_vl // (2 if cfg.newton3 else 1), (seed, cfg.id)
            assert port.force_rel_error(got, f_vl) <= FP64_TOL, (seed, cfg.id)
        else:   # fp32 variant
            assert abs(count - c_vl) <= max(2, 1e-6 * c_vl), (seed, cfg.id, count, c_vl)
            assert port.force_rel_error(got, f_vl) <= 1e-4, (seed, cfg.id)


# -- dynamic pruning of the tiled Verlet walk ---------------------

@pytest.mark.parametrize("traj", ["traj_small", "traj_faces", "traj_config1"])
def test_pruned_walk_trajectories_match_reference(pkg, traj):
    """Inner lists re-pruned almost every step (delta 0.01: a 0.005 move
    re-prunes) and never (pruning off) both reproduce the reference's 100-step
    VL trajectories; with delta 0.01 several prune walks happen per window."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    z = golden(f"{traj}.npz")
    L = z["domain"]
    ids = [str(s) for s in z["config_ids"]]
    # config 1's reference run is LC-C08; VL agrees with it to ~5e-14 there
    # (sites at (i + 0.5) * 1.1 keep particles off the faces)
    cases = [(k, c) for k, c in enumerate(ids) if c.startswith("VL")] or [(0, "VL-List_Iter-NoN3L-SoA")]
    for k, cid in cases:
        for delta in (0.01, 0.0):
            params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                                        delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
            cfg = P.parse_configuration(cid)
            parts = P.ParticleSet(z["pos0"], z["vel0"], layout=cfg.layout)
            sim = Simulation(parts, params, cfg)
            sim.calc.set_prune(delta)
            sim.run(33, record=False)              # the last window: iterations 22..32
            prunes = sim.calc.prune_count()
            sim.run(int(z["steps"]) - 33, record=False)
            sim.check()
            if delta == 0.0:
                assert prunes == -1
            else:
                assert prunes >= 2, prunes
            dpos = parts.numpy("pos") - z[f"pos_{k}"]
            dpos -= L * np.rint(dpos / L)
            assert np.linalg.norm(dpos) / np.linalg.norm(z[f"pos_{k}"]) <= FP64_TOL, (cid, delta)
            assert port.force_rel_error(parts.numpy("vel"), z[f"vel_{k}"]) <= FP64_TOL, (cid, delta)


def test_pruned_walk_full_size_is_the_full_walk(pkg, config2_snapshot):
    """BASELINE config 2 (1,048,576 particles), 33 steps (3 rebuild windows):
    per step the pruned walks (default delta = skin / 3, and a tight 0.02)
    count exactly the pairs of the unpruned walk, and the trajectories agree
    within the fp64 bar (the only difference is the grouping of the batched
    reciprocal)."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    pos, vel, params = config2_snapshot
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    runs = {}
    for delta in (0.0, None, 0.02):
        parts = P.ParticleSet(pos, vel, layout="SoA")
        sim = Simulation(parts, params, cfg)
        sim.calc.set_prune(delta)
        counts, prunes = [], []
        for s in range(33):
            sim.step()
            counts.append(sim.calc.last_eval_count)
            if s % 11 == 10:
                prunes.append(sim.calc.prune_count())
        sim.flush()
        sim.check()
        runs[delta] = (parts.numpy("pos"), parts.numpy("vel"), counts, prunes)
    p0, v0, c0, n0 = runs[0.0]
    assert n0 == [-1, -1, -1]
    for delta in (None, 0.02):
        p1, v1, c1, n1 = runs[delta]
        assert c1 == c0, delta
        assert min(n1) >= (1 if delta is None else 3), (delta, n1)
        L = params.domain_size
        d = p1 - p0
        d -= L * np.rint(d / L)
        assert np.linalg.norm(d) / np.linalg.norm(p0) <= FP64_TOL, delta
        assert port.force_rel_error(v1, v0) <= FP64_TOL, delta


def test_cell_reorder_is_invisible(pkg, config2_snapshot):
    """Simulation(reorder=k) keeps the particle arrays in cell order inside the
    loop and restores the caller's order on flush: 33 config-2 steps with a
    reorder at every rebuild give the unreordered trajectory bit for bit (VL
    SoA with the fused kick, VL AoS), across run() boundaries and an outside
    rebuild (potential_energy) in between, which drops the order; linked
    cells are left in the caller's order."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    pos, vel, params = config2_snapshot
    for cid, fuse in (("VL-List_Iter-NoN3L-SoA", True), ("VL-List_Iter-NoN3L-AoS", False),
                      ("LC-C08-N3L-AoS-CSF1", False)):
        cfg = P.parse_configuration(cid)
        out = []
        for reorder in (0, 1):
            parts = P.ParticleSet(pos, vel, layout=cfg.layout)
            sim = Simulation(parts, params, cfg, fuse_kick_drift=fuse, reorder=reorder)
            sim.run(12)
            if reorder and cid.startswith("VL"):
                assert sim._perm is not None and not sim._permuted
                assert not torch.equal(sim._perm, torch.arange(parts.n, device=sim._perm.device))
            elif reorder:   # linked cells keep the reference's index order
                assert sim._perm is None
            sim.run(11)
            if cid.startswith("VL"):
                sim.calc.potential_energy(parts, rebuild=True)   # a rebuild on the caller's order
            sim.run(10)
            sim.check()
            out.append((parts.numpy("pos"), parts.numpy("vel"), parts.numpy("force")))
        for a, b in zip(*out):
            assert np.array_equal(a, b), cid


def test_warm_reorder_keeps_the_trajectory(pkg, config2_snapshot):
    """bench.py's warm_reorder(): a cell reorder taken outside the timed loop
    (arrays permuted, flush path run once, a rebuild forced on the next step)
    leaves the trajectory within the fp64 bar of the plain loop (the extra
    rebuild changes list order, so summation order, only)."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    pos, vel, params = config2_snapshot
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    out = []
    for reorder in (0, 8):
        parts = P.ParticleSet(pos, vel, layout=cfg.layout)
        sim = Simulation(parts, params, cfg, fuse_kick_drift=True, reorder=reorder)
        for _ in range(11):
            sim.step()
        sim.check()
        sim.warm_reorder()
        for _ in range(22):
            sim.step()
        sim.check()
        if reorder:
            assert sim._perm is not None and not sim._permuted
        out.append((parts.numpy("pos"), parts.numpy("vel")))
    L = params.domain_size
    d = out[1][0] - out[0][0]
    d -= L * np.rint(d / L)
    assert np.linalg.norm(d) / np.linalg.norm(out[0][0]) <= FP64_TOL
    assert port.force_rel_error(out[1][1], out[0][1]) <= FP64_TOL


@pytest.mark.parametrize("cid", ["VL-List_Iter-NoN3L-AoS", "LC-C08-N3L-SoA-CSF1"])
def test_blow_up_reports_the_reference_iteration(pkg, cid):
    """Two particles driven into each other blow up (integrator.py:108-116)
    in the reference at iteration 34; the device loop reads its status bit
    only at rebuilds, yet reports that iteration and keeps exactly the
    records of the 34 completed iterations, like the reference's report."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import simulate
    pos = np.array([[3.0, 5.0, 5.0], [7.0, 5.0, 5.0], [1.0, 1.0, 1.0]])
    vel = np.array([[100.0, 0, 0], [-100.0, 0, 0], [0, 0, 0]])
    op = port.Params(domain_size=(10.0, 10.0, 10.0), cutoff=2.5, skin=0.3, rebuild_interval=10,
                     delta_t=2e-3, boundary=(port.PERIODIC,) * 3)
    done = []
    with pytest.raises(port.BlowUp):
        port.simulate_fixed(port.Particles(pos, vel), op, port.parse(cid), steps=100,
                            on_step=lambda it: done.append(it))
    params = P.SimulationParams(domain_size=(10.0, 10.0, 10.0), cutoff=2.5, skin=0.3, rebuild_interval=10,
                                delta_t=2e-3, boundary=(P.PERIODIC,) * 3)
    rep = simulate(P.ParticleSet(pos, vel), params, P.parse_configuration(cid), steps=100)
    assert rep.error and rep.error.startswith("BlowUpError"), rep.error
    assert f"at iteration {len(done)}" in rep.error, (rep.error, len(done))
    assert len(rep.records) == len(done) == 34
