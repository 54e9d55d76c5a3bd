"""Pin the oracle (CPU restatement) against the reference's own outputs.

The fixtures in tests/golden/ were produced by oracle/make_golden.py from the
real reference (numba kernels, /root/reference/pkg/src/mdtune).  The oracle
must reproduce them: geometry/stencils/cell arrays/Verlet lists bit-exactly,
forces and counts bit-exactly (same arithmetic order, contraction off), and
the simulate() trajectories bit-exactly.
"""

import numpy as np
import pytest

from conftest import golden, system_names
from oracle import port


def _params(d, rebuild=5):
    per = tuple(port.PERIODIC if f else port.REFLECTIVE for f in d["periodic"])
    return port.Params(domain_size=d["domain"], cutoff=float(d["cutoff"]),
                       skin=float(d["skin"]), rebuild_interval=rebuild, boundary=per)


def _particles(d):
    nt = int(d["n_types"])
    return port.Particles(d["pos"], type_id=d["tid"],
                          sigma=[1.0 - 0.2 * t for t in range(nt)],
                          epsilon=[1.0 + 0.5 * t for t in range(nt)],
                          mass=[1.0 + t for t in range(nt)])


def test_geometry_and_stencils_match_reference():
    z = golden("geometry.npz")
    for k in range(int(z["n_cases"])):
        g = port.make_geometry(z[f"g{k}_in_domain"], z[f"g{k}_in_scalars"][0],
                               z[f"g{k}_in_scalars"][1], z[f"g{k}_in_periodic"].astype(bool))
        assert g.dims_owned == tuple(z[f"g{k}_dims_owned"])
        assert g.cell_length == tuple(z[f"g{k}_cell_length"])
        assert g.overlap == tuple(z[f"g{k}_overlap"])
        assert g.halo == tuple(z[f"g{k}_halo"])
        assert g.dims == tuple(z[f"g{k}_dims"])
        assert np.array_equal(port.pruned_stencil(g), z[f"g{k}_pruned"])
        for major in range(3):
            assert np.array_equal(port.forward_stencil(g, major), z[f"g{k}_forward{major}"])


@pytest.mark.parametrize("name", system_names())
def test_cell_binning_bit_exact(name):
    d = golden(f"sys_{name}.npz")
    params = _params(d)
    p = _particles(d)
    for csf, tag in ((1.0, "csf1"), (0.5, "csf05")):
        g = port.make_geometry(params.domain_size, params.interaction_length, csf,
                               params.periodic_flags())
        grid = port.Grid(g)
        grid.rebuild(p)
        assert np.array_equal(grid.src, d[f"{tag}_src"])
        assert np.array_equal(grid.shift, d[f"{tag}_shift"])
        assert np.array_equal(grid.start, d[f"{tag}_start"])
        assert np.array_equal(grid.end, d[f"{tag}_end"])


@pytest.mark.parametrize("name", system_names())
def test_verlet_lists_bit_exact(name):
    d = golden(f"sys_{name}.npz")
    params = _params(d)
    g = port.make_geometry(params.domain_size, params.interaction_length, 1.0,
                           params.periodic_flags())
    vl = port.VerletLists(g)
    vl.rebuild(_particles(d))
    assert np.array_equal(vl.noff, d["vl_noff"])
    assert np.array_equal(vl.nbr, d["vl_nbr"])


@pytest.mark.parametrize("name", system_names())
def test_all_30_configurations_bit_exact(name):
    d = golden(f"sys_{name}.npz")
    params = _params(d)
    ids = [str(s) for s in d["config_ids"]]
    assert ids == [c.id for c in port.all_configs()]
    for k, cid in enumerate(ids):
        p = _particles(d)
        _, count = port.compute_forces(p, port.parse(cid), params, workers=1)
        assert count == d["counts"][k], cid
        assert np.array_equal(np.asarray(p.forces), d["forces"][k]), cid


@pytest.mark.parametrize("name", ["small_periodic", "crit1_0"])
def test_worker_count_independent(name):
    d = golden(f"sys_{name}.npz")
    params = _params(d)
    for cfg in port.all_configs():
        a, b = _particles(d), _particles(d)
        port.compute_forces(a, cfg, params, workers=1)
        port.compute_forces(b, cfg, params, workers=4)
        assert port.force_rel_error(b.forces, a.forces) <= 1e-12, cfg.id


@pytest.mark.parametrize("name", ["small_periodic", "mixed", "blob", "tight"])
def test_oracle_vs_brute_force(name):
    d = golden(f"sys_{name}.npz")
    params = _params(d)
    p = _particles(d)
    ref, directed = port.brute_forces(p.positions, p.type_id, p.epsilon, p.sigma,
                                      params.cutoff, params.domain_size, params.periodic_flags())
    for k, cfg in enumerate(port.all_configs()):
        assert port.force_rel_error(d["forces"][k], ref) <= 1e-9, cfg.id
        assert d["counts"][k] * (2 if cfg.newton3 else 1) == directed, cfg.id


@pytest.mark.parametrize("traj", ["traj_small", "traj_faces", "traj_config1"])
def test_simulate_trajectory_bit_exact(traj):
    z = golden(f"{traj}.npz")
    L = float(z["domain"][0])
    for k, cid in enumerate(str(s) for s in z["config_ids"]):
        params = port.Params(domain_size=(L, L, L), cutoff=2.5, skin=0.3, rebuild_interval=10,
                             delta_t=1e-3, boundary=(port.PERIODIC,) * 3)
        p = port.Particles(z["pos0"], z["vel0"])
        port.simulate_fixed(p, params, port.parse(cid), steps=int(z["steps"]))
        assert np.array_equal(np.asarray(p.positions), z[f"pos_{k}"]), cid
        assert np.array_equal(np.asarray(p.velocities), z[f"vel_{k}"]), cid


def _reflect_gravity_setup(z, cid_layout_obj=None):
    L = float(z["domain"][0])
    bnd = tuple(port.PERIODIC if f else port.REFLECTIVE for f in z["periodic"])
    params = port.Params(domain_size=(L, L, L), cutoff=2.5, skin=0.3, rebuild_interval=6,
                         delta_t=float(z["dt"]), boundary=bnd, gravity=float(z["gravity"]))
    # the two types of make_golden._types(2): sigma 1, 0.8; epsilon 1, 1.5; mass 1, 2
    p = port.Particles(z["pos0"], z["vel0"], type_id=z["tid"], sigma=(1.0, 0.8),
                       epsilon=(1.0, 1.5), mass=(1.0, 2.0))
    return params, p


def test_reflect_gravity_trajectory_bit_exact():
    """Reflective walls (y, z) + periodic x, gravity, two types with masses 1
    and 2 (integrator.py:47-51, :98-128): the oracle's integrator replays the
    reference's trajectories bit for bit, and the fixture did reflect."""
    z = golden("traj_reflect_gravity.npz")
    for k, cid in enumerate(str(s) for s in z["config_ids"]):
        assert int(z[f"reflections_{k}"]) > 0
        params, p = _reflect_gravity_setup(z)
        port.simulate_fixed(p, params, port.parse(cid), steps=int(z["steps"]))
        assert np.array_equal(np.asarray(p.positions), z[f"pos_{k}"]), cid
        assert np.array_equal(np.asarray(p.velocities), z[f"vel_{k}"]), cid
        assert np.array_equal(np.asarray(p.forces), z[f"force_{k}"]), cid


# -- thermostat, live statistics, controller-driven loop -------

def test_live_stats_oracle_matches_reference():
    z = golden("thermo_stats.npz")
    for name in (str(s) for s in z["ls_names"]):
        a = z[f"ls_{name}_in"]
        per = port.PERIODIC if a[5] else port.REFLECTIVE
        params = port.Params(domain_size=a[:3], cutoff=float(a[3]), skin=float(a[4]),
                             boundary=(per,) * 3, thread_count=int(a[6]))
        p = port.Particles(z[f"ls_{name}_pos"])
        assert np.array_equal(port.compute_live_stats(p, params), z[f"ls_{name}_out"]), name


def test_temperature_and_thermostat_oracle_match_reference():
    z = golden("thermo_stats.npz")
    for name in (str(s) for s in z["th_names"]):
        nt, soa, target, mdt = z[f"th_{name}_in"]
        nt = int(nt)
        vel0 = z[f"th_{name}_vel0"]
        p = port.Particles(np.zeros_like(vel0), vel0, z[f"th_{name}_tid"],
                           sigma=[1.0 - 0.2 * t for t in range(nt)],
                           epsilon=[1.0 + 0.5 * t for t in range(nt)],
                           mass=[1.0 + t for t in range(nt)], layout="SoA" if soa else "AoS")
        assert port.current_temperature(p) == float(z[f"th_{name}_t"]), name
        port.apply_thermostat(p, target, mdt)
        assert np.array_equal(np.asarray(p.velocities), z[f"th_{name}_vel"]), name


def test_thermostat_rejects_zero_velocities_with_positive_target():
    p = port.Particles(np.zeros((4, 3)))
    with pytest.raises(ValueError):
        port.apply_thermostat(p, 1.0, 0.1)
    port.apply_thermostat(p, 0.0, 0.1)          # target 0: unchanged, no error
    with pytest.raises(ValueError):
        port.current_temperature(port.Particles(np.zeros((0, 3))))


def test_controlled_loop_oracle_matches_reference():
    """The reference's TuningController + FullSearchStrategy run (thermostat
    on, layout switches, forced trial rebuilds) replayed through the oracle's
    restatement of simulate(): bit-exact final state."""
    from conftest import ScriptedController, Thermostat
    z = golden("traj_tuned.npz")
    L = float(z["domain"][0])
    interval, spc, R, tint = (int(x) for x in z["tuning"])
    params = port.Params(domain_size=(L, L, L), cutoff=2.5, skin=0.3, rebuild_interval=R,
                         delta_t=1e-3, boundary=(port.PERIODIC,) * 3,
                         thermostat=Thermostat(float(z["thermo"][0]), float(z["thermo"][1]), tint))
    p = port.Particles(z["pos0"], z["vel0"])
    ctl = ScriptedController(z, port.parse)
    seq = port.simulate_controlled(p, params, ctl, steps=int(z["steps"]))
    assert [c for c, _ in seq] == [str(s) for s in z["seq_cfg"]]
    assert ctl.trial_iterations == int(z["trial_iterations"])
    assert p.layout == str(z["layout"])
    assert np.array_equal(np.asarray(p.positions), z["pos"])
    assert np.array_equal(np.asarray(p.velocities), z["vel"])
    assert np.array_equal(np.asarray(p.forces), z["force"])
    assert port.current_temperature(p) == float(z["final_temperature"])


@pytest.mark.parametrize("name", system_names())
def test_sampled_brute_force_matches_reference(name):
    """port.sampled_forces (the cell-list brute force used to check the
    BASELINE-size snapshots on sampled rows) reproduces the reference's forces
    and its directed within-cutoff count on every golden system."""
    d = golden(f"sys_{name}.npz")
    params = _params(d)
    p = _particles(d)
    rows = np.arange(p.n)
    f, cnt = port.sampled_forces(p.positions, rows, params.cutoff, params.domain_size,
                                 params.periodic_flags(), tid=p.type_id, sigma=p.sigma,
                                 epsilon=p.epsilon, workers=3)
    k = [c.id for c in port.all_configs()].index("VL-List_Iter-NoN3L-AoS")
    assert port.force_rel_error(f, d["forces"][k]) <= 1e-12
    assert int(cnt.sum()) == int(d["counts"][k])
