"""GPU parity at BASELINE size against the oracle (not against the GPU's own
other paths): the bench workload (config 2, 1,048,576 particles) and
configs 3, 4 and 5, on identical seeded inputs.

* cell assignment (GridState src/shift/start/end, CSF 1 and 0.5) and the
  Verlet pair lists (VerletListState noff/nbr) bit-exact against
  oracle/port.py, the restatement pinned bit-exactly to the reference
  (tests/test_oracle_golden.py);
* forces within 1e-10 (relative Frobenius, the north_star fp64 bar) and exact
  eval counts for the tiled Verlet walk and every container family against
  the oracle's LC-C08 ForceCalculator (containers.py:378-488);
* K-step trajectories of the bench's own loop (tiled walk with dynamic
  pruning, particle arrays kept in cell order, kick fused into the next drift)
  against the oracle's simulate (simulation.py:126-197);
* config 5 (67,108,864 particles) against the reference's brute-force oracle
  (tests/conftest.py:22-44) run over every row through a cell list;
* the device integrator's reflective walls, gravity and two-type masses
  against trajectories the real reference wrote (tests/golden/
  traj_reflect_gravity.npz, oracle/make_golden.py).
"""

import os

import numpy as np
import pytest

from conftest import golden
from oracle import port

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FP64_TOL = 1e-10
FP32_TOL = 1e-4
# fp32 pair test of the -FP32 variant (cell-relative float coordinates,
# vl.cu:vl_force32_kernel): |r2_f32 - r2| stays below ~1e-6 rc^2; pairs closer
# than this band to the cutoff may flip, no other pair can.
FP32_BAND = 4e-6
WORKERS = len(os.sched_getaffinity(0))


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA")
    import paper_2505_03438_b200 as P
    from paper_2505_03438_b200 import calculator
    return P, calculator


def _oparams(params, **kw):
    bnd = tuple(port.PERIODIC if b == "periodic" else port.REFLECTIVE for b in params.boundary)
    args = dict(domain_size=tuple(params.domain_size), cutoff=params.cutoff, skin=params.skin,
                rebuild_interval=params.rebuild_interval, delta_t=params.delta_t, boundary=bnd,
                thread_count=WORKERS)
    args.update(kw)
    return port.Params(**args)


def _oracle_forces(pos, params, cid="LC-C08-N3L-AoS-CSF1"):
    """The oracle's ForceCalculator on the snapshot: (forces (N,3), count)."""
    op = _oparams(params)
    p = port.Particles(pos)
    with port.Pool(WORKERS) as pool:
        fc = port.ForceCalculator(p, op)
        cfg = port.parse(cid)
        p.convert_layout(cfg.layout)
        fc.rebuild(p, cfg)
        fc.refresh(p, cfg)
        n = fc.compute(p, cfg, pool)
    return np.ascontiguousarray(p.forces), n


def _band_pairs(pos, noff, nbr, params, band=FP32_BAND):
    """Unique Verlet pairs (minimum image) whose r^2 lies within band*rc^2 of
    rc^2: the only pairs the fp32 pair test may classify differently."""
    i = np.repeat(np.arange(len(noff) - 1), np.diff(noff))
    j = np.asarray(nbr, dtype=np.int64)
    keep = i < j
    i, j = i[keep], j[keep]
    L = np.asarray(params.domain_size, dtype=np.float64)
    per = np.array([b == "periodic" for b in params.boundary])
    d = pos[i] - pos[j]
    d[:, per] -= L[per] * np.rint(d[:, per] / L[per])
    r2 = np.einsum("ij,ij->i", d, d)
    rc2 = params.cutoff ** 2
    return int(np.count_nonzero(np.abs(r2 - rc2) <= band * rc2))


def _gpu_forces(P, calc, pos, params, cid):
    cfg = P.parse_configuration(cid)
    parts = P.ParticleSet(pos, layout=cfg.layout)
    _, count = calc.compute_forces(parts, cfg, params)
    return parts.numpy("force"), count, cfg


def _check_families(P, calc, pos, params, ids, ref_f, ref_n3l, band=None):
    for cid in ids:
        f, count, cfg = _gpu_forces(P, calc, pos, params, cid)
        unique = count if cfg.newton3 else count // 2
        if cfg.precision == "fp32":
            assert abs(count - 2 * ref_n3l) <= 2 * band, (cid, count, 2 * ref_n3l, band)
            assert port.force_rel_error(f, ref_f) <= FP32_TOL, cid
            continue
        assert unique == ref_n3l and (cfg.newton3 or count % 2 == 0), (cid, count, ref_n3l)
        err = port.force_rel_error(f, ref_f)
        assert err <= FP64_TOL, (cid, err)


# -- config 2 (the bench workload) -------------------------------------------

@pytest.fixture(scope="module")
def config2_oracle(config2_snapshot):
    pos, vel, params = config2_snapshot
    f, n = _oracle_forces(pos, params)
    vl = port.VerletLists(port.make_geometry(np.asarray(params.domain_size), params.cutoff + params.skin,
                                             1.0, np.ones(3, bool)))
    vl.rebuild(port.Particles(pos))
    return f, n, vl.noff, vl.nbr


def test_config2_cell_assignment_bit_exact(pkg, config2_snapshot):
    P, calc = pkg
    pos, vel, params = config2_snapshot
    per = np.ones(3, dtype=bool)
    for csf in (1.0, 0.5):
        og = port.Grid(port.make_geometry(np.asarray(params.domain_size), params.cutoff + params.skin,
                                          csf, per))
        og.rebuild(port.Particles(pos))
        for layout in ("AoS", "SoA"):
            parts = P.ParticleSet(pos, layout=layout)
            fc = calc.ForceCalculator(parts, params)
            fc.rebuild(parts, P.Configuration("LC", "C08", True, layout, csf))
            g = fc.grid_state(csf)
            fc.close()
            assert np.array_equal(g["src"], og.src), (csf, layout)
            assert np.array_equal(g["shift"], og.shift), (csf, layout)
            assert np.array_equal(g["start"], og.start), (csf, layout)
            assert np.array_equal(g["end"], og.end), (csf, layout)


def test_config2_verlet_pairs_bit_exact(pkg, config2_snapshot, config2_oracle):
    """VerletListState.rebuild (containers.py:343-375) on 1,048,576 particles:
    the tiled build's lists, exported in the reference's order, equal the
    oracle's noff / nbr (72 M entries) element for element."""
    P, calc = pkg
    pos, vel, params = config2_snapshot
    _, _, noff, nbr = config2_oracle
    for layout in ("SoA", "AoS"):
        parts = P.ParticleSet(pos, layout=layout)
        fc = calc.ForceCalculator(parts, params)
        fc.rebuild(parts, P.parse_configuration(f"VL-List_Iter-NoN3L-{layout}"))
        gnoff, gnbr = fc.verlet_lists()
        fc.close()
        assert np.array_equal(gnoff, noff), layout
        assert np.array_equal(gnbr, nbr), layout


def test_config2_forces_every_family_vs_oracle(pkg, config2_snapshot, config2_oracle):
    """Forces (<= 1e-10) and exact eval counts at 1,048,576 particles for the
    tiled walk, each LC traversal family at both CSFs, VCL, and the fp32
    variant (<= 1e-4, counts within the fp32 band) against the oracle."""
    P, calc = pkg
    pos, vel, params = config2_snapshot
    ref_f, ref_n, noff, nbr = config2_oracle
    band = _band_pairs(pos, noff, nbr, params)
    ids = ["VL-List_Iter-NoN3L-SoA", "VL-List_Iter-NoN3L-AoS", "LC-C08-N3L-AoS-CSF1",
           "LC-C08-NoN3L-SoA-CSF0.5", "LC-C18-N3L-SoA-CSF1", "LC-C18-NoN3L-AoS-CSF0.5",
           "LC-SLI-N3L-SoA-CSF1", "LC-SLI-NoN3L-AoS-CSF0.5", "LC-C01-NoN3L-SoA-CSF1",
           "LC-C01-NoN3L-AoS-CSF0.5", "VCL-ClusterIter-N3L-AoS", "VCL-ClusterIter-NoN3L-SoA",
           "VL-List_Iter-NoN3L-SoA-FP32", "VL-List_Iter-NoN3L-AoS-FP32"]
    _check_families(P, calc, pos, params, ids, ref_f, ref_n, band)


def test_config2_bench_loop_trajectory_vs_oracle(pkg, config2_snapshot):
    """22 steps (two rebuild windows at R = 10) of the bench's own loop --
    tiled walk with dynamic pruning, particle arrays permuted to cell order at
    every rebuild, kick fused into the next drift -- against the oracle's
    simulate with the same configuration: positions (modulo the box) and
    velocities within 1e-10."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    pos, vel, params = config2_snapshot
    steps = 22
    cid = "VL-List_Iter-NoN3L-SoA"
    parts = P.ParticleSet(pos, vel, layout="SoA")
    sim = Simulation(parts, params, P.parse_configuration(cid), fuse_kick_drift=True, reorder=1)
    sim.run(steps, record=False)
    sim.check()
    assert sim.calc.prune_count() >= 2           # the inner lists were rewritten in the run
    ref = port.Particles(pos, vel)
    with port.Pool(WORKERS) as pool:
        port.simulate_fixed(ref, _oparams(params), port.parse(cid), steps=steps, pool=pool)
    L = np.asarray(params.domain_size)
    dpos = parts.numpy("pos") - np.asarray(ref.positions)
    dpos -= L * np.rint(dpos / L)
    assert np.linalg.norm(dpos) / np.linalg.norm(ref.positions) <= FP64_TOL
    assert port.force_rel_error(parts.numpy("vel"), np.asarray(ref.velocities)) <= FP64_TOL


def test_config2_linked_cells_trajectory_vs_oracle(pkg, config2_snapshot):
    """22 steps of LC-C08-N3L-AoS-CSF1 at 1,048,576 particles: the device loop
    reproduces the oracle's, including the periodic-crossing drop the
    build-time src/shift refresh implies."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import simulate
    pos, vel, params = config2_snapshot
    steps, cid = 22, "LC-C08-N3L-AoS-CSF1"
    parts = P.ParticleSet(pos, vel)
    rep = simulate(parts, params, P.parse_configuration(cid), steps=steps, record=False)
    assert rep.error is None
    ref = port.Particles(pos, vel)
    with port.Pool(WORKERS) as pool:
        port.simulate_fixed(ref, _oparams(params), port.parse(cid), steps=steps, pool=pool)
    L = np.asarray(params.domain_size)
    dpos = parts.numpy("pos") - np.asarray(ref.positions)
    dpos -= L * np.rint(dpos / L)
    assert np.linalg.norm(dpos) / np.linalg.norm(ref.positions) <= FP64_TOL
    assert port.force_rel_error(parts.numpy("vel"), np.asarray(ref.velocities)) <= FP64_TOL


# -- configs 3 and 4 ------------------------------------------------------------

def test_config3_slab_forces_vs_oracle(pkg):
    """Config 3 (2,097,152 particles, FCC slab + vacuum, 128 x 128 x 640)."""
    P, calc = pkg
    from paper_2505_03438_b200 import systems
    pos, vel, params = systems.config3_inputs()
    ref_f, ref_n = _oracle_forces(pos, params)
    ids = ["VL-List_Iter-NoN3L-SoA", "LC-SLI-N3L-SoA-CSF1", "LC-C08-N3L-AoS-CSF0.5",
           "VCL-ClusterIter-NoN3L-SoA"]
    _check_families(P, calc, pos, params, ids, ref_f, ref_n)


def test_config4_forces_vs_oracle(pkg):
    """Config 4 (4,194,304 particles at rho = 0.4) after its quench
    (systems.config4_state: relaxed, equilibrated at T = 1.4, rescaled to
    T = 0.7 and run until droplets form), fp64 and the fp32 variant."""
    P, calc = pkg
    from paper_2505_03438_b200 import systems
    pos, vel, params = systems.config4_state(quench_steps=int(os.environ.get("MDG_TEST_QUENCH", "200")))
    ref_f, ref_n = _oracle_forces(pos, params)
    vl = port.VerletLists(port.make_geometry(np.asarray(params.domain_size), params.cutoff + params.skin,
                                             1.0, np.ones(3, bool)))
    vl.rebuild(port.Particles(pos))
    band = _band_pairs(pos, vl.noff, vl.nbr, params)
    ids = ["VL-List_Iter-NoN3L-SoA", "LC-SLI-N3L-SoA-CSF1", "LC-C18-N3L-AoS-CSF0.5",
           "VL-List_Iter-NoN3L-SoA-FP32"]
    _check_families(P, calc, pos, params, ids, ref_f, ref_n, band)


# -- config 5 ---------------------------------------------------------------------

def test_config5_forces_vs_brute_force_oracle(pkg):
    """Config 5 (67,108,864 particles, FCC 256^3, tiled lists past 2^32
    entries) against the reference's brute-force oracle (every row, through a
    cell list: port.sampled_forces): forces within 1e-10 and the exact
    directed count."""
    P, calc = pkg
    from paper_2505_03438_b200 import systems
    pos, vel, params = systems.config5_inputs()
    del vel
    parts = P.ParticleSet(pos, layout="SoA")
    fc = calc.ForceCalculator(parts, params)
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    fc.rebuild(parts, cfg)
    fc.refresh(parts, cfg)
    n_vl = fc.compute(parts, cfg)
    fc.close()
    f_gpu = parts.numpy("force")
    del parts
    torch.cuda.empty_cache()
    f_ref, cnt = port.sampled_forces(pos, np.arange(len(pos)), params.cutoff, params.domain_size,
                                     (True, True, True))
    assert n_vl == int(cnt.sum()), (n_vl, int(cnt.sum()))
    assert port.force_rel_error(f_gpu, f_ref) <= FP64_TOL


# -- device integrator: reflective walls, gravity, two types -----------------------

def _reflect_setup(P, z, layout="AoS"):
    L = z["domain"]
    bnd = tuple(P.PERIODIC if f else P.REFLECTIVE for f in z["periodic"])
    params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=6,
                                delta_t=float(z["dt"]), boundary=bnd, gravity=float(z["gravity"]))
    types = [P.ParticleTypeInfo(t, 1.0 + 0.5 * t, 1.0 - 0.2 * t, 1.0 + t) for t in range(2)]
    parts = P.ParticleSet(z["pos0"], z["vel0"], type_ids=z["tid"], types=types, layout=layout)
    return parts, params


def _traj_err(parts, z, k):
    L = z["domain"]
    per = np.asarray(z["periodic"], dtype=bool)
    dpos = parts.numpy("pos") - z[f"pos_{k}"]
    dpos[:, per] -= L[per] * np.rint(dpos[:, per] / L[per])
    return (np.linalg.norm(dpos) / np.linalg.norm(z[f"pos_{k}"]),
            port.force_rel_error(parts.numpy("vel"), z[f"vel_{k}"]))


def test_reflect_gravity_trajectories_match_reference(pkg):
    """The device loop (drift_wrap / reflect, gravity, finish_kick, the
    masses of two types; integrate.cu) reproduces the real reference's
    trajectories with reflections (integrator.py:47-51, :98-128)."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import simulate
    z = golden("traj_reflect_gravity.npz")
    for k, cid in enumerate(str(s) for s in z["config_ids"]):
        parts, params = _reflect_setup(P, z)
        rep = simulate(parts, params, P.parse_configuration(cid), steps=int(z["steps"]))
        assert rep.error is None, rep.error
        ep, ev = _traj_err(parts, z, k)
        assert ep <= FP64_TOL and ev <= FP64_TOL, (cid, ep, ev)


@pytest.mark.parametrize("mode", ["fused", "graphs"])
def test_reflect_gravity_fused_and_graph_loops_match_reference(pkg, mode):
    """The bench loop's fused kick+drift kernel and the CUDA-graph steady
    state take the same reflective / gravity / two-type branches."""
    P, calc = pkg
    from paper_2505_03438_b200.simulation import Simulation
    z = golden("traj_reflect_gravity.npz")
    ids = [str(s) for s in z["config_ids"]]
    for cid in ("VL-List_Iter-NoN3L-SoA", "LC-C08-N3L-SoA-CSF1"):
        k = ids.index(cid)
        cfg = P.parse_configuration(cid)
        parts, params = _reflect_setup(P, z, cfg.layout)
        sim = Simulation(parts, params, cfg, fuse_kick_drift=(mode == "fused"),
                         graphs=(mode == "graphs"))
        sim.run(int(z["steps"]), record=False)
        sim.check()
        ep, ev = _traj_err(parts, z, k)
        assert ep <= FP64_TOL and ev <= FP64_TOL, (cid, mode, ep, ev)


def test_three_types_200k_forces_vs_oracle(pkg):
    """Three particle types (Lorentz-Berthelot mixing, forces.py:12-22) on
    200,000 relaxed particles: the tiled walk's multi-type path (types staged
    in the window), LC-SLI and the fp32 variant against the oracle."""
    P, calc = pkg
    from paper_2505_03438_b200 import systems
    n = 200_000
    pos, L, rng = systems.uniform_box(n, 0.7, seed=5)
    tid = (np.arange(n) % 3).astype(np.int64)
    types = [P.ParticleTypeInfo(t, 1.0 + 0.5 * t, 1.0 - 0.2 * t, 1.0 + t) for t in range(3)]
    params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                                boundary=(P.PERIODIC,) * 3)
    parts = P.ParticleSet(pos, type_ids=tid, types=types)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    pos = parts.numpy("pos")
    op = _oparams(params)
    p = port.Particles(pos, type_id=tid, sigma=[1.0, 0.8, 0.6], epsilon=[1.0, 1.5, 2.0],
                       mass=[1.0, 2.0, 3.0])
    with port.Pool(WORKERS) as pool:
        fc = port.ForceCalculator(p, op)
        cfg = port.parse("LC-C08-N3L-AoS-CSF1")
        fc.rebuild(p, cfg)
        fc.refresh(p, cfg)
        ref_n = fc.compute(p, cfg, pool)
    ref_f = np.ascontiguousarray(p.forces)
    for cid in ("VL-List_Iter-NoN3L-SoA", "VL-List_Iter-NoN3L-AoS", "LC-SLI-N3L-SoA-CSF1",
                "VL-List_Iter-NoN3L-SoA-FP32"):
        cfgd = P.parse_configuration(cid)
        q = P.ParticleSet(pos, type_ids=tid, types=types, layout=cfgd.layout)
        _, count = calc.compute_forces(q, cfgd, params)
        unique = count if cfgd.newton3 else count // 2
        tol = FP32_TOL if cfgd.precision == "fp32" else FP64_TOL
        if cfgd.precision != "fp32":
            assert unique == ref_n, (cid, unique, ref_n)
        assert port.force_rel_error(q.numpy("force"), ref_f) <= tol, cid
