"""CPU-only checks: the C-ABI library loads and exports every symbol of
include/mdg.h; host-side geometry/stencils through the ABI equal the
reference's (golden); the host mirror of the configuration space and params
behaves like the reference's."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

from paper_2505_03438_b200 import _lib
import paper_2505_03438_b200 as P


def test_header_and_export_list_agree():
    hdr = open(os.path.join(ROOT, "include", "mdg.h")).read()
    declared = set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(mdg_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = _lib.lib()
    for name in _lib.EXPORTS:
        assert hasattr(L, name), name
    assert L.mdg_version().decode().startswith("mdg")


def _geom(domain, per, ell, csf):
    d = np.ascontiguousarray(domain, dtype=np.float64)
    p = np.ascontiguousarray(per, dtype=np.int32)
    so, ov, ha, di = (np.zeros(3, np.int32) for _ in range(4))
    cl = np.zeros(3)
    _lib.check(_lib.lib().mdg_geometry_for(d.ctypes.data, p.ctypes.data, ell, csf, so.ctypes.data,
                                           cl.ctypes.data, ov.ctypes.data, ha.ctypes.data,
                                           di.ctypes.data))
    return so, cl, ov, ha, di


def _stencil(domain, per, ell, csf, kind, major=0):
    d = np.ascontiguousarray(domain, dtype=np.float64)
    p = np.ascontiguousarray(per, dtype=np.int32)
    out = np.zeros(3 * 124, np.int32)
    cnt = ctypes.c_int()
    _lib.check(_lib.lib().mdg_stencil_for(d.ctypes.data, p.ctypes.data, ell, csf, kind, major,
                                          ctypes.byref(cnt), out.ctypes.data))
    return out[:3 * cnt.value].reshape(-1, 3).astype(np.int64)


def test_abi_geometry_and_stencils_match_reference():
    z = golden("geometry.npz")
    for k in range(int(z["n_cases"])):
        dom, (ell, csf), per = z[f"g{k}_in_domain"], z[f"g{k}_in_scalars"], z[f"g{k}_in_periodic"]
        so, cl, ov, ha, di = _geom(dom, per, ell, csf)
        assert tuple(so) == tuple(z[f"g{k}_dims_owned"])
        assert np.array_equal(cl, z[f"g{k}_cell_length"])
        assert tuple(ov) == tuple(z[f"g{k}_overlap"])
        assert tuple(ha) == tuple(z[f"g{k}_halo"])
        assert tuple(di) == tuple(z[f"g{k}_dims"])
        assert np.array_equal(_stencil(dom, per, ell, csf, 0), z[f"g{k}_pruned"])
        for major in range(3):
            assert np.array_equal(_stencil(dom, per, ell, csf, 1, major), z[f"g{k}_forward{major}"])


def test_abi_rejects_bad_geometry():
    with pytest.raises(ValueError):
        _geom((9.0, 9.0, 9.0), (1, 1, 1), 3.0, 0.7)


def test_configuration_space_mirrors_reference():
    space = P.enumerate_configurations()
    assert len(space) == 30 and len({c.id for c in space}) == 30
    from oracle import port
    assert [c.id for c in space] == [c.id for c in port.all_configs()]
    for c in space:
        assert P.parse_configuration(c.id) == c
    with pytest.raises(ValueError):
        P.Configuration("VL", "List_Iter", True, "AoS")
    with pytest.raises(ValueError):
        P.Configuration("LC", "C01", True, "AoS")
    with pytest.raises(ValueError):
        P.Configuration("LC", "C08", True, "AoS", 0.25)
    with pytest.raises(ValueError):
        P.parse_configuration("LC-C04-N3L-AoS-CSF1")


def test_params_validation_mirrors_reference():
    with pytest.raises(ValueError):
        P.SimulationParams(domain_size=(5.0, 9.0, 9.0), cutoff=2.5, skin=0.3,
                           boundary=(P.PERIODIC,) * 3)
    P.SimulationParams(domain_size=(5.0, 9.0, 9.0), cutoff=2.5, skin=0.3,
                       boundary=(P.REFLECTIVE, P.PERIODIC, P.PERIODIC))
    with pytest.raises(ValueError):
        P.SimulationParams(domain_size=(9.0, 9.0, 9.0), cutoff=0.0)


def test_config_struct_mapping():
    s = _lib.config_struct(P.parse_configuration("LC-SLI-NoN3L-SoA-CSF0.5"))
    assert (s.container, s.traversal, s.newton3, s.layout, s.csf) == (_lib.LC, _lib.SLI, 0, _lib.SOA, 0.5)
    s = _lib.config_struct(P.parse_configuration("VL-List_Iter-NoN3L-AoS"))
    assert (s.container, s.traversal, s.layout) == (_lib.VL, _lib.LIST_ITER, _lib.AOS)


def test_particle_layout_round_trip_cpu_tensors():
    rng = np.random.default_rng(0)
    p = P.ParticleSet(rng.uniform(0, 9, (50, 3)), rng.normal(size=(50, 3)), device="cpu")
    pos = p.numpy("pos")
    p.convert_layout(P.SOA)
    assert tuple(p.pos.shape) == (3, 50)
    p.convert_layout(P.AOS)
    assert np.array_equal(p.numpy("pos"), pos)
    e = P.ParticleSet(np.zeros((0, 3)), device="cpu")
    e.convert_layout(P.SOA)
    assert tuple(e.pos.shape) == (3, 0)


def test_native_host_integrator_matches_reference_numpy_bit_exact():
    """libmdg's host integrator (used by the host drop-in loop) reproduces the
    reference's numpy drift/boundaries/kick sequence bit for bit."""
    from oracle import port
    from paper_2505_03438_b200 import hostloop
    rng = np.random.default_rng(5)
    n = 2000
    for boundary in ((P.PERIODIC,) * 3, (P.REFLECTIVE, P.PERIODIC, P.REFLECTIVE)):
        params = P.SimulationParams(domain_size=(9.0, 10.0, 11.0), cutoff=2.5, skin=0.3,
                                    delta_t=0.01, boundary=boundary, gravity=-1.5)
        pos = rng.uniform(-0.5, 1.05, (n, 3)) * params.domain_size
        vel = rng.normal(0, 3.0, (n, 3))
        frc = rng.normal(0, 50.0, (n, 3))
        tid = np.arange(n) % 2
        for layout in ("AoS", "SoA"):
            a = hostloop.HostParticleSet(pos, vel, tid, sigma=[1, .8], epsilon=[1, 1.5],
                                         mass=[1.0, 2.0], layout=layout)
            a.view("force")[:] = frc
            b = port.Particles(pos, vel, tid, sigma=[1, .8], epsilon=[1, 1.5], mass=[1.0, 2.0],
                               layout=layout)
            b.view("force")[:] = frc
            pp = port.Params(domain_size=params.domain_size, cutoff=2.5, skin=0.3, delta_t=0.01,
                             boundary=boundary, gravity=-1.5)
            assert not hostloop.host_drift_wrap(a, params, params.delta_t)
            port.drift_with_force(b, pp.delta_t)
            port.apply_boundaries(b, pp)
            np.copyto(b.view("old_force"), b.view("force"))
            assert np.array_equal(a.positions, b.positions)
            assert np.array_equal(a.velocities, b.velocities)
            a.view("force")[:] *= 0.5
            b.view("force")[:] *= 0.5
            hostloop.host_finish_kick(a, params.delta_t, params.gravity)
            port.apply_gravity(b, pp.gravity)
            port.finish_kick(b, pp.delta_t)
            assert np.array_equal(a.velocities, b.velocities)
            assert np.array_equal(a.forces, b.forces)


def test_fused_kick_drift_equals_kick_then_drift():
    """mdg_host_kick_drift_range (mdg_host_run's per-chunk pass) = finish_kick
    then the swapped drift, bit for bit, for every layout / typing /
    boundary combination."""
    import ctypes
    from paper_2505_03438_b200 import _lib, hostloop
    lib = _lib.lib()
    rng = np.random.default_rng(9)
    n = 3001
    for boundary in ((P.PERIODIC,) * 3, (P.REFLECTIVE, P.PERIODIC, P.REFLECTIVE)):
        params = P.SimulationParams(domain_size=(9.0, 10.0, 11.0), cutoff=2.5, skin=0.3,
                                    delta_t=0.01, boundary=boundary, gravity=-1.5)
        pos = rng.uniform(0.0, 1.0, (n, 3)) * params.domain_size
        vel = rng.normal(0, 3.0, (n, 3))
        fnew = rng.normal(0, 50.0, (n, 3))
        fold = rng.normal(0, 50.0, (n, 3))
        for typed in (False, True):
            tid = np.arange(n) % 2 if typed else np.zeros(n, dtype=np.int64)
            mass = [1.0, 2.0] if typed else [1.3]
            for layout in ("AoS", "SoA"):
                mk = lambda: hostloop.HostParticleSet(pos, vel, tid, sigma=[1] * len(mass),
                                                      epsilon=[1] * len(mass), mass=mass,
                                                      layout=layout)
                a, b = mk(), mk()
                for q in (a, b):
                    q.view("force")[:] = fnew
                    q.view("old_force")[:] = fold
                # reference: kick, then the drift with F -> F_old swapped
                hostloop.host_finish_kick(b, params.delta_t, params.gravity)
                b.force, b.old_force = b.old_force, b.force
                L = np.ascontiguousarray(params.domain_size, dtype=np.float64)
                per = np.ascontiguousarray(params.periodic_flags().astype(np.int32))
                m = np.ascontiguousarray(mass, dtype=np.float64)
                t32 = np.ascontiguousarray(tid, dtype=np.int32)
                ly = _lib.AOS if layout == "AoS" else _lib.SOA
                bad = ctypes.c_int()
                P_ = hostloop._ptr
                assert lib.mdg_host_drift_wrap_range_ex(n, 0, n, ly, P_(b.pos), P_(b.vel), P_(b.force),
                                                        P_(b.old_force), P_(t32) if typed else None,
                                                        P_(m), P_(L), P_(per), params.delta_t, 1,
                                                        ctypes.byref(bad)) == 0
                for lo, hi in ((0, 1000), (1000, n)):
                    assert lib.mdg_host_kick_drift_range(n, lo, hi, ly, P_(a.pos), P_(a.vel), P_(a.force),
                                                         P_(a.old_force), P_(t32) if typed else None,
                                                         P_(m), P_(L), P_(per), params.delta_t, 1, -1.5,
                                                         ctypes.byref(bad)) == 0
                    assert bad.value == 0
                # b's current forces now live in b.old_force (swapped); a's in a.force
                assert np.array_equal(a.positions, b.positions), (boundary, typed, layout)
                assert np.array_equal(a.velocities, b.velocities), (boundary, typed, layout)
                assert np.array_equal(a.forces, b.old_forces), (boundary, typed, layout)


def test_native_host_integrator_flags_blow_up():
    from paper_2505_03438_b200 import hostloop
    params = P.SimulationParams(domain_size=(10.0, 10.0, 10.0), cutoff=3.0,
                                boundary=(P.PERIODIC,) * 3)
    for bad in ([-10.5, 5.0, 5.0], [25.0, 5.0, 5.0], [np.nan, 5.0, 5.0]):
        p = hostloop.HostParticleSet(np.array([bad]))
        assert hostloop.host_drift_wrap(p, params, 0.0)


def test_extended_space_keeps_reference_ids():
    ext = P.extended_configurations()
    assert [c.id for c in ext[:30]] == [c.id for c in P.enumerate_configurations()]
    assert [c.id for c in ext[30:]] == ["VL-List_Iter-NoN3L-AoS-FP32", "VL-List_Iter-NoN3L-SoA-FP32",
                                        "VCL-ClusterIter-N3L-AoS", "VCL-ClusterIter-N3L-SoA",
                                        "VCL-ClusterIter-NoN3L-AoS", "VCL-ClusterIter-NoN3L-SoA"]
    vcl = P.parse_configuration("VCL-ClusterIter-N3L-AoS")
    assert vcl.newton3 and _lib.config_struct(vcl).container == _lib.VCL
    with pytest.raises(ValueError):
        P.Configuration("VCL", "List_Iter", False, "AoS")
    with pytest.raises(ValueError):
        P.Configuration("VCL", "ClusterIter", False, "AoS", 0.5)
    assert P.parse_configuration("VL-List_Iter-NoN3L-SoA-FP32").precision == "fp32"
    with pytest.raises(ValueError):
        P.Configuration("LC", "C08", True, "AoS", 1.0, "fp32")
    s = _lib.config_struct(P.parse_configuration("VL-List_Iter-NoN3L-AoS-FP32"))
    assert s.precision == 1


def test_pairwise_order_matches_numpy_sum():
    """The device reductions (stats.cu PairwiseTree) replay numpy's pairwise
    summation; pin that order against np.sum itself, bit for bit, on lengths
    that hit every branch (< 8, <= 128, odd splits)."""
    from oracle import port
    rng = np.random.default_rng(11)
    for n in [1, 2, 7, 8, 9, 15, 16, 127, 128, 129, 255, 256, 257, 1000, 4099, 65537]:
        a = rng.random(n) * rng.standard_normal(n) * 1e3
        assert port.pairwise_sum(a) == np.sum(a), n
    v = rng.standard_normal((1000, 3))
    assert np.array_equal(np.sum(v * v, axis=1), (v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2])
    c = rng.integers(0, 40, 999)
    assert np.array_equal((c - 13.7) ** 2, (c - 13.7) * (c - 13.7))


def test_livestats_feature_order():
    from paper_2505_03438_b200.livestats import FEATURE_NAMES, LiveStatistics
    assert FEATURE_NAMES[0] == "meanParticlesPerBin" and FEATURE_NAMES[-1] == "skin"
    s = LiveStatistics(1.0, 2.0, 3.0, 4.0, 5, 6, 7, 0.3)
    assert list(s.feature_vector()) == [1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 0.3]


def test_host_wrap_matches_np_mod_on_edges():
    """The integrator's np.mod fast path (no fmod inside [-L, 2L], host.cpp /
    integrate.cu) against numpy's np.mod, bit for bit, on the edge values."""
    from paper_2505_03438_b200 import hostloop
    L = 11.18183
    e = np.nextafter
    xs = np.array([0.0, -0.0, 1e-300, -1e-300, -5e-324, L, e(L, 0), e(L, 3 * L), 2 * L, e(2 * L, 0),
                   -L, e(-L, 0), -1e-17, -L / 3, 1.5 * L, 0.7 * L, e(0.0, 1), 3 * L / 2 + 1e-9,
                   -0.9999999999 * L, 1.9999999999 * L])
    rng = np.random.default_rng(3)
    xs = np.concatenate([xs, rng.uniform(-L, 2 * L, 5000)])
    pos = np.repeat(xs[:, None], 3, axis=1)
    params = P.SimulationParams(domain_size=(L, L, L), cutoff=2.5, skin=0.3,
                                boundary=(P.PERIODIC,) * 3)
    p = hostloop.HostParticleSet(pos)
    assert not hostloop.host_drift_wrap(p, params, 0.001)
    want = np.mod(pos, L)
    got = p.pos
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_dataset_columns_match_reference_format():
    """§8(f) row 3: the GPU sweep writes the reference's CSV layout
    (dataset.py:143-146): 8 features in livestats order, cost:<id> per
    configuration, final 'label'."""
    from paper_2505_03438_b200 import dataset
    cols = dataset.dataset_columns()
    assert cols[:8] == ["meanParticlesPerBin", "relStdDevParticlesPerBin", "medianParticlesPerBin",
                        "maxParticlesPerBin", "numBins", "numEmptyBins", "threadCount", "skin"]
    assert cols[8:-1] == [f"cost:{c.id}" for c in P.enumerate_configurations()]
    assert cols[-1] == "label"
    assert dataset.evidence_cost(100.0, 1100.0, 10) == 210.0
    with pytest.raises(ValueError):
        dataset.evidence_cost(1.0, 1.0, 0)


def test_integration_stub_matches_the_abi_struct():
    """INTEGRATION.md's ctypes stub declares mdg_config exactly as
    include/mdg.h and _lib.MdgConfig do (six fields, 32 bytes), so a
    maintainer copying it hands libmdg the layout it reads."""
    import ctypes
    import re
    from paper_2505_03438_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"class _Cfg\(ctypes.Structure\):.*?\n(    _fields_ = \[.*?\])\n", text, re.S)
    assert m, "stub not found"
    I, D = ctypes.c_int, ctypes.c_double
    ns = {"I": I, "D": D}
    exec(m.group(1).strip(), ns)
    stub = [(n, t) for n, t in ns["_fields_"]]
    assert stub == list(_lib.MdgConfig._fields_)

    class Stub(ctypes.Structure):
        _fields_ = stub
    assert ctypes.sizeof(Stub) == ctypes.sizeof(_lib.MdgConfig) == 32
    hdr = open(os.path.join(ROOT, "include", "mdg.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} mdg_config;", hdr, re.S).group(1)
    names = re.findall(r"(?:int|double)\s+(\w+);", body)
    assert names == [n for n, _ in stub]
