"""The reference's OWN tuning machinery driving the device loop.

``mdtune.tuning.TuningController`` with the reference's strategies
(PredictiveStrategy tuning.py:104-116 / predict_cost :33-82, FullSearch,
ExpertStrategy fuzzy.py:397-411 with the shipped rule base) selects among the
GPU configurations from device-event timings (``simulate`` hands CUDA-event
build / force nanoseconds to ``record_timings``, simulation.py:155-181), and
the controller's live statistics come from the device (``mdg_live_stats``).

The reference is the staged, unmodified package under ``baseline/_ref``
(pip-installed from /root/reference, git-ignored, travels with the
snapshot); without it these tests skip.  Every decision the controller made
is recorded and replayed through the oracle's loop (oracle/port.py
``simulate_controlled``): the device trajectory must equal the oracle's under
the same configuration sequence within the fp64 bar.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT
from oracle import port

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

_REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(_REF) and _REF not in sys.path:
    sys.path.append(_REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mdg_numba_cache")
tuning = pytest.importorskip("mdtune.tuning", reason="reference not staged under baseline/_ref")

FP64_TOL = 1e-10


class _Replay:
    """Replays a recorded (configuration, forced, mode) sequence through the
    controller protocol (for the oracle loop)."""

    def __init__(self, seq):
        self.seq = seq
        self.mode = "steady"

    def configuration_for_iteration(self, it):
        cfg, forced, self.mode = self.seq[it]
        return port.parse(cfg.id), forced

    def record_timings(self, force_ns, build_ns):
        pass

    def record_failure(self, error=None):
        return False


def _recording(base):
    seq = []

    class Recording(base):
        def configuration_for_iteration(self, iteration):
            cfg, forced = super().configuration_for_iteration(iteration)
            seq.append((cfg, bool(forced), self.mode))
            return cfg, forced
    return Recording, seq


def _system(P, n=20_000, seed=3, density=0.75):
    from paper_2505_03438_b200 import systems
    pos, L, rng = systems.uniform_box(n, density, seed=seed)
    vel = systems.thermal_velocities(rng, np.ones(n), 0.7)
    params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=5,
                                delta_t=1e-3, total_iterations=0, boundary=(P.PERIODIC,) * 3)
    parts = P.ParticleSet(pos, vel)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"),
                            steps=30)
    return parts.numpy("pos"), parts.numpy("vel"), params


def _run(P, strategy, steps, interval, space=None, samples=2):
    from dataclasses import replace

    from paper_2505_03438_b200.simulation import simulate
    pos, vel, params = _system(P)
    params = replace(params, total_iterations=steps)
    parts = P.ParticleSet(pos, vel)
    Rec, seq = _recording(tuning.TuningController)
    rep = simulate(parts, params, strategy, tuning_interval=interval, samples_per_config=samples,
                   space=space, controller_cls=Rec)
    return rep, seq, parts, pos, vel, params


def _replay_on_oracle(seq, pos, vel, params):
    op = port.Params(domain_size=tuple(params.domain_size), cutoff=params.cutoff, skin=params.skin,
                     rebuild_interval=params.rebuild_interval, delta_t=params.delta_t,
                     boundary=(port.PERIODIC,) * 3, thread_count=len(os.sched_getaffinity(0)))
    ref = port.Particles(pos, vel)
    port.simulate_controlled(ref, op, _Replay(seq), steps=len(seq))
    return ref


def _assert_matches(parts, ref, params):
    L = np.asarray(params.domain_size)
    ref.convert_layout("AoS")
    dpos = parts.numpy("pos") - np.asarray(ref.positions)
    dpos -= L * np.rint(dpos / L)
    assert np.linalg.norm(dpos) / np.linalg.norm(ref.positions) <= FP64_TOL
    assert port.force_rel_error(parts.numpy("vel"), np.asarray(ref.velocities)) <= FP64_TOL


def test_predictive_strategy_selects_from_device_timings():
    """PredictiveStrategy over the reference's 30 ids: phase 0 trials every
    configuration on device timings, later phases trial the predicted-best
    (plus retrials); every trial iteration delivers positive device
    timings; the run equals the oracle's under the same decisions."""
    import paper_2505_03438_b200 as P
    steps, interval = 150, 75
    rep, seq, parts, pos, vel, params = _run(P, tuning.PredictiveStrategy(), steps, interval)
    assert rep.error is None, rep.error
    trials = rep.tuning_log                               # the controller's own trial rows
    assert len(trials) == rep.trial_iterations > 30      # phase 0 sampled the whole space
    assert all(r.force_time_nanos > 0 and r.build_time_nanos > 0 for r in trials)
    assert len(rep.phase_selections) == 2
    sampled = {r.configuration_id for r in trials}
    assert len(sampled) == 30
    # the phase-0 winner is the cheapest configuration by the controller's own cost
    assert rep.phase_selections[0][1] in sampled
    _assert_matches(parts, _replay_on_oracle(seq, pos, vel, params), params)


def test_full_search_and_expert_strategies_on_device():
    """FullSearch over the extended space (the 30 + fp32 Verlet + VCL ids)
    and ExpertStrategy with the reference's shipped rule base (its
    candidates come from the device live statistics) both run the real
    controller on device timings; the exact-arithmetic runs replay on the
    oracle."""
    import paper_2505_03438_b200 as P
    from mdtune.fuzzy import ExpertStrategy
    from mdtune.rules import default_rule_base
    ext = P.extended_configurations()
    rep, seq, parts, pos, vel, params = _run(P, tuning.FullSearchStrategy(), 90, 90, space=ext,
                                             samples=1)
    assert rep.error is None, rep.error
    assert {r.configuration_id for r in rep.tuning_log} == {c.id for c in ext}
    assert rep.phase_selections[0][1] in {c.id for c in ext}
    space = P.enumerate_configurations()
    rb = default_rule_base(space)
    rep, seq, parts, pos, vel, params = _run(P, ExpertStrategy(rb), 60, 30, space=space)
    assert rep.error is None, rep.error
    assert rep.trial_iterations > 0 and len(rep.phase_selections) == 2
    assert all(r.force_time_nanos > 0 for r in rep.tuning_log)
    _assert_matches(parts, _replay_on_oracle(seq, pos, vel, params), params)
