"""Where the end-to-end (host-array) step spends its time, config 2.

    python tools/e2e_breakdown.py [--n 1048576] [--steps 22] [--config VL-List_Iter-NoN3L-SoA]

Times the pieces of hostloop.HostSimulation.step separately (wall clock, the
GPU calls synchronise): host drift, H2D + compute + D2H, host kick.
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import hostloop, systems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_048_576)
    ap.add_argument("--steps", type=int, default=22)
    ap.add_argument("--config", default="VL-List_Iter-NoN3L-SoA")
    a = ap.parse_args()
    pos, vel, params = systems.config2_inputs(n=a.n)
    parts = P.ParticleSet(pos, vel)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    cfg = P.parse_configuration(a.config)
    p = hostloop.HostParticleSet(parts.numpy("pos"), parts.numpy("vel"))
    sim = hostloop.HostSimulation(p, params, cfg)
    sim.run(2)
    tot = {"drift": 0.0, "rebuild": 0.0, "compute(h2d+gpu+d2h)": 0.0, "kick": 0.0}
    t_all = time.perf_counter()
    for _ in range(a.steps):
        t0 = time.perf_counter()
        hostloop.host_drift_wrap(p, params, params.delta_t)
        t1 = time.perf_counter()
        rebuild = sim.active != cfg.id or sim.since >= params.rebuild_interval
        if p.layout != cfg.layout:
            p.convert_layout(cfg.layout)
        if rebuild:
            sim.calc.rebuild(p, cfg)
        t2 = time.perf_counter()
        sim.calc.refresh(p, cfg)
        sim.calc.compute(p, cfg)
        t3 = time.perf_counter()
        hostloop.host_finish_kick(p, params.delta_t, params.gravity)
        t4 = time.perf_counter()
        sim.active = cfg.id
        sim.since = 0 if rebuild else sim.since + 1
        tot["drift"] += t1 - t0
        tot["rebuild"] += t2 - t1
        tot["compute(h2d+gpu+d2h)"] += t3 - t2
        tot["kick"] += t4 - t3
    dt = time.perf_counter() - t_all
    print(f"{a.config}: {a.n * a.steps / dt / 1e6:.1f} MUPS end to end, {dt / a.steps * 1e3:.3f} ms/step")
    for k, v in tot.items():
        print(f"  {k:24s} {v / a.steps * 1e3:8.3f} ms/step")
    print(f"  host threads: {os.cpu_count()}")


if __name__ == "__main__":
    main()
