"""e2e MUPS of hostloop.HostSimulation.run vs the chunk count (config 2).

    python tools/e2e_chunks.py [--chunks 2,4,8,16] [--steps 44]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.hostloop import HostParticleSet, HostSimulation  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", default="2,4,8,16")
    ap.add_argument("--steps", type=int, default=44)
    ap.add_argument("--config", default="VL-List_Iter-NoN3L-SoA")
    a = ap.parse_args()
    pos, vel, params = systems.config2_inputs()
    parts = P.ParticleSet(pos, vel)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    hp, hv = parts.numpy("pos"), parts.numpy("vel")
    cfg = P.parse_configuration(a.config)
    for k in [int(x) for x in a.chunks.split(",")]:
        p = HostParticleSet(hp, hv)
        sim = HostSimulation(p, params, cfg, chunks=k)
        sim.run(2)
        for rep in range(2):
            t0 = time.perf_counter()
            sim.run(a.steps)
            dt = time.perf_counter() - t0
            print(f"chunks {k:3d} rep {rep}: {len(hp) * a.steps / dt / 1e6:8.1f} MUPS "
                  f"({dt / a.steps * 1e3:.3f} ms/step)", flush=True)
        del sim, p


if __name__ == "__main__":
    main()
