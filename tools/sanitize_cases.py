"""Small systems through every kernel family built on shared-memory atomics,
mbarrier / bulk-copy rings or fp64 RED, for compute-sanitizer (one tool per
run; tools/sanitize.sh):

* the tiled Verlet walk (producer warp + bulk copies + mbarriers), its prune
  walk (inner lists re-written every step: delta tiny) and the fp32 walk;
* the tile build (lane-per-row scan, shared-memory windows);
* linked cells C08 (colour launches), C18 / SLI (fp64 RED), C01;
* Verlet cluster lists N3L (shuffle-reduced reactions + fp64 atomics);
* the fused kick+drift loop, the cell reorder, the live statistics and the
  thermostat reductions.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.calculator import compute_forces  # noqa: E402
from paper_2505_03438_b200.simulation import Simulation  # noqa: E402

IDS = ["VL-List_Iter-NoN3L-SoA", "VL-List_Iter-NoN3L-AoS", "VL-List_Iter-NoN3L-SoA-FP32",
       "LC-C08-N3L-SoA-CSF1", "LC-C08-NoN3L-AoS-CSF0.5", "LC-C18-N3L-AoS-CSF1",
       "LC-SLI-N3L-SoA-CSF1", "LC-SLI-NoN3L-AoS-CSF0.5", "LC-C01-NoN3L-SoA-CSF1",
       "VCL-ClusterIter-N3L-AoS", "VCL-ClusterIter-NoN3L-SoA"]


def main():
    pos, vel, L = systems.sc_lattice(n_side=16, seed=2)      # 4,096 particles
    params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=4,
                                delta_t=2e-3, boundary=(P.PERIODIC,) * 3,
                                thermostat=P.ThermostatParams(0.7, 0.1, 3))
    for cid in IDS:
        cfg = P.parse_configuration(cid)
        parts = P.ParticleSet(pos, layout=cfg.layout)
        _, n = compute_forces(parts, cfg, params)
        print(cid, "count", n, flush=True)
    # the loop: fused kick+drift, reorder at every rebuild, prune every step
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    parts = P.ParticleSet(pos, vel, layout="SoA")
    sim = Simulation(parts, params, cfg, fuse_kick_drift=True, reorder=1)
    sim.calc.set_prune(0.002)
    sim.run(12, record=False)
    sim.check()
    print("prunes", sim.calc.prune_count(), "T", sim.calc.temperature(parts),
          "stats", sim.calc.live_stats(parts).feature_vector()[:4], flush=True)
    print("sanitize cases done")


if __name__ == "__main__":
    main()
