"""Device loop with and without the CUDA-graph steady state (mdg_step_graph):
ms per step for BASELINE config 1 (8,000 particles) and config 2 (1,048,576)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.simulation import Simulation  # noqa: E402

for name, n in (("config1", 8000), ("config2", 1_048_576)):
    if name == "config1":
        pos, vel, L = systems.sc_lattice(n_side=20, seed=0)
        params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                                    delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
    else:
        pos, vel, params = systems.config2_inputs(n=n)
        tmp = P.ParticleSet(pos, vel)
        systems.relax_on_device(tmp, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
        pos, vel = tmp.numpy("pos"), tmp.numpy("vel")
    for cid in ("VL-List_Iter-NoN3L-SoA", "LC-C08-N3L-SoA-CSF1"):
        cfg = P.parse_configuration(cid)
        for graphs in (False, True):
            parts = P.ParticleSet(pos, vel, layout=cfg.layout)
            sim = Simulation(parts, params, cfg, graphs=graphs)
            sim.run(22, record=False)
            torch.cuda.synchronize()
            steps = 220 if name == "config1" else 110
            t = time.perf_counter()
            sim.run(steps, record=False)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t) / steps
            print(f"{name} {cid} graphs={graphs}: {dt * 1e3:.4f} ms/step  {n / dt / 1e6:.1f} MUPS")
