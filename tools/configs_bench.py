"""Device-timed MUPS of every BASELINE configuration on ONE GPU (22 warm-up steps) (informational;
bench.py's line is config 2).  Config 1 runs its BASELINE configuration
(LC-C08-N3L-SoA-CSF1) and the VL walk; configs 2-5 the VL walk.  Configs 2 and
4 are relaxed first (uniform inputs overlap); 3 and 5 are FCC.

    python tools/configs_bench.py [--configs 1,2,3,4,5] [--steps 22] [--n5-side 256]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.simulation import Simulation  # noqa: E402


def inputs(k, a):
    if k == 1:
        pos, vel, L = systems.sc_lattice()
        params = P.SimulationParams(domain_size=L, cutoff=2.5, skin=0.3, rebuild_interval=10,
                                    delta_t=1e-3, boundary=(P.PERIODIC,) * 3)
        return pos, vel, params, False
    if k == 2:
        pos, vel, params = systems.config2_inputs()
        return pos, vel, params, True
    if k == 3:
        pos, vel, params = systems.config3_inputs()
        return pos, vel, params, False
    if k == 4:   # relaxed, equilibrated at T = 1.4, quenched to T = 0.7 (droplets)
        stats = []
        pos, vel, params = systems.config4_state(equil_steps=a.quench // 2, quench_steps=a.quench,
                                                 stats=stats)
        print(json.dumps({"config": 4, "quench_steps": a.quench,
                          "live_stats_before_after": [s.feature_vector()[:6].tolist() for s in stats]}),
              flush=True)
        return pos, vel, params, False
    pos, vel, params = systems.config5_inputs(n_side=a.n5_side)
    return pos, vel, params, False


def run(k, cid, a):
    t0 = time.time()
    pos, vel, params, relax = inputs(k, a)
    parts = P.ParticleSet(pos, vel)
    del pos, vel
    if relax:
        systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    cfg = P.parse_configuration(cid)
    parts.convert_layout(cfg.layout)
    # cell-order arrays pay off for inputs in random particle order (configs 2
    # and 4: uniform random positions); the lattice generators (1, 3, 5) emit
    # particles in a spatially coherent order already
    reorder = a.reorder if k in (2, 4) else 0
    sim = Simulation(parts, params, cfg, fuse_kick_drift=True, reorder=reorder)
    # warm-up through run() as timed below: the native loop's step graphs are
    # captured and instantiated here, not inside the timed steps
    sim.run(22, record=False)
    sim.check()
    sim.warm_reorder()
    torch.cuda.synchronize()
    a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    sim.run(a.steps, record=False)   # flushes; fixed-configuration spans in one native call (mdg_run)
    b0.record()
    b0.synchronize()
    ms = a0.elapsed_time(b0)
    sim.check()
    n = parts.n
    out = {"config": k, "configuration": cid, "n": n, "steps": a.steps, "ms_per_step": round(ms / a.steps, 4),
           "mups": round(n * a.steps / (ms * 1e-3) / 1e6, 1),
           "unique_pairs": sim.calc.last_eval_count // (1 if cfg.newton3 else 2),
           "gpu_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2),
           "setup_s": round(time.time() - t0, 1)}
    print(json.dumps(out), flush=True)
    del sim, parts
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=22)
    ap.add_argument("--reorder", type=int, default=8,
                    help="cell-order arrays every K rebuilds for configs 2 and 4 (VL; 0 = off)")
    ap.add_argument("--n5-side", type=int, default=256)
    ap.add_argument("--quench", type=int, default=4000, help="config 4: steps at T=0.7 after half as many at 1.4")
    a = ap.parse_args()
    for k in [int(x) for x in a.configs.split(",")]:
        cids = (["LC-C08-N3L-SoA-CSF1", "VL-List_Iter-NoN3L-SoA"] if k == 1 else
                ["VL-List_Iter-NoN3L-SoA", "VL-List_Iter-NoN3L-SoA-FP32"] if k == 4 else   # + the fp32 variant
                ["VL-List_Iter-NoN3L-SoA"])
        for cid in cids:
            try:
                run(k, cid, a)
            except Exception as exc:
                print(json.dumps({"config": k, "configuration": cid, "error": f"{type(exc).__name__}: {exc}"}),
                      flush=True)
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
