"""GPU timeline of the bench loop around one Verlet rebuild (config 2): every
kernel / memset / copy with its start, duration and the idle gap before it
(CUPTI via torch.profiler; no ncu), to see where the rebuild step waits.

    python tools/timeline_probe.py [--steps 13]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.simulation import Simulation  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=13)
    a = ap.parse_args()
    pos, vel, params = systems.config2_inputs()
    parts = P.ParticleSet(pos, vel)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    parts.convert_layout(cfg.layout)
    sim = Simulation(parts, params, cfg, fuse_kick_drift=True, reorder=16)
    for _ in range(22):
        sim.step()
    sim.check()
    sim.warm_reorder()
    # align so that the profiled window starts two steps before a rebuild
    while sim.since != params.rebuild_interval - 2:
        sim.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(a.steps):
            sim.step()
        sim.flush()
        torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            evs.append((e.time_range.start, e.time_range.end, e.name[:70]))
    evs.sort()
    t0 = evs[0][0]
    prev_end = evs[0][0]
    rows = []
    for s, e, n in evs:
        rows.append({"t_us": round(s - t0, 1), "dur_us": round(e - s, 1), "gap_us": round(s - prev_end, 1), "name": n})
        prev_end = max(prev_end, e)
    total = evs[-1][1] - t0
    busy = sum(e - s for s, e, _ in evs)
    print(json.dumps({"window_us": round(total, 1), "busy_us": round(busy, 1), "idle_us": round(total - busy, 1)}))
    for r in rows:
        if r["gap_us"] > 3 or r["dur_us"] > 20:
            print(f'{r["t_us"]:10.1f} {r["dur_us"]:8.1f} gap {r["gap_us"]:7.1f}  {r["name"]}')


if __name__ == "__main__":
    main()
