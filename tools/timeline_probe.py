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
    ap.add_argument("--config", type=int, default=2, help="BASELINE config (tools/configs_bench.py inputs)")
    ap.add_argument("--summary", action="store_true", help="per-kernel totals instead of the timeline")
    ap.add_argument("--all", action="store_true", help="every event of the timeline (default: gaps > 3 us or > 20 us)")
    a = ap.parse_args()
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import configs_bench
    a.quench, a.n5_side = 4000, 256
    pos, vel, params, relax = configs_bench.inputs(a.config, a)
    parts = P.ParticleSet(pos, vel)
    if relax:
        systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    parts.convert_layout(cfg.layout)
    sim = Simulation(parts, params, cfg, fuse_kick_drift=True, reorder=16 if a.config in (2, 4) else 0)
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
    print(json.dumps({"config": a.config, "steps": a.steps, "window_us": round(total, 1),
                      "busy_us": round(busy, 1), "idle_us": round(total - busy, 1)}))
    if a.summary:
        agg = {}
        for s, e, n in evs:
            t = agg.setdefault(n, [0.0, 0])
            t[0] += e - s
            t[1] += 1
        for n, (us, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:16]:
            print(f"  {us / a.steps:9.1f} us/step  x{cnt / a.steps:5.2f}  {n}")
        return
    for r in rows:
        if a.all or r["gap_us"] > 3 or r["dur_us"] > 20:
            print(f'{r["t_us"]:10.1f} {r["dur_us"]:8.1f} gap {r["gap_us"]:7.1f}  {r["name"]}')


if __name__ == "__main__":
    main()
