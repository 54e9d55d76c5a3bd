"""Per-kernel device times of the Verlet rebuild on config 2 (CUPTI through
torch.profiler, no ncu): binning, sort, build positions, tile plan, the tile
build, and the first (prune) walk that follows it.

    python tools/rebuild_probe.py [--reps 5] [--n 1048576]

Env knobs of libmdg (MDG_VLT_*) pass through, so A/B runs are
`MDG_VLT_BT=320 python tools/rebuild_probe.py`.
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.calculator import ForceCalculator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_048_576)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--config", default="VL-List_Iter-NoN3L-SoA")
    a = ap.parse_args()
    pos, vel, params = systems.config2_inputs(n=a.n)
    parts = P.ParticleSet(pos, vel)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    cfg = P.parse_configuration(a.config)
    parts.convert_layout(cfg.layout)
    calc = ForceCalculator(parts, params)
    for _ in range(2):
        calc.rebuild(parts, cfg)
        calc.compute_async(parts, cfg)
    torch.cuda.synchronize()
    walls = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        calc.rebuild(parts, cfg)
        calc.compute_async(parts, cfg)
        e1.record()
        e1.synchronize()
        walls.append(e0.elapsed_time(e1))
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            calc.rebuild(parts, cfg)
            calc.compute_async(parts, cfg)
        torch.cuda.synchronize()
    rows = []
    for ev in prof.key_averages():
        dt = getattr(ev, "device_time_total", None)
        if dt is None:
            dt = ev.cuda_time_total
        if dt <= 0:
            continue
        rows.append((dt / a.reps, ev.count // a.reps, ev.key[:90]))
    rows.sort(reverse=True)
    env = {k: v for k, v in os.environ.items() if k.startswith("MDG_")}
    print(json.dumps({"config": cfg.id, "n": a.n, "env": env,
                      "rebuild_plus_walk_ms": round(statistics.median(walls), 4),
                      "kernel_sum_us": round(sum(r[0] for r in rows), 1)}))
    for us, cnt, name in rows:
        print(f"  {us:9.1f} us  x{cnt:<3d} {name}")


if __name__ == "__main__":
    main()
