"""Device-timed sweep of every configuration on one synthetic system.

    python tools/sweep.py [--n 1048576] [--reps 5]

Prints one JSON line per configuration: rebuild / refresh / compute times
(CUDA events, median of reps) and the eval count.  This is the landscape the
tuner samples; bench.py uses the winner.
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


def timed(fn, reps):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_048_576)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    pos, vel, params = systems.config2_inputs(n=a.n)
    parts = P.ParticleSet(pos, vel)
    relax_cfg = P.parse_configuration("LC-C01-NoN3L-AoS-CSF1")
    systems.relax_on_device(parts, params, relax_cfg)
    for cfg in P.extended_configurations():
        if a.only and a.only not in cfg.id:
            continue
        p = parts.copy()
        p.convert_layout(cfg.layout)
        calc = ForceCalculator(p, params)
        calc.rebuild(p, cfg)
        t_rebuild = timed(lambda: calc.rebuild(p, cfg), 2)
        t_refresh = timed(lambda: calc.refresh(p, cfg), a.reps)
        calc.compute_async(p, cfg)
        t_compute = timed(lambda: calc.compute_async(p, cfg), a.reps)
        count = calc.last_eval_count
        unique = count if cfg.newton3 else count // 2   # pairs per force evaluation
        print(json.dumps({"config": cfg.id, "n": a.n, "rebuild_ms": round(t_rebuild, 3),
                          "refresh_ms": round(t_refresh, 3), "compute_ms": round(t_compute, 3),
                          "eval_count": count,
                          "gpairs_per_s": round(unique / t_compute / 1e6, 2)}), flush=True)
        calc.close()


if __name__ == "__main__":
    main()
