"""Probe for the dynamic-pruning design: how the tiled walk's time
scales with the list radius, and how far particles move per step on config 2.

    python tools/prune_probe.py

Prints one JSON line per skin (walk ms, list entries) and one line with the
per-step maximum displacement over an 11-step window.
"""

import dataclasses
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.calculator import ForceCalculator  # noqa: E402
from paper_2505_03438_b200.simulation import Simulation  # noqa: E402


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
    pos, vel, params = systems.config2_inputs()
    parts = P.ParticleSet(pos, vel)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-C01-NoN3L-AoS-CSF1"))
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    for skin in (0.3, 0.2, 0.15, 0.1, 0.05, 0.0):
        pr = dataclasses.replace(params, skin=skin)
        p = parts.copy()
        p.convert_layout(cfg.layout)
        calc = ForceCalculator(p, pr)
        calc.rebuild(p, cfg)
        calc.refresh(p, cfg)
        calc.compute_async(p, cfg)
        t = timed(lambda: calc.compute_async(p, cfg), 9)
        print(json.dumps({"skin": skin, "ell": 2.5 + skin, "compute_ms": round(t, 4),
                          "evals": calc.last_eval_count}), flush=True)
    p = parts.copy()
    p.convert_layout(cfg.layout)
    sim = Simulation(p, params, config=cfg)
    sim.run(11)
    L = torch.tensor(params.domain_size, dtype=torch.float64, device=p.pos.device)
    x0 = p.positions.clone()
    prev = x0.clone()
    rows = []
    for s in range(22):
        sim.run(1)
        x = p.positions
        d = x - x0
        d -= L * torch.round(d / L)
        e = x - prev
        e -= L * torch.round(e / L)
        rows.append((round(float(d.norm(dim=1).max()), 5), round(float(e.norm(dim=1).max()), 5)))
        prev = x.clone()
    print(json.dumps({"max_disp_since_0_and_per_step": rows}))


if __name__ == "__main__":
    main()
