"""Per-step device times of the bench loop (config 2, fused kick+drift), to
see the rebuild step against the steady steps and the launch/sync gaps.

    python tools/step_probe.py
"""
import gc
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.simulation import Simulation  # noqa: E402


def main():
    if os.environ.get("PROBE_NOGC"):
        gc.disable()
    pos, vel, params = systems.config2_inputs()
    parts = P.ParticleSet(pos, vel)
    systems.relax_on_device(parts, params, P.parse_configuration("LC-SLI-N3L-AoS-CSF1"))
    cfg = P.parse_configuration("VL-List_Iter-NoN3L-SoA")
    if "--sorted" in sys.argv:
        # probe only: the particle arrays in CSF-1 cell order (what a periodic
        # spatial reorder of the state would give)
        L = float(params.domain_size[0])
        nc = int(L // (params.cutoff + params.skin))
        x = parts.view("pos")
        c = torch.clamp((x / (L / nc)).floor().long(), 0, nc - 1)
        key = (c[:, 0] * nc + c[:, 1]) * nc + c[:, 2]
        order = torch.argsort(key * 4096 + (x[:, 2] / (L / nc) * 4095).long().clamp(0, 4095) % 4096)
        parts = P.ParticleSet(parts.view("pos")[order].clone(), parts.view("vel")[order].clone())
    parts.convert_layout(cfg.layout)
    k = int(sys.argv[sys.argv.index('--reorder') + 1]) if '--reorder' in sys.argv else 0
    sim = Simulation(parts, params, cfg, fuse_kick_drift=True, reorder=k)
    for _ in range(11):
        sim.step()
    sim.check()
    sim.warm_reorder()
    torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=parts.pos.device)
    for mode in ("back-to-back", "l2-flushed"):
        ev = []
        host = []
        for k in range(int(os.environ.get('PROBE_STEPS', 22))):
            if mode == "l2-flushed":
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            t0 = time.perf_counter()
            sim.step()
            host.append(round((time.perf_counter() - t0) * 1e3, 3))
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        ms = [round(a.elapsed_time(b), 4) for a, b in ev]
        print(json.dumps({"mode": mode, "ms": ms, "mean": round(sum(ms) / len(ms), 4)}))
        print(json.dumps({"mode": mode, "host_ms": host}))
    # the same steps with no per-step events: one interval over 22 steps
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(22):
        sim.step()
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"mode": "one interval", "mean": round(a.elapsed_time(b) / 22, 4)}))


if __name__ == "__main__":
    main()
