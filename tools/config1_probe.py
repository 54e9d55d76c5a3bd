"""BASELINE config 1 (8,000 particles) on its own configuration: per-step device
time of the loop, for the launch list.
    python tools/config1_probe.py [CONFIG_ID] [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03438_b200 as P  # noqa: E402
from paper_2505_03438_b200 import systems  # noqa: E402
from paper_2505_03438_b200.simulation import Simulation  # noqa: E402

cid = sys.argv[1] if len(sys.argv) > 1 else "LC-C08-N3L-SoA-CSF1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 44
pos, vel, params = systems.config1_params()
cfg = P.parse_configuration(cid)
parts = P.ParticleSet(pos, vel, layout=cfg.layout)
sim = Simulation(parts, params, cfg, fuse_kick_drift=not os.environ.get("PROBE_GRAPHS"), graphs=bool(os.environ.get("PROBE_GRAPHS")))
for _ in range(11):
    sim.step()
sim.check()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time
a.record()
t0 = time.perf_counter()
if os.environ.get("PROBE_EAGER"):
    for _ in range(steps):
        sim.step()
else:
    sim.run(steps, record=False)   # native fixed-configuration spans (mdg_run)
t1 = time.perf_counter()
sim.flush()
b.record()
b.synchronize()
print(cid, "ms/step", round(a.elapsed_time(b) / steps, 4), "host enqueue ms/step", round((t1 - t0) * 1e3 / steps, 4))
if "--profile" in sys.argv:
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            sim.step()
        sim.flush()
        torch.cuda.synchronize()
    rows = []
    for ev in prof.key_averages():
        dt = getattr(ev, "device_time_total", 0.0)
        if dt > 0:
            rows.append((dt / steps, ev.count / steps, ev.key[:80]))
    rows.sort(reverse=True)
    print("kernel sum us/step", round(sum(r[0] for r in rows), 2))
    for us, cnt, name in rows:
        print(f"  {us:8.2f} us/step  x{cnt:5.2f}  {name}")
