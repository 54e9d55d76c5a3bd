#!/bin/bash
# per-step times of bench.py's timed loop: spikes (> 1.5 ms) by step index
# usage: tools/spike_probe.sh TAG [bench args...]   (run under gpurun)
mkdir -p gpurun_out/sp
tag=$1; shift
MDG_BENCH_STEPS=1 python bench.py --no-e2e --no-cpu "$@" > gpurun_out/sp/$tag.json 2> gpurun_out/sp/$tag.err
python - "$tag" <<'PY'
import json, statistics, sys
t = sys.argv[1]
d = json.loads(open(f"gpurun_out/sp/{t}.json").read().strip().splitlines()[-1])
st = hm = None
for l in open(f"gpurun_out/sp/{t}.err"):
    l = l.strip()
    try:
        if l.startswith("["):
            st = json.loads(l)
        elif l.startswith("host_ms "):
            hm = json.loads(l[8:])
    except Exception:
        pass
print(t, "MUPS", d["value"], "ms/step", d["ms_per_step"], "median", statistics.median(st),
      "spikes>1.5ms (step, device ms, host ms of that step() and the one before):",
      [(i, x, hm[i] if hm else None, hm[i - 1] if hm and i else None) for i, x in enumerate(st) if x > 1.5], "clock samples", d["clocks"]["samples"])
PY
grep "cudaMallocs by torch" gpurun_out/sp/$tag.err
grep "reorder steps\|grid_rebuild: waited" gpurun_out/sp/$tag.err | cut -c1-400
