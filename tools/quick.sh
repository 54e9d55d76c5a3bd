#!/bin/bash
# quick A/B on the GPU box: bench (device arm only) + optional pytest filter
# usage: tools/quick.sh TAG [pytest -k expr]
mkdir -p gpurun_out/q
tag=$1; shift
python bench.py --no-e2e --no-cpu > gpurun_out/q/$tag.json 2> gpurun_out/q/$tag.err
python - "$tag" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/q/{sys.argv[1]}.json").read().strip().splitlines()[-1])
r=d["roofline"]
print(sys.argv[1], "MUPS", d["value"], "ms/step", d["ms_per_step"], "kernel_ms", r["kernel_ms_avg"], "frac", r["frac"])
PY
if [ -n "$1" ]; then python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/q/$tag.test.log 2>&1; tail -2 gpurun_out/q/$tag.test.log; fi
