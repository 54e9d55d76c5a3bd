#!/bin/bash
# The reference's full acceptance suite (tests/test_acceptance.py, criteria
# 1-9 + the heating-sphere family switch) against the GPU backend through the
# plugin (run under gpurun; the reference staged under baseline/_ref).
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$(realpath -m "${1:-$ROOT/gpurun_out/ref_acceptance.log}")
mkdir -p "$(dirname "$OUT")"
cd "$ROOT/baseline/_ref/ref_tests"
export PYTHONPATH="$ROOT/baseline/_ref:$ROOT"
export NUMBA_CACHE_DIR=/tmp/mdg_numba_cache
python -m pytest -p paper_2505_03438_b200.plugin -p no:cacheprovider --rootdir . -rA --durations=20 \
    test_acceptance.py > "$OUT" 2>&1
rc=$?
tail -25 "$OUT"
exit $rc
