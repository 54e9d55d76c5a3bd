#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py, ONE tool per call (several
# tools in one call have left B200 boxes unusable, B200_PROFILING.md):
#   tools/sanitize.sh racecheck|memcheck|synccheck|initcheck
set -u
tool=${1:-memcheck}
mkdir -p gpurun_out/san
compute-sanitizer --tool "$tool" --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_cases.py > "gpurun_out/san/$tool.log" 2>&1
rc=$?
echo "rc=$rc"; tail -6 "gpurun_out/san/$tool.log"
exit $rc
