#!/bin/bash
# The measurement package of a round on one B200 (run under gpurun):
# bench lines (ours, reference arm), the ncu launch list of the timed loop,
# `ncu --set full` of one rebuild window of walks and of the tile build.
# Outputs in gpurun_out/; summarise with tools/launch_list.py and
# tools/ncu_summary.py into profiles/.
set -u
MDG_BENCH_STEPS=1 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 22 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:vlt_force_kernel -s 11 -c 11 \
    -o gpurun_out/walk_window python bench.py --steps 11 --warmup 11 --no-e2e --no-cpu > gpurun_out/ncu_walk.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:vlt_build_kernel -c 1 \
    -o gpurun_out/build1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_build.log 2>&1
ls -la gpurun_out
