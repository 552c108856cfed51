#!/bin/bash
# Bench line + ncu launch list (cold, serialised per-launch times) for profiles/.
set -x
python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
    python bench.py --steps 1 --warmup 1 --no-agg --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
tail -c 300 gpurun_out/bench_r1.json
