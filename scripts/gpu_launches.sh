#!/bin/bash
# Bench lines + ncu launch list (per-kernel durations, cold-cache serialised) for the given configs.
# usage: gpu_launches.sh "<configs>" [steps]
mkdir -p gpurun_out
for c in $1; do
  timeout 600 python bench.py --config $c --steps ${2:-30} --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_$c=$?
  python scripts/launch_summary.py gpurun_out/launches_$c.csv
done
