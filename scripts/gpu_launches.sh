#!/bin/bash
# ncu launch list of a short bench run for config $1 -> gpurun_out/launches_$1.csv, summarised per kernel
mkdir -p gpurun_out
c=${1:-c2}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c ${2:-400} --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --tts-seeds 0 > /dev/null 2>&1; echo ncu_launch_$c=$?
python scripts/launch_summary.py gpurun_out/launches_$c.csv $c | tee gpurun_out/launch_summary_$c.csv; mkdir -p gpurun_out/prof; cp profiles/ncu_summary.json gpurun_out/prof/
