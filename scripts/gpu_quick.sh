#!/bin/bash
# Quick GPU iteration: parity tests, one bench line per config given, optional ncu --set full of a kernel regex.
# usage: gpu_quick.sh "<configs>" [kernel_regex] [ncu_config]
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for c in $1; do FFSAT_BENCH_DUMP=1 timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; tail -3 gpurun_out/bench_$c.err; done
if [ -n "$2" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o gpurun_out/prof_$2 -f python bench.py --config ${3:-c2} --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$2.log 2>&1; echo ncu=$?
fi
cat gpurun_out/bench_*.json
timeout 300 python scripts/diag_step.py c2 > gpurun_out/diag_c2.txt 2>&1; cat gpurun_out/diag_c2.txt
