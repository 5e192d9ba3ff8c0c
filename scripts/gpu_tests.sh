#!/bin/bash
# GPU iteration: the -m gpu suite (optionally a -k filter), smoke, and quick bench lines for the given configs.
# usage: gpu_tests.sh "<pytest -k expr or empty>" "<configs>"
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_gpu.log 2>&1; else timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; fi
echo pytest=$?; tail -30 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -25
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
for c in $2; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --tts-seeds 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; tail -3 gpurun_out/bench_$c.err; head -c 700 gpurun_out/bench_$c.json; echo; done
