#!/bin/bash
# perf iteration: gpu tests (filter), bench lines, ncu --set full of one kernel (summary written back)
# usage: gpu_perf.sh "<pytest -k>" "<configs>" "<kernel regex>" "<ncu config>" "<tag>"
mkdir -p gpurun_out
if [ -n "$1" ]; then timeout 1500 python -m pytest tests -m gpu -q -k "$1" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log; fi
for c in $2; do FFSAT_BENCH_DUMP=1 timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --tts-seeds 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; python - <<PY
import json
d=json.load(open("gpurun_out/bench_$c.json")); r=d["roofline"]
print("$c", "ms/step %.4f"%d["ms_per_step"], "value %.3e"%d["value"], "e2e %.3e"%d["e2e"]["value"], r["bound"], "frac %.3f"%r["frac"], "kernel_ms %.4f"%r["kernel_ms"], r["eval_phase_ms"])
PY
done
if [ -n "$3" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$3" -s 12 -c 1 -o gpurun_out/prof_$5 -f python bench.py --config $4 --steps 5 --warmup 3 --no-cpu-baseline --tts-seeds 0 > gpurun_out/ncu_$5.log 2>&1; echo ncu=$?
  python scripts/ncu_summary.py gpurun_out/prof_$5.ncu-rep > gpurun_out/ncu_$5.txt 2>&1; head -60 gpurun_out/ncu_$5.txt
  rm -f gpurun_out/prof_$5.ncu-rep
fi
