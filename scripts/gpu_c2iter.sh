#!/bin/bash
# c2 kernel iteration: the GPU suite (optionally filtered), the default bench line, and one ncu --set full capture of
# the no-check TMEM kernel.  usage: gpu_c2iter.sh "<pytest -k expr or empty>" [ncu]
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_gpu.log 2>&1; else timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; fi
echo pytest=$?; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --tts-seeds 0 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_c2.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("value", d["value"] / 1e9, "ms_per_step", d["ms_per_step"], "kernel", r["kernel"], r["kernel_ms"], "bound", r["bound"], round(r["frac"], 3),
      {k: round(v["frac"], 3) for k, v in r["resources"].items()}, "e2e", d["e2e"]["value"] / 1e9)
PY
if [ -n "$2" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:fast_tmem_kernel.*bool.0" -s 12 -c 1 -o gpurun_out/prof_tmem -f python bench.py --no-cpu-baseline --tts-seeds 0 --steps 5 --warmup 3 > gpurun_out/ncu.log 2>&1; echo ncu=$?
  ncu -i gpurun_out/prof_tmem.ncu-rep --page details --csv > gpurun_out/prof_tmem_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_tmem.ncu-rep --page raw --csv > gpurun_out/prof_tmem_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_tmem.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_tmem_sass.csv 2>/dev/null
  rm -f gpurun_out/prof_tmem.ncu-rep
fi
