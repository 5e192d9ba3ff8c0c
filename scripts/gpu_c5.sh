#!/bin/bash
# c5 iteration: global-path tests, the c5 bench line (default and FFSAT_OWN=0), optional ncu of the owner kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "${1:-owner or c5 or global or batch or determin or long_fast or c4 or sharded or dist}" > gpurun_out/pytest_gpu.log 2>&1
echo pytest=$?; tail -8 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench_c5=$?; tail -2 gpurun_out/bench_c5.err
FFSAT_OWN=1 timeout 600 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_own.json 2> gpurun_out/bench_c5_own.err; echo bench_c5_own=$?
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_c5*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f, "value", d["value"] / 1e9, "ms", d["ms_per_step"], r.get("kernel"), r.get("kernel_ms"), r.get("bound"), round(r.get("frac", 0), 3),
              r.get("eval_phase_ms"), {k: round(v["frac"], 3) for k, v in r["resources"].items()})
    except Exception as e:
        print(f, "parse error", e)
PY
if [ -n "$2" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:owner_ -s 2 -c 1 -o gpurun_out/prof_own -f env FFSAT_OWN=1 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_own.log 2>&1; echo ncu=$?
  python scripts/ncu_summary.py gpurun_out/prof_own.ncu-rep > gpurun_out/ncu_own_summary.txt 2>&1; head -40 gpurun_out/ncu_own_summary.txt
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv env FFSAT_OWN=1 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
  python scripts/launch_summary.py gpurun_out/launches_c5.csv 2>/dev/null | head -12
  ncu -i gpurun_out/prof_own.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_own_sass.csv 2>/dev/null
  ncu -i gpurun_out/prof_own.ncu-rep --page raw --csv > gpurun_out/prof_own_raw.csv 2>/dev/null
  rm -f gpurun_out/prof_own.ncu-rep
fi
