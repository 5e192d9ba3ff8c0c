#!/bin/bash
# product-tree iteration: its tests, the c3 bench line (tree and FFSAT_TREE=0), optional ncu of the tree kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "${1:-tree or long or c3 or card or rq1 or root or paper}" > gpurun_out/pytest_gpu.log 2>&1
echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log
for c in c3 ${2:-}; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; tail -2 gpurun_out/bench_$c.err
  FFSAT_TREE=0 timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_roots.json 2> gpurun_out/bench_${c}_roots.err; echo bench_${c}_roots=$?
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_c3*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f, "value", d["value"] / 1e9, "ms", d["ms_per_step"], r.get("kernel"), r.get("kernel_ms"), r.get("bound"), round(r.get("frac", 0), 3))
    except Exception as e:
        print(f, "parse error", e)
PY
if [ -n "$3" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_tree_kernel -s 2 -c 1 -o gpurun_out/prof_tree -f python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_tree.log 2>&1; echo ncu=$?
  python scripts/ncu_summary.py gpurun_out/prof_tree.ncu-rep > gpurun_out/ncu_tree_summary.txt 2>&1; head -60 gpurun_out/ncu_tree_summary.txt
  ncu -i gpurun_out/prof_tree.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_tree_cuda.csv 2>/dev/null
  ncu -i gpurun_out/prof_tree.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_tree_sass.csv 2>/dev/null
  rm -f gpurun_out/prof_tree.ncu-rep
fi
