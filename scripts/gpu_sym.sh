#!/bin/bash
# root-path iteration: parity tests, bench c3 for each value of $SYMENV (e.g. "FFSAT_SYM_RECOMPUTE=0 FFSAT_SYM_RECOMPUTE=1")
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/pytest_sym.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_sym.log
for e in ${SYMENV:-NONE=0}; do
  env $e timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$e.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_c3_$e.json')); print('c3 $e', round(d['value']/1e9,3), 'ms/step', round(d['ms_per_step'],3), 'root ms', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],4))"
done
if [ -n "$1" ]; then env $1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_item -s 2 -c 1 -o gpurun_out/prof_sym -f python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu=$?; fi
