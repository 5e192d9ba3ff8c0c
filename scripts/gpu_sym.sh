#!/bin/bash
# root-path iteration: parity tests, bench c3 per FFSAT_SYM_VARIANT, optional ncu of the root kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/pytest_sym.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_sym.log
for v in ${VARIANTS:-0 1 2 3}; do
  FFSAT_SYM_VARIANT=$v timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_v$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_c3_v$v.json')); print('c3 variant $v', round(d['value']/1e9,3), round(d['ms_per_step'],3), 'root ms', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],4))"
done
if [ -n "$1" ]; then FFSAT_SYM_VARIANT=$1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_item -s 2 -c 1 -o gpurun_out/prof_sym -f python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu=$?; fi
