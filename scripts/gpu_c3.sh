#!/bin/bash
mkdir -p gpurun_out
true
for v in 2 1 0; do FFSAT_SYM_TMEM=$v timeout 600 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_t$v.json 2>gpurun_out/bench_c3_t$v.err; echo bench_c3_tmem$v=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_c3_t$v.json')); r=d['roofline']; print('tmem=$v', d['ms_per_step'], r['frac'], r['eval_phase_ms'])"; done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:sym_tmem_kernel.*4, .int.16, .bool.1" -s 1 -c 1 -o gpurun_out/prof_symt -f python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_symt.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py gpurun_out/prof_symt.ncu-rep > gpurun_out/ncu_symt.txt 2>&1; head -50 gpurun_out/ncu_symt.txt; rm -f gpurun_out/prof_symt.ncu-rep
