#!/bin/bash
# Full GPU session: parity tests, default bench line (c2, with cpu_baseline), the other configs, the reference
# arm, the ncu launch list of the default bench and one --set full capture per dominant kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_launch=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_launch3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_wide -s 5 -c 1 -o gpurun_out/prof_tiled -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_tiled=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_item -s 2 -c 1 -o gpurun_out/prof_sym -f python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu_sym=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_global -s 2 -c 1 -o gpurun_out/prof_global -f python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu_global=$?
for f in gpurun_out/bench_*.json; do echo $f; head -c 600 $f; echo; done
