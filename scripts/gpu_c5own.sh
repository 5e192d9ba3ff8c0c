#!/bin/bash
# full -m gpu suite, smoke, c5 + c4 + c2 bench lines with the grouped owner kernel on by default, c5 launch list with
# DRAM bytes, and one ncu --set full of owner_grp_kernel on c5
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -6 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
for c in c5 c4 c2; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --tts-seeds 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; head -c 300 gpurun_out/bench_$c.json; echo; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --tts-seeds 0 > /dev/null 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:owner_grp -c 1 -o gpurun_out/ncu_c5_owner_grp -f python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --tts-seeds 0 > /dev/null 2>&1; echo ncu=$?
