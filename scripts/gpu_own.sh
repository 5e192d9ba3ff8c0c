#!/bin/bash
# owner-computes on c5: parity tests, then the c5 bench line for the default path and FFSAT_OWN=1 at 1 / 2 / 4 points
# per thread, and an ncu --set full capture of the owner kernel (usage: gpu_own.sh [ppt for ncu])
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "owner or c5" > gpurun_out/pytest_own.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_own.log
timeout 300 python bench.py --config c5 --steps 30 --warmup 5 --no-cpu-baseline --tts-seeds 0 > gpurun_out/own_c5_default.json 2> gpurun_out/own_c5_default.err; echo default=$?; head -c 330 gpurun_out/own_c5_default.json; echo
for p in 1 2 4; do
  FFSAT_OWN=1 FFSAT_OWN_PPT=$p timeout 300 python bench.py --config c5 --steps 30 --warmup 5 --no-cpu-baseline --tts-seeds 0 > gpurun_out/own_c5_p$p.json 2> gpurun_out/own_c5_p$p.err; echo own_p$p=$?; head -c 330 gpurun_out/own_c5_p$p.json; echo; tail -2 gpurun_out/own_c5_p$p.err
done
P=${1:-}
if [ -n "$P" ]; then
  FFSAT_OWN=1 FFSAT_OWN_PPT=$P timeout 600 ncu --set full --clock-control none --import-source on -k regex:owner_grp -c 1 -o gpurun_out/own_grp_p$P -f python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --tts-seeds 0 > gpurun_out/ncu_own.log 2>&1; echo ncu=$?
  FFSAT_OWN=1 FFSAT_OWN_PPT=$P timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/own_launches_p$P.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --tts-seeds 0 > /dev/null 2>&1; echo launches=$?
fi
