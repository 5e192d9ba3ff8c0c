#!/bin/bash
# c5 with the grouped owner kernel at 8 / 4 / 2 threads per variable (32 / 16 / 8-point x^T slices), 2 runs each,
# and the owner parity tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "owner" 2>&1 | tail -2
for l in 8 4 2; do for r in 1 2; do FFSAT_OWN_LANES=$l timeout 300 python bench.py --config c5 --steps 30 --warmup 5 --no-cpu-baseline --tts-seeds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('lanes=$l', d['ms_per_step'], d['roofline']['resources']['alu']['time_ms'])"; done; done
L=${1:-}
if [ -n "$L" ]; then FFSAT_OWN_LANES=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:owner_grp -c 1 -o gpurun_out/own_grp_l$L -f python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --tts-seeds 0 > /dev/null 2>&1; echo ncu=$?; fi
