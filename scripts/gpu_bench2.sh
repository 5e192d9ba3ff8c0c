#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "pgd_steps" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err; echo bench=$?; tail -3 gpurun_out/bench_c2_full.err; cat gpurun_out/bench_c2_full.json
timeout 900 python bench.py --gpus 2 --steps 50 --warmup 5 --tts-seeds 1 > gpurun_out/bench_c2_g2.json 2> gpurun_out/bench_c2_g2.err; echo bench2=$?; tail -5 gpurun_out/bench_c2_g2.err; cat gpurun_out/bench_c2_g2.json
