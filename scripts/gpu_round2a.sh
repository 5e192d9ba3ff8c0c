#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -q > gpurun_out/pytest_dist_gpu.log 2>&1; echo pytest_dist=$?; tail -3 gpurun_out/pytest_dist_gpu.log
timeout 1500 python scripts/table2_portfolio.py gpurun_out/table2_portfolio.json 10 > gpurun_out/table2.log 2>&1; echo table2=$?; cat gpurun_out/table2.log | tail -16
