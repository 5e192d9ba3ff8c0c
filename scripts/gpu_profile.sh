set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fast_tiled -s 3 -c 1 -o gpurun_out/prof_tiled python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:check_kernel -s 0 -c 1 -o gpurun_out/prof_check python bench.py --steps 12 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1; echo ncu3=$?
ls -la gpurun_out
