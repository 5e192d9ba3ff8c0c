mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fast_global_long -s 2 -c 1 -o gpurun_out/prof_long -f python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_long.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_global_kernel" -s 2 -c 1 -o gpurun_out/prof_short -f python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_short.log 2>&1; echo ncu=$?
