for cps in 4 8 16; do for u in 128 512 2048; do
  FFSAT_GLOBAL_CPS=$cps FFSAT_GLOBAL_UNIT=$u timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c5_${cps}_${u}.json 2>/dev/null
done; done
for cps in 4 8 16; do FFSAT_GLOBAL_CPS=$cps timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/c4_${cps}.json 2>/dev/null; done
