#!/bin/bash
# Full GPU session: parity tests, smoke, default bench line (c2, with cpu_baseline and time-to-solve), the other
# configs, the reference arm, ncu launch lists and one --set full capture per dominant kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref=$?
for c in c2 c3 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --tts-seeds 0 > /dev/null 2>&1; echo ncu_launch_$c=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_wide -s 5 -c 1 -o gpurun_out/prof_tiled -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline --tts-seeds 0 > /dev/null 2>&1; echo ncu_tiled=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_item -s 2 -c 1 -o gpurun_out/prof_sym -f python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu_sym=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_global_kernel -s 2 -c 1 -o gpurun_out/prof_global -f python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu_global=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_global_long -s 2 -c 1 -o gpurun_out/prof_long -f python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_long=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_global_kernel -s 2 -c 1 -o gpurun_out/prof_short -f python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_short=$?
for f in gpurun_out/bench_*.json; do echo $f; head -c 400 $f; echo; done
# summarise on the box (the .ncu-rep files exceed gpurun's 64 MiB merge limit), ship the summaries back
python scripts/profiles_summarize.py r01 > gpurun_out/profiles_summarize.log 2>&1; echo summarize=$?
mkdir -p gpurun_out/profiles_r01 && cp profiles/* gpurun_out/profiles_r01/
rm -f gpurun_out/*.ncu-rep
