#!/bin/bash
# Round-2 evidence (end of round): GPU tests, smoke, every bench line, the reference arm, a 2-rank dry run, ncu
# launch lists (per-kernel time + DRAM bytes -> profiles/ncu_summary.json) and --set full captures of the dominant
# kernels, summarised into profiles/ with tag r02.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
for c in c1 c3 c3b256 c4 c4p c5; do timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref=$?
timeout 900 python bench.py --gpus 2 --steps 50 --warmup 5 --tts-seeds 1 > gpurun_out/bench2_c2.json 2> gpurun_out/bench2_c2.err; echo bench2_c2=$?
timeout 900 python bench.py --gpus 2 --config c5 --steps 10 --warmup 3 > gpurun_out/bench2_c5.json 2> gpurun_out/bench2_c5.err; echo bench2_c5=$?
for c in c2 c3 c4 c5; do bash scripts/gpu_launches.sh $c 600 > gpurun_out/launches_$c.log 2>&1; echo launches_$c=$?; done
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
B="python bench.py --no-cpu-baseline --tts-seeds 0"
timeout 900 $N -k "regex:fast_tmem_kernel.*bool.0" -s 12 -c 1 -o gpurun_out/prof_tmem -f $B --steps 5 --warmup 3 > /dev/null 2>&1; echo ncu_tmem=$?
timeout 900 $N -k "regex:fast_tmem_kernel.*bool.1" -s 2 -c 1 -o gpurun_out/prof_tmem_chk -f $B --steps 5 --warmup 3 > /dev/null 2>&1; echo ncu_tmem_chk=$?
timeout 900 $N -k "regex:sym_tree_kernel" -s 1 -c 1 -o gpurun_out/prof_tree -f $B --config c3 --steps 3 --warmup 1 > /dev/null 2>&1; echo ncu_tree=$?
timeout 900 $N -k "regex:owner_grp_kernel" -s 2 -c 1 -o gpurun_out/prof_own -f $B --config c5 --steps 3 --warmup 1 > /dev/null 2>&1; echo ncu_own=$?
timeout 900 $N -k "regex:fast_global_long" -s 2 -c 1 -o gpurun_out/prof_long -f $B --config c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo ncu_long=$?
timeout 900 $N -k "regex:fast_global_kernel" -s 2 -c 1 -o gpurun_out/prof_short -f $B --config c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo ncu_short=$?
python scripts/profiles_summarize.py r02 > gpurun_out/profiles_summarize.log 2>&1; echo summarize=$?
mkdir -p gpurun_out/profiles_r02 && cp profiles/* gpurun_out/profiles_r02/
rm -f gpurun_out/*.ncu-rep
for f in gpurun_out/bench*.json; do echo $f; head -c 600 $f; echo; done
