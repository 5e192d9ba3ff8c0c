#!/bin/bash
# compute-sanitizer over a small-size subset of the GPU parity suite: memcheck, racecheck, synccheck, initcheck
mkdir -p gpurun_out
SEL="${SEL:-test_host_buffer or test_long_fast_only_global or test_bit_packed_check or test_c1_3sat or test_mixed_all_kinds or test_edge_cases or test_wide_and_narrow or test_uniform_check or test_rq1_workloads or test_long_cardinality_fp64 or test_check_U or test_initial_points or (test_product_tree_path and (256 or 513)) or test_fista_schedule or test_tmem_tiled_kernel or test_owner_computes_sliced}"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 --target-processes all python -m pytest tests/test_parity_gpu.py -q -x -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3
done
