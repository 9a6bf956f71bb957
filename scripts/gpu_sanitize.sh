#!/bin/bash
# compute-sanitizer passes over the small parity cases (race
# detection on the compaction atomics and the shared-memory walk state).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K='pipeline_case_matches_reference and (p13_exp_b0 or p53_exp_2p20_e16_N12 or p53_exp_F128 or p53_exp_ragged) or fused_and_host or search_batch_matches'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py -q -x -k "$K" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -n 4 gpurun_out/sanitize_$tool.log
  # the classic family's per-warp queue (shared memory + atomics) in all three
  # modes, and the device generation
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py tests/test_devgen_gpu.py -q -x \
     -k "(iteration_sums and lefevre) or device_pack_equals_reference_fixture or resident" > gpurun_out/sanitize2_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize2_$tool.log
  tail -n 4 gpurun_out/sanitize2_$tool.log
done
