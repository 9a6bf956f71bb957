#!/bin/bash
# Full evidence run (one GPU): parity, calibration metrics, ncu full capture
# with source, launch list, bench (ours + reference arm), config-2 search bench.
mkdir -p gpurun_out
T=${TAG:-r3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
TAG=$T bash scripts/gpu_metrics.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1_reg|phase2_reg|phase3_kernel" -c 3 \
   -o gpurun_out/prof_full_$T -f python scripts/profile_step.py --no-peak > gpurun_out/ncu_full_$T.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 900 python scripts/bench_search.py > gpurun_out/bench_search_$T.json 2> gpurun_out/bench_search_$T.err
tail -n 3 gpurun_out/pytest_gpu_$T.log; cat gpurun_out/bench_$T.json gpurun_out/bench_ref_$T.json gpurun_out/bench_search_$T.json
