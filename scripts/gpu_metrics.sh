#!/bin/bash
# Targeted ncu metric capture for the roofline calibration (one GPU).
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed_pipe_fmaheavy.sum,smsp__inst_executed_pipe_fmalite.sum,smsp__inst_executed_pipe_xu.sum,smsp__inst_executed_pipe_fp64.sum,smsp__inst_executed_pipe_cbu.sum,smsp__inst_executed_pipe_lsu.sum,smsp__inst_executed_pipe_adu.sum,smsp__inst_executed_pipe_uniform.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__sass_branch_targets_threads_divergent.sum,smsp__sass_branch_targets.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"phase1|phase2|phase3|int_peak" --csv \
  --log-file gpurun_out/metrics_${TAG:-run}.csv python scripts/profile_step.py ${PROFILE_ARGS} > gpurun_out/metrics_${TAG:-run}.log 2>&1
echo "metrics rc=$?"
