#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r4.log
tail -n 3 gpurun_out/pytest_gpu_r4.log
TAG=r4 bash scripts/gpu_metrics.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1_reg|phase2_reg|phase3_kernel" -c 3 \
   -o gpurun_out/prof_full_r4 -f python scripts/profile_step.py --no-peak > gpurun_out/ncu_full_r4.log 2>&1
tail -n 2 gpurun_out/ncu_full_r4.log
TAG=r4 bash scripts/gpu_configs.sh
