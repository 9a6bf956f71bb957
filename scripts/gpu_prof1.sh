#!/bin/bash
mkdir -p gpurun_out
T=${TAG:-p1}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=$T bash scripts/gpu_metrics.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase[12]_reg" -c 2 \
   -o gpurun_out/prof_full_$T -f python scripts/profile_step.py --no-peak > gpurun_out/ncu_full_$T.log 2>&1
tail -n 2 gpurun_out/ncu_full_$T.log
