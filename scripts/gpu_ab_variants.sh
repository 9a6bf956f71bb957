#!/bin/bash
# parity tier on the main library AND on every variant library, then timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
for lib in paper_1211_3056_b200/_lib/variants/*.so; do
  n=$(basename $lib .so)
  HRB_LIB=$lib timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$n.log 2>&1; echo "pytest[$n] rc=$?"; tail -n 1 gpurun_out/pytest_gpu_$n.log
done
export VARIANT_SPECS="${VARIANT_SPECS:-eps20:--log2-args_36_--eps-bits_20}"
bash scripts/gpu_variants.sh
bash scripts/gpu_variants.sh
