#!/bin/bash
# parity tier + phase timings of the variant libraries (two passes for noise)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
export VARIANT_SPECS="${VARIANT_SPECS:-eps20:--log2-args_36_--eps-bits_20}"
bash scripts/gpu_variants.sh
bash scripts/gpu_variants.sh
