#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
for env in "" "HRB_NO_GRAPH=1"; do
for spec in "main:" "s36:--log2-args 36" "log36:--fn log --start 0x6A09E667F3BCD --log2-args 36"; do
  n=${spec%%:*}; a=${spec#*:}
  env $env timeout 600 python bench.py --no-cpu-baseline --no-e2e $a > gpurun_out/q_$n.json 2> gpurun_out/q_$n.err
  python -c "
import json; d=json.load(open('gpurun_out/q_$n.json')); r=d['roofline']
print('$env', '$n', round(d['ms_per_step'],4), round(d['value']/1e12,1), d['config']['candidates'])" 2>&1 | tail -1
done; done
