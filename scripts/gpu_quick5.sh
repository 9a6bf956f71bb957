#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
for spec in "lef:--algo lefevre" "main:"; do
  n=${spec%%:*}; a=${spec#*:}
  timeout 600 python bench.py --no-cpu-baseline --no-e2e $a > gpurun_out/q_$n.json 2> gpurun_out/q_$n.err
  python -c "
import json; d=json.load(open('gpurun_out/q_$n.json')); r=d['roofline']
print('$n', round(d['ms_per_step'],4), round(d['value']/1e12,1), [round(x,4) for x in r['phase_ms_incl_compaction']], d['config']['phase1_fail'], d['config']['candidates'])" 2>&1 | tail -1
done
