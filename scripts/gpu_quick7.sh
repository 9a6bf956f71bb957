#!/bin/bash
# parity tier + device and end-to-end timings: main library vs the variants
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
for pass in 1 2; do
for lib in paper_1211_3056_b200/_lib/libhrb200.so paper_1211_3056_b200/_lib/variants/*.so; do
  n=$(basename $lib .so)
  HRB_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/e2e_$n.json 2> gpurun_out/e2e_$n.err
  python -c "
import json; d=json.load(open('gpurun_out/e2e_$n.json')); r=d['roofline']; e=d['e2e']
print('$n', round(d['ms_per_step'],4), 'e2e_ms', round(e['ms_per_step'],4), round(e['value']/1e12,1), [round(x,4) for x in r['phase_ms_incl_compaction']], d['config']['candidates'])" 2>&1 | tail -1
done
done
