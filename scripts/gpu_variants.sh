#!/bin/bash
# Quick phase timings of every variant library (no CPU baseline, no e2e).
mkdir -p gpurun_out
for lib in paper_1211_3056_b200/_lib/variants/*.so; do
  n=$(basename $lib .so)
  for spec in "main:" ${VARIANT_SPECS}; do
    t=${spec%%:*}; a=${spec#*:}; a=${a//_/ }
    HRB_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 $a > gpurun_out/var_${n}_$t.json 2> gpurun_out/var_${n}_$t.err
    python -c "
import json; d=json.load(open('gpurun_out/var_${n}_$t.json')); r=d['roofline']
print('$n $t', round(d['ms_per_step'],4), [round(x,4) for x in r['phase_ms_incl_compaction']], d['config']['candidates'])" 2>&1 | tail -1
  done
done
