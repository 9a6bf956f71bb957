#!/bin/bash
# Interleaved A/B timings of the variant libraries (default workload, no e2e,
# no CPU baseline): ROUNDS passes over every variant, one bench line each.
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-2}); do
  for lib in paper_1211_3056_b200/_lib/variants/*.so; do
    n=$(basename $lib .so)
    HRB_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-e2e-full --wide-delta 0 --steps 20 ${BENCH_ARGS} \
      > gpurun_out/ab_${n}_$r.json 2> gpurun_out/ab_${n}_$r.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_${n}_$r.json')); r=d['roofline']
print('$n', round(d['ms_per_step'],4), [round(x,4) for x in r['phase_ms_incl_compaction']])" 2>&1 | tail -1
  done
done
