#!/bin/bash
# parity tier, then per variant library: the e2e probe in a fresh process
# (first call on an unsized workspace) and the bench's device + e2e timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
for lib in paper_1211_3056_b200/_lib/variants/*.so; do
  n=$(basename $lib .so)
  echo "probe $n: $(HRB_LIB=$lib timeout 300 python scripts/e2e_probe.py 2>&1 | tail -1)"
done
for pass in 1 2; do
for lib in paper_1211_3056_b200/_lib/variants/*.so; do
  n=$(basename $lib .so)
  HRB_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/e2e_$n.json 2> gpurun_out/e2e_$n.err
  python -c "
import json; d=json.load(open('gpurun_out/e2e_$n.json')); e=d['e2e']
print('$n', round(d['ms_per_step'],4), 'e2e_ms', round(e['ms_per_step'],4))" 2>&1 | tail -1
done
done
