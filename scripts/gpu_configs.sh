#!/bin/bash
# BASELINE configs 4 (log over [1,2) at 2^36 from X ~ sqrt(2)) and 5 (eps
# sweep at 2^36 exp), plus the classic-walk variant of config 3.
mkdir -p gpurun_out
T=${TAG:-r4}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for e in 16 20 24 28 32; do
  timeout 600 python bench.py --log2-args 36 --eps-bits $e --steps 5 --no-e2e --cpu-seconds 3 > gpurun_out/cfg5_eps${e}_$T.json 2>> gpurun_out/cfg_$T.err
done
timeout 600 python bench.py --fn log --start 0x6A09E667F3BCD --log2-args 36 --steps 5 --no-e2e --cpu-seconds 3 > gpurun_out/cfg4_log_$T.json 2>> gpurun_out/cfg_$T.err
timeout 900 python bench.py --algo lefevre --steps 5 --no-e2e --cpu-seconds 3 > gpurun_out/cfg3_lefevre_$T.json 2>> gpurun_out/cfg_$T.err
tail -n 5 gpurun_out/cfg_$T.err
for f in gpurun_out/cfg*_$T.json; do python -c "
import json,sys; d=json.load(open('$f')); c=d['config']; print('$f', round(d['value']/1e12,2), 'T args/s', round(d['ms_per_step'],3), 'ms', c['phase1_fail'], c['phase2_survivors'], c['candidates'], d.get('cpu_baseline',{}).get('counts_match_gpu'))"; done
