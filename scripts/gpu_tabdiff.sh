#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/bench_tabdiff.py > gpurun_out/bench_tabdiff.json 2> gpurun_out/bench_tabdiff.err
cat gpurun_out/bench_tabdiff.json; tail -n 3 gpurun_out/bench_tabdiff.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:tabdiff -c 2 --csv --log-file gpurun_out/metrics_tabdiff.csv python scripts/bench_tabdiff.py --reps 1 > /dev/null 2>&1
grep -E "dram__bytes|duration|throughput|issue" gpurun_out/metrics_tabdiff.csv | tail -12 | cut -d, -f5,13,14,15 
