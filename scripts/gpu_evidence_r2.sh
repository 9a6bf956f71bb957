#!/bin/bash
# Round-2 evidence (one GPU): parity, bench (ours + reference arm), the
# launch list and full ncu captures, configs 2-5, the high-degree path, the
# device confirmation, a two-rank run on one GPU.
mkdir -p gpurun_out
T=${TAG:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
TAG=$T bash scripts/gpu_metrics.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1_reg|phase2_reg|phase3_kernel" -c 3 \
   -o gpurun_out/prof_full_$T -f python scripts/profile_step.py --no-peak > gpurun_out/ncu_full_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1_wide|phase2_wide|phase3_wide|wseed" -c 4 \
   -o gpurun_out/prof_wide_$T -f python scripts/wide_probe.py --deltas 4 --steps 1 > gpurun_out/ncu_wide_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1_reg" -c 1 \
   -o gpurun_out/prof_classic_$T -f python scripts/profile_step.py --no-peak --algo lefevre > gpurun_out/ncu_classic_$T.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pack_blocks" -c 1 \
   -o gpurun_out/prof_gen_$T -f python scripts/devgen_probe.py > gpurun_out/ncu_gen_$T.log 2>&1
timeout 300 python scripts/devgen_probe.py > gpurun_out/devgen_$T.json 2> gpurun_out/devgen_$T.err
timeout 600 python scripts/e2e_full_probe.py --interval 40 > gpurun_out/e2e_full_probe_$T.json 2> gpurun_out/e2e_full_probe_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-e2e-full --wide-delta 0 > gpurun_out/ncu_launch_$T.log 2>&1
timeout 900 python scripts/bench_search.py --verdicts > gpurun_out/bench_search_$T.json 2> gpurun_out/bench_search_$T.err
for e in 16 20 24 28 32; do
  timeout 600 python bench.py --log2-args 36 --eps-bits $e --steps 5 --no-e2e --cpu-seconds 3 > gpurun_out/cfg5_eps${e}_$T.json 2>> gpurun_out/cfg_$T.err
done
timeout 900 python bench.py --fn log --start 0x6A09E667F3BCD --log2-args 36 --steps 5 --no-e2e --cpu-seconds 3 --wide-delta 0 > gpurun_out/cfg4_log_$T.json 2>> gpurun_out/cfg_$T.err
timeout 900 python bench.py --algo lefevre --steps 5 --no-e2e --cpu-seconds 3 --wide-delta 0 --no-e2e-full > gpurun_out/cfg3_lefevre_$T.json 2>> gpurun_out/cfg_$T.err
timeout 900 python scripts/wide_probe.py --deltas 3,4,5,6,7,8 --check > gpurun_out/wide_probe_$T.jsonl 2> gpurun_out/wide_probe_$T.err
timeout 300 python scripts/confirm_probe.py --host > gpurun_out/confirm_probe_$T.json 2> gpurun_out/confirm_probe_$T.err
HRB_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --log2-args 36 --no-e2e --wide-delta 0 > gpurun_out/multirank2_$T.json 2> gpurun_out/multirank2_$T.err
echo "multirank rc=$?"
tail -n 3 gpurun_out/pytest_gpu_$T.log gpurun_out/smoke_$T.log
# keep the merge-back under 64 MiB: the captures as CSV pages, not .ncu-rep
for rep in gpurun_out/prof_*_$T.ncu-rep; do
  [ -f "$rep" ] || continue
  b=${rep%.ncu-rep}
  ncu -i "$rep" --page raw --csv > "${b}_raw.csv" 2>/dev/null
  ncu -i "$rep" --page source --csv --print-source sass > "${b}_src.csv" 2>/dev/null
  gzip -f "${b}_src.csv"
  rm -f "$rep"
done
du -sh gpurun_out
