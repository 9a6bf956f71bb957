#!/bin/bash
# Round-end evidence (one GPU): parity, calibration metrics, ncu full capture
# of the three phase kernels, launch list of the bench command, the bench
# (ours + reference arm), config 2 (search only), configs 3-lefevre / 4 / 5.
mkdir -p gpurun_out
T=${TAG:-r5}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
TAG=$T bash scripts/gpu_metrics.sh
TAG=${T}_lef PROFILE_ARGS="--algo lefevre --no-peak" bash scripts/gpu_metrics.sh
M=$(grep -o 'M=.*' scripts/gpu_metrics.sh | head -1 | cut -c3-)
timeout 600 ncu --metrics $M --clock-control none -k regex:"search_batch|search_verdict" --csv \
  --log-file gpurun_out/metrics_search_$T.csv python scripts/bench_search.py --reps 1 --no-cpu --verdicts > gpurun_out/metrics_search_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"phase1_reg|phase2_reg|phase3_kernel" -c 3 \
   -o gpurun_out/prof_full_$T -f python scripts/profile_step.py --no-peak > gpurun_out/ncu_full_$T.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 900 python scripts/bench_search.py --verdicts > gpurun_out/bench_search_$T.json 2> gpurun_out/bench_search_$T.err
for e in 16 20 24 28 32; do
  timeout 600 python bench.py --log2-args 36 --eps-bits $e --steps 5 --no-e2e --cpu-seconds 3 > gpurun_out/cfg5_eps${e}_$T.json 2>> gpurun_out/cfg_$T.err
done
timeout 600 python bench.py --fn log --start 0x6A09E667F3BCD --log2-args 36 --steps 5 --no-e2e --cpu-seconds 3 > gpurun_out/cfg4_log_$T.json 2>> gpurun_out/cfg_$T.err
timeout 900 python bench.py --algo lefevre --steps 5 --no-e2e --cpu-seconds 3 > gpurun_out/cfg3_lefevre_$T.json 2>> gpurun_out/cfg_$T.err
tail -n 3 gpurun_out/pytest_gpu_$T.log gpurun_out/smoke_$T.log
cat gpurun_out/bench_$T.json
HRB_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --log2-args 36 --no-e2e > gpurun_out/multirank2_$T.json 2> gpurun_out/multirank2_$T.err
echo "multirank rc=$?"
# where the end-to-end call's time goes (fresh process: unsized workspace)
timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e_probe_$T.log 2>&1
tail -n 1 gpurun_out/e2e_probe_$T.log
