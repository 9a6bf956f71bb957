#!/bin/bash
# Multi-rank bench logic on a one-GPU box: every rank on cuda:0 over gloo
# (HRB_BENCH_ONE_DEVICE=1); partition, max-over-ranks timing and the
# end-of-run gather run exactly as under NCCL.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
HRB_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --log2-args 36 --no-e2e > gpurun_out/multirank2.json 2> gpurun_out/multirank2.err
echo "rc=$?"; cat gpurun_out/multirank2.json; tail -n 5 gpurun_out/multirank2.err
timeout 600 python bench.py --log2-args 36 --eps-bits 16 --steps 5 --no-e2e --cpu-seconds 3 > gpurun_out/cfg5_eps16_r5.json 2> gpurun_out/cfg5_eps16_r5.err
cat gpurun_out/cfg5_eps16_r5.json; tail -n 3 gpurun_out/cfg5_eps16_r5.err
