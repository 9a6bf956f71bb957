"""bench.py under torchrun with two ranks on one GPU (HRB_BENCH_ONE_DEVICE=1:
both ranks on cuda:0, gloo for the collectives): exercises the rank
partition, the barriers, the max-over-ranks timing and the end-of-run
gather on every GPU test run.  The merged counters must equal a one-rank
run over the same total range (weak scaling: 2 x 2^30 arguments)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _last_json(out: str) -> dict:
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


def test_two_ranks_on_one_gpu_equal_one_rank():
    common = ["--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-e2e-full", "--wide-delta", "0"]
    env = dict(os.environ, HRB_BENCH_ONE_DEVICE="1", NCCL_DEBUG="WARN")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                          "--log2-args", "30", *common], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=900)
    assert two.returncode == 0, two.stderr[-3000:]
    line2 = _last_json(two.stdout)
    one = subprocess.run([sys.executable, "bench.py", "--log2-args", "31", *common], cwd=ROOT, capture_output=True,
                         text=True, timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    line1 = _last_json(one.stdout)
    assert line2["n_gpus"] == 2 and line1["n_gpus"] == 1
    for k in ("phase1_fail", "phase2_survivors", "candidates"):
        assert line2["config"][k] == line1["config"][k], k
    assert line2["value"] > 0 and line2["ms_per_step"] > 0
