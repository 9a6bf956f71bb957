"""Stage times of run_range over one 2^40 interval with the device
generation (bench e2e_full's configuration), warm, median of 5: planning,
pack_plan (device generation + download + batch), execute_batch_host
(upload + phases + download), confirmation, and run_range itself.  One GPU.

    python scripts/e2e_stages.py [--log2-args 40]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def med(f, n=5):
    import torch

    f()
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts)) * 1e3, r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-args", type=int, default=40)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    import torch

    from paper_1211_3056_b200 import FpFormat, PhaseConfig, PipelineConfig, PolyGenConfig, hostgen
    from paper_1211_3056_b200.device import pack_columns_device
    from paper_1211_3056_b200.funnel import execute_batch_host, run_range
    from paper_1211_3056_b200.slices import pack_plan, plan_arrays

    pg = PolyGenConfig(tau=512, N=1 << 15, mu=16, nu=32, delta=2, limbs=8, frac_bits=96, guard=32)
    cfg = PipelineConfig("exp", FpFormat(53, 32), pg, PhaseConfig("regular", phase2_split=8, N1=1 << 15))
    count = 1 << a.log2_args
    w = a.workers
    out = {}
    out["plan_ms"], plan = med(lambda: plan_arrays("exp", 0, cfg.fmt, pg, 0, count))
    hc = hostgen.make_cfg("exp", cfg.fmt, pg, 0, 64)
    out["devgen_call_ms"], _ = med(lambda: pack_columns_device(hc, plan.bstart, plan.bcount, plan.n_p, plan.tau,
                                                               plan.e_out))
    out["pack_plan_ms"], batch = med(lambda: pack_plan(plan, 64, workers=w, device=True))
    out["execute_host_ms"], so = med(lambda: execute_batch_host(batch, cfg, "regular", workers=w, confirm=False))
    out["execute_host_confirm_ms"], so = med(lambda: execute_batch_host(batch, cfg, "regular", workers=w))
    out["device_ms"] = so.stats.rows[0].wall_ms
    out["run_range_ms"], rr = med(lambda: run_range("exp", 0, 0, count, cfg, interval_args=count, workers=w))
    out["records_equal"] = rr.records == so.records
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
