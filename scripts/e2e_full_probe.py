"""Where run_range's end-to-end time goes over a 2^40-argument range
(BASELINE configs[2]): planning, native host generation + packing, device
phases, host bookkeeping, confirmation.  One GPU.

    python scripts/e2e_full_probe.py [--log2-args 40] [--interval 38]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-args", type=int, default=40)
    ap.add_argument("--interval", type=int, default=38)
    ap.add_argument("--eps-bits", type=int, default=32)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    import torch

    from paper_1211_3056_b200 import FpFormat, PhaseConfig, PipelineConfig, PolyGenConfig
    from paper_1211_3056_b200.funnel import execute_batch, run_range
    from paper_1211_3056_b200.slices import pack_plan, plan_arrays

    pg = PolyGenConfig(tau=512, N=1 << 15, mu=16, nu=32, delta=2, limbs=8, frac_bits=96, guard=32)
    cfg = PipelineConfig("exp", FpFormat(53, a.eps_bits), pg, PhaseConfig("regular", phase2_split=8, N1=1 << 15))
    count = 1 << a.log2_args
    out = {"workers": a.workers, "cpus": os.cpu_count()}
    t = time.perf_counter()
    plan = plan_arrays("exp", 0, cfg.fmt, pg, 0, count)
    out["plan_s"] = time.perf_counter() - t
    for w in sorted({1, a.workers}):
        t = time.perf_counter()
        batch = pack_plan(plan, 64, workers=w)
        out[f"pack_s_w{w}"] = time.perf_counter() - t
    t = time.perf_counter()
    so = execute_batch(batch, cfg, "regular", workers=a.workers)
    torch.cuda.synchronize()
    out["execute_batch_s"] = time.perf_counter() - t
    t = time.perf_counter()
    so = execute_batch(batch, cfg, "regular", workers=a.workers)
    torch.cuda.synchronize()
    out["execute_batch_s_2nd"] = time.perf_counter() - t
    out["phase_rows"] = [[r.phase, r.domains_in, r.domains_out, r.wall_ms] for r in so.stats.rows]
    for k in range(2):
        t = time.perf_counter()
        rr = run_range("exp", 0, 0, count, cfg, interval_args=1 << a.interval, workers=a.workers)
        torch.cuda.synchronize()
        out[f"run_range_s_{k}"] = time.perf_counter() - t
    out["records"] = len(rr.records)
    out["records_equal_single_slice"] = rr.records == so.records
    out["args_per_s"] = count / out["run_range_s_1"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
