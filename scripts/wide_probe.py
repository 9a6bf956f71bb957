"""High-degree path at full size: host model time, device step (inputs
resident), host-buffer call, confirmation, and the records against the
delta = 2 pipeline over the same range.  One GPU.

    python scripts/wide_probe.py --log2-args 40 --deltas 4,5,6 [--check]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-args", type=int, default=40)
    ap.add_argument("--start", type=lambda x: int(x, 0), default=0)
    ap.add_argument("--eps-bits", type=int, default=32)
    ap.add_argument("--deltas", default="4,5,6")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--check", action="store_true", help="compare records with the delta = 2 pipeline")
    a = ap.parse_args()
    import torch

    from paper_1211_3056_b200 import FpFormat, PhaseConfig, PipelineConfig, PolyGenConfig
    from paper_1211_3056_b200.funnel import confirm_candidates, run_range
    from paper_1211_3056_b200.wide import (WideDeviceSlice, WideGenConfig, WideRunner, candidates_of, prepare_wide,
                                           run_wide_host)

    fmt = FpFormat(53, a.eps_bits)
    count = 1 << a.log2_args
    workers = os.cpu_count() or 1
    want = None
    if a.check:
        pg = PolyGenConfig(tau=512, N=1 << 15, mu=16, nu=32, delta=2, limbs=8, frac_bits=96, guard=32)
        cfg = PipelineConfig("exp", fmt, pg, PhaseConfig("regular", phase2_split=8, N1=1 << 15))
        t = time.perf_counter()
        want = run_range("exp", 0, a.start, count, cfg, interval_args=1 << 38, workers=workers).records
        print(json.dumps({"delta": 2, "records": len(want), "run_range_s": time.perf_counter() - t}), flush=True)
    for d in [int(x) for x in a.deltas.split(",")]:
        w = WideGenConfig.for_degree(d)
        out = {"delta": d, "super_args_log2": int(np.log2(w.tau * w.N)), "F": w.frac_bits}
        t = time.perf_counter()
        batch = prepare_wide("exp", 0, a.start, count, fmt, w, workers=workers)
        out["host_model_s"] = time.perf_counter() - t
        out["super_domains"] = batch.n_super
        ds = WideDeviceSlice(batch)
        runner = WideRunner(ds, 2, 8, sub_cap=max(1 << 16, batch.n_total // 4), cand_cap=1 << 20)
        runner.launch()
        torch.cuda.synchronize()
        c0 = runner.counts_host().copy()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        stream = torch.cuda.current_stream()
        ms = []
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            runner.launch()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        assert np.array_equal(runner.counts_host(), c0)
        out["device_ms"] = float(np.median(ms))
        out["device_args_per_s"] = count / (out["device_ms"] / 1e3)
        out["counts"] = [int(x) for x in c0[:4]]
        res = run_wide_host(batch, cand_cap=1 << 20)
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            res = run_wide_host(batch, cand_cap=1 << 20)
            ts.append(time.perf_counter() - t)
        out["e2e_ms"] = 1e3 * float(np.median(ts))
        tf = []
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            b2 = prepare_wide("exp", 0, a.start, count, fmt, w, workers=workers)
            r2 = run_wide_host(b2, cand_cap=1 << 20)
            recs = confirm_candidates("exp", candidates_of(b2, r2), fmt, workers)
            tf.append(time.perf_counter() - t)
        out["e2e_full_s"] = float(np.median(tf))
        out["e2e_full_args_per_s"] = count / out["e2e_full_s"]
        out["records"] = len(recs)
        if want is not None:
            out["records_equal_delta2"] = [(r.argument, r.distance.raw, r.domain_id) for r in recs] == \
                [(r.argument, r.distance.raw, r.domain_id) for r in want]
        print(json.dumps(out), flush=True)
        del ds, runner, flush
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
