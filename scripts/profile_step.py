"""One hrb_run_slice of the bench workload plus the INT-peak probe, for ncu
(launch lists and metric captures).  Not a bench: prints no timing."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-args", type=int, default=40)
    ap.add_argument("--eps-bits", type=int, default=32)
    ap.add_argument("--algo", default="regular")
    ap.add_argument("--fn", default="exp")
    ap.add_argument("--start", type=lambda x: int(x, 0), default=0)
    ap.add_argument("--launches", type=int, default=1)
    ap.add_argument("--no-peak", action="store_true")
    ap.add_argument("--cand-cap", type=int, default=1 << 20)
    a = ap.parse_args()
    ns = argparse.Namespace(log2_args=a.log2_args, eps_bits=a.eps_bits, algo=a.algo, log2_super=24, log2_N=15,
                            fn=a.fn, start=a.start)
    import torch

    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner

    batch, _ = bench.prepare_rank(ns, 0, 1, os.cpu_count() or 1)
    ds = DeviceSlice(batch)
    r = FusedRunner(ds, 2 if a.algo == "regular" else 0, 1, 8, sub_cap=batch.n_total * 2, cand_cap=a.cand_cap)
    for _ in range(a.launches):
        r.launch()
    torch.cuda.synchronize()
    print("counts", r.counts_host().tolist())
    if not a.no_peak:
        print("int_peak", bench.int_peak())


if __name__ == "__main__":
    main()
