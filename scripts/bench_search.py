"""Config 2 (BASELINE.json configs[1]): exp binary64, one binade slice of
2^32 arguments = 2^17 linearised degree-1 problems of N = 2^15 (the
reference's linear_problem_batch, divergence.py:32-93), search only:
classic Lefevre loop vs the regular-control-flow variant on one B200.
Per algorithm: device time (CUDA events, R launches), arguments/s, quotient
steps/s, iteration statistics and warp divergence (NMDM over warps of 32
consecutive problems, divergence.py:96-110); the oracle port of the same
cores on the host threads beside it.  Prints one JSON line."""
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
    ap.add_argument("--log2-problems", type=int, default=17)
    ap.add_argument("--log2-N", type=int, default=15)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--verdicts", action="store_true", help="also time the lockstep form (hrb_search_verdicts)")
    a = ap.parse_args()
    import torch

    from paper_1211_3056_b200 import _native as nat
    from paper_1211_3056_b200.divergence import linear_problem_batch, problem_arrays, warp_summary
    from paper_1211_3056_b200.fpformat import FpFormat

    t0 = time.perf_counter()
    probs = linear_problem_batch("exp", FpFormat(53, 32), 0, 1 << a.log2_N, 1 << a.log2_problems,
                                 workers=os.cpu_count() or 1)
    gen_s = time.perf_counter() - t0
    A, B, E, N, W = problem_arrays(probs)
    n = len(A)
    args_total = int(N.astype(np.int64).sum())
    dev = torch.device("cuda")
    ins = [torch.from_numpy(x.view(np.int64)).to(dev) for x in (A, B, E, N)]
    ok = torch.empty(n, dtype=torch.uint8, device=dev)
    d, it, pl = (torch.empty(n, dtype=torch.int64, device=dev) for _ in range(3))
    ph = torch.empty(n, dtype=torch.uint8, device=dev)
    lib = nat.load()
    out = {"config": f"exp p=53 binade [1,2) 2^{a.log2_problems} problems x N=2^{a.log2_N} "
                     f"(= 2^{a.log2_problems + a.log2_N} args), eps=2^-31, W=64", "problem_gen_s": gen_s, "algos": {}}
    import oracle

    for name, code, mode in (("lefevre", 0, 1), ("lefevre_swap", 1, 1), ("regular", 2, 1), ("regular_unrolled", 3, 1)):
        def launch():
            nat.check("hrb_search_batch", lib.hrb_search_batch(code, mode, 64, n, *(x.data_ptr() for x in ins),
                                                               ok.data_ptr(), d.data_ptr(), it.data_ptr(),
                                                               pl.data_ptr(), ph.data_ptr(), nat.stream_ptr()))
        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            launch()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        iters = it.cpu().numpy().view(np.uint64)
        ws = warp_summary(iters)
        rec = {"kernel_ms": ms, "args_per_s": args_total / (ms / 1e3), "searches_per_s": n / (ms / 1e3),
               "quotient_steps_per_s": float(iters.sum()) / (ms / 1e3), "it_min": int(iters.min()),
               "it_max": int(iters.max()), "it_mean": float(iters.mean()), "mean_nmdm": ws.mean_nmdm,
               "warps_spread_le2": ws.spread_ok_fraction(2), "fail_rate": float(1 - ok.float().mean())}
        if not a.no_cpu:
            oracle.build()
            t = time.perf_counter()
            wok, wd, wit, _, _ = oracle.search_batch(name, mode, 1 << 64, A, B, E, N)
            cs = time.perf_counter() - t
            rec["cpu_port_args_per_s"] = args_total / cs
            rec["cpu_threads"] = oracle.threads()
            rec["bit_exact_vs_oracle"] = bool(np.array_equal(wit, iters) and np.array_equal(wd, d.cpu().numpy().view(np.uint64))
                                              and np.array_equal(wok, ok.cpu().numpy()))
        out["algos"][name] = rec
    if a.verdicts:  # the phases' lockstep form of the regular family (verdict, d, iterations only)
        for name, code in (("regular_lockstep", 2), ("regular_unrolled_lockstep", 3)):
            def launch_v():
                nat.check("hrb_search_verdicts", lib.hrb_search_verdicts(code, 64, n, *(x.data_ptr() for x in ins),
                                                                         ok.data_ptr(), d.data_ptr(), it.data_ptr(),
                                                                         nat.stream_ptr()))
            for _ in range(3):
                launch_v()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                launch_v()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            iters = it.cpu().numpy().view(np.uint64)
            rec = {"kernel_ms": ms, "args_per_s": args_total / (ms / 1e3),
                   "quotient_steps_per_s": float(iters.sum()) / (ms / 1e3),
                   "it_mean": float(iters.mean()), "mean_nmdm": warp_summary(iters).mean_nmdm}
            if not a.no_cpu:  # (verdict, d, iterations) against the oracle, as for the general forms
                base = "regular" if code == 2 else "regular_unrolled"
                wok, wd, wit, _, _ = oracle.search_batch(base, 1, 1 << 64, A, B, E, N)
                rec["bit_exact_vs_oracle"] = bool(np.array_equal(wit, iters)
                                                  and np.array_equal(wd, d.cpu().numpy().view(np.uint64))
                                                  and np.array_equal(wok, ok.cpu().numpy()))
            out["algos"][name] = rec
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
