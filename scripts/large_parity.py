"""Full-size parity (not part of the test suite): 2^40-argument slices of
several functions, starts, ε and both search families through the fused
device call (hrb_run_slice) and the host-buffer call, each compared with the
CPU oracle on every output -- failing ids, surviving (domain, j) rows and
candidates (argument, distance, domain).  Prints one JSON line per slice.

    python scripts/large_parity.py > gpurun_out/large_parity.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle  # noqa: E402

CASES = [  # (fn, start, log2 args, eps bits, algo)
    ("exp", 0, 40, 32, "regular"),
    ("exp", 1 << 51, 40, 32, "regular"),
    ("exp", 0x123456789AB0, 40, 24, "regular"),
    ("log", 0x6A09E667F3BCD, 40, 32, "regular"),
    ("exp2", 0x10000000000, 40, 32, "regular"),
    ("exp", 0, 38, 32, "lefevre"),
    ("log", 0x6A09E667F3BCD, 38, 28, "lefevre"),
]


def run(fn, start, log2, eps, algo):
    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner, run_host

    argv, sys.argv = sys.argv, ["bench.py", "--fn", fn, "--start", str(start), "--log2-args", str(log2), "--eps-bits", str(eps),
                "--algo", algo]
    args = bench.parse()
    sys.argv = argv
    t0 = time.time()
    batch, _ = bench.prepare_rank(args, 0, 1, os.cpu_count() or 1)
    code = {"regular": 2, "lefevre": 0}[algo]
    ds = DeviceSlice(batch)
    fr = FusedRunner(ds, code, 1, 8, sub_cap=batch.n_total // 4 + 4096, cand_cap=1 << 22)
    while True:  # size the outputs from the true counts, as bench.py does
        fr.launch()
        torch.cuda.synchronize()
        c = fr.counts_host()
        if c[1] <= fr.sub_cap and c[2] <= fr.cand_cap:
            break
        fr = FusedRunner(ds, code, 1, 8, sub_cap=max(fr.sub_cap, int(c[1]) + 1024),
                         cand_cap=max(fr.cand_cap, int(c[2]) + 1024))
    r = fr.result()
    fails = oracle.phase1(batch, algo, 1)
    rows = oracle.phase2(batch, algo, 1, 8, fails)
    m, dist, dom = oracle.phase3(batch, rows)
    dev_ok = (np.array_equal(r.fail_ids + np.uint64(batch.id0), fails)
              and np.array_equal((r.sub_keys >> np.uint64(8)) + np.uint64(batch.id0), rows[0])
              and np.array_equal(r.sub_keys & np.uint64(255), rows[1].astype(np.uint64))
              and np.array_equal(r.cand_index, m) and np.array_equal(r.cand_dist, dist)
              and np.array_equal(r.cand_dom + np.uint64(batch.id0), dom))
    counts, hf, hm, hd, hdom, _ = run_host(batch, code, 1, 8, cand_cap=max(1 << 20, len(m) + 1024))
    host_ok = (np.array_equal(hf, r.fail_ids) and np.array_equal(hm, r.cand_index)
               and np.array_equal(hd, r.cand_dist) and np.array_equal(hdom, r.cand_dom))
    return {"fn": fn, "start": hex(start), "args": f"2^{log2}", "eps": f"2^-{eps}", "algo": algo,
            "super_domains": int(batch.n_super), "domains": int(batch.n_total), "phase1_fails": int(len(fails)),
            "survivors": int(len(rows[0])), "candidates": int(len(m)), "device_equals_oracle": bool(dev_ok),
            "host_equals_device": bool(host_ok), "seconds": round(time.time() - t0, 1)}


def main():
    import random

    ap = argparse.ArgumentParser()
    ap.add_argument("--random", type=int, default=0, help="also run this many random 2^40 slices")
    ap.add_argument("--minutes", type=float, default=20.0)
    ap.add_argument("--seed", type=int, default=20261017)
    ap.add_argument("--no-fixed", action="store_true", help="skip the fixed CASES")
    a = ap.parse_args()
    oracle.build()
    oracle.set_threads(os.cpu_count() or 1)
    cases = [] if a.no_fixed else list(CASES)
    rng = random.Random(a.seed)
    for _ in range(a.random):
        fn = rng.choice(["exp", "log", "exp2"])
        cases.append((fn, rng.randrange(0, (1 << 52) - (1 << 40)), 40, rng.randint(24 if fn == "log" else 20, 36),
                      "regular" if rng.random() < 0.8 else "lefevre"))
    t0 = time.time()
    for c in cases:
        if time.time() - t0 > 60 * a.minutes:
            break
        try:
            print(json.dumps(run(*c)), flush=True)
        except (ValueError, OverflowError) as exc:  # rejected on the host, as the reference would
            print(json.dumps({"fn": c[0], "start": hex(c[1]), "status": "rejected", "why": str(exc)[:100]}), flush=True)


if __name__ == "__main__":
    main()
