"""Long randomised parity soak on the GPU (not part of the test suite): the
tests/test_gpu_fuzz.py configuration generator over many more seeds, each
configuration through both the fused device call (hrb_run_slice) and the
host-buffer call (hrb_run_slice_host, streamed upload), compared with the
CPU oracle (pinned to the reference by tests/golden).  Writes one JSON
summary.

    python scripts/fuzz_soak.py --seeds 2000:2300 --minutes 20 > gpurun_out/fuzz_soak.json
"""
import argparse
import json
import os
import random
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from test_gpu_fuzz import _config  # noqa: E402


def check(seed):
    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner, run_host
    from paper_1211_3056_b200.funnel import prepare_slice

    rng = random.Random(seed)
    fn, binade, start, count, cfg, algo, split = _config(rng)
    desc = {"seed": seed, "fn": fn, "binade": binade, "start": start, "count": count, "algo": algo, "split": split,
            "F": cfg.polygen.frac_bits, "W": cfg.word_bits, "N": cfg.polygen.N, "tau": cfg.polygen.tau,
            "eps_bits": cfg.fmt.eps_bits}
    try:
        batch = prepare_slice(fn, binade, start, count, cfg, workers=min(8, os.cpu_count() or 1))
    except (ValueError, OverflowError) as exc:
        return dict(desc, status="rejected", why=str(exc)[:120])
    code = {"regular": 2, "lefevre": 0}[algo]
    fr = FusedRunner(DeviceSlice(batch), code, 1, split, sub_cap=batch.n_total * 2 * split + 1024, cand_cap=1 << 22)
    fr.launch()
    r = fr.result()
    fails = oracle.phase1(batch, algo, 1)
    rows = oracle.phase2(batch, algo, 1, split, fails)
    m, dist, dom = oracle.phase3(batch, rows)
    ok = (np.array_equal(r.fail_ids + np.uint64(batch.id0), fails)
          and np.array_equal((r.sub_keys >> np.uint64(8)) + np.uint64(batch.id0), rows[0])
          and np.array_equal(r.sub_keys & np.uint64(255), rows[1].astype(np.uint64))
          and np.array_equal(r.cand_index, m) and np.array_equal(r.cand_dist, dist)
          and np.array_equal(r.cand_dom + np.uint64(batch.id0), dom))
    counts, hf, hm, hd, hdom, _ = run_host(batch, code, 1, split, cand_cap=1 << 22)
    ok_host = (np.array_equal(hf, r.fail_ids) and np.array_equal(hm, r.cand_index)
               and np.array_equal(hd, r.cand_dist) and np.array_equal(hdom, r.cand_dom))
    return dict(desc, status="pass" if ok and ok_host else "FAIL", device_equals_oracle=bool(ok),
                host_equals_device=bool(ok_host), n_super=int(batch.n_super), fails=int(len(fails)),
                survivors=int(len(rows[0])), candidates=int(len(m)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", default="2000:2300")
    ap.add_argument("--minutes", type=float, default=20.0)
    a = ap.parse_args()
    lo, hi = (int(x) for x in a.seeds.split(":"))
    oracle.build()
    t0 = time.time()
    results = []
    for seed in range(lo, hi):
        if time.time() - t0 > 60 * a.minutes:
            break
        try:
            results.append(check(seed))
        except Exception as exc:  # an error is a failure of the run, recorded with its traceback tail
            results.append({"seed": seed, "status": "ERROR", "why": traceback.format_exc()[-400:]})
        print(json.dumps(results[-1]), file=sys.stderr, flush=True)
    summary = {k: sum(1 for r in results if r["status"] == k) for k in ("pass", "rejected", "FAIL", "ERROR")}
    summary.update({"seeds": [lo, lo + len(results)], "seconds": round(time.time() - t0, 1),
                    "algos": {k: sum(1 for r in results if r.get("algo") == k and r["status"] == "pass")
                              for k in ("regular", "lefevre")},
                    "F": sorted({r["F"] for r in results if r["status"] == "pass"}),
                    "W": sorted({r["W"] for r in results if r["status"] == "pass"}),
                    "failures": [r for r in results if r["status"] in ("FAIL", "ERROR")]})
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
