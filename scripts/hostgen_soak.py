"""Soak: the native host generator (libhrbhost.so) against the exact Python
path (mpmath Taylor models + Fraction checks) on random configurations,
super-domain by super-domain, and the native confirmation against
decide_hr.  CPU only.

    python scripts/hostgen_soak.py --supers 1000000 --out profiles/r02/hostgen_soak.json
"""
import argparse
import json
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1211_3056_b200 import hostgen, slices  # noqa: E402
from paper_1211_3056_b200.fpformat import FpFormat  # noqa: E402
from paper_1211_3056_b200.taylor import PolyGenConfig  # noqa: E402

PACKED = ("coef", "G", "s2abs", "n_dom", "dom_n", "last_n", "dom_base", "m0", "shift_bound_ok")


def one(rng, max_supers):
    p = rng.choice([53, 53, 53, 40, 24])
    binade = rng.choice([0, 0, 0, -1, -3])
    fmt = FpFormat(p, rng.choice([16, 20, 24, 32, 40]))
    lgN = rng.choice([6, 8, 10, 12, 15]) if p > 24 else rng.choice([4, 6, 8])
    mu = 1 << rng.choice([0, 1, 2, 3])
    nu = 1 << rng.choice([1, 2, 3, 4, 5])
    pg = PolyGenConfig(tau=mu * nu, N=1 << lgN, mu=mu, nu=nu, delta=rng.choice([1, 2, 2]),
                       limbs=rng.choice([5, 6, 8, 8]), frac_bits=rng.choice([64, 80, 96, 96, 128]),
                       guard=rng.choice([0, 16, 32]))
    block = pg.tau * pg.N
    n_blocks = rng.randrange(1, max_supers + 1)
    total = 1 << (p - 1)
    count = min(n_blocks * block + rng.randrange(0, block), total)
    start = rng.randrange(0, total - count + 1)
    plan = slices.plan_arrays("exp", binade, fmt, pg, start, count)
    try:
        want = slices.pack_plan(plan, 64, workers=1, native=False)
        err = None
    except (ValueError, ArithmeticError) as e:
        want, err = None, type(e).__name__
    try:
        got = slices.pack_plan(plan, 64, workers=4, native=True)
        gerr = None
    except (ValueError, ArithmeticError) as e:
        got, gerr = None, type(e).__name__
    if err or gerr:
        return len(plan), err == gerr, 0
    ok = all(np.array_equal(getattr(got, k), getattr(want, k)) for k in PACKED)
    cfg = hostgen.make_cfg("exp", fmt, pg, binade, 64)
    st = hostgen.pack_columns(cfg, plan.bstart, plan.bcount, plan.n_p, plan.tau, plan.e_out, 1)[3]
    return len(plan), ok, int((st == 0).sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--supers", type=int, default=100000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-per-config", type=int, default=4000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rng = random.Random(a.seed)
    t0 = time.time()
    total = native = configs = bad = 0
    while total < a.supers:
        n, ok, nat = one(rng, a.max_per_config)
        total += n
        native += nat
        configs += 1
        if not ok:
            bad += 1
            print(json.dumps({"mismatch_config": configs, "seed": a.seed}), flush=True)
        if configs % 20 == 0:
            print(f"{configs} configs, {total} super-domains ({native} native), {bad} mismatches, "
                  f"{time.time() - t0:.0f} s", flush=True)
    res = {"configs": configs, "super_domains": total, "native_super_domains": native, "mismatches": bad,
           "seed": a.seed, "seconds": time.time() - t0,
           "what": "slices.pack_plan native vs Python (mpmath) path: coef, G, s2abs, geometry, shift flags"}
    print(json.dumps(res))
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
