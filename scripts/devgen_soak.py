"""Device generation soak (not part of the test suite): random planned
slices (precision, eps, binade, N, tau, delta, limbs, F, guard, word size)
through hrb_pack_blocks and through the host library (itself soaked against
the mpmath path, scripts/hostgen_soak.py); every column and every fallback
flag must agree.  One JSON summary line.

    python scripts/devgen_soak.py --minutes 15 --seed 1 > gpurun_out/devgen_soak.json
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


def random_plan(rng):
    from paper_1211_3056_b200 import slices
    from paper_1211_3056_b200.fpformat import FpFormat
    from paper_1211_3056_b200.taylor import PolyGenConfig

    p = rng.choice([11, 16, 24, 32, 40, 53, 53, 53, 64])
    fmt = FpFormat(p, rng.randint(6, min(60, 2 * p)))
    N = 1 << rng.randint(2, 16)
    tau = 1 << rng.randint(0, 10)
    mu = 1 << rng.randint(0, tau.bit_length() - 1)
    F = rng.choice([40, 48, 64, 80, 96, 96, 112, 128, 160, 192])
    W = rng.choice([32, 64]) if F >= 64 else 32
    guard = rng.choice([0, 8, 16, 32, 32, 64])
    pg = PolyGenConfig(tau=tau, N=N, mu=mu, nu=tau // mu, delta=rng.choice([1, 2, 2]), limbs=rng.randint(1, 12),
                       frac_bits=F, guard=guard)
    binade = rng.choice([0, 0, 0, -1, -2, -9, -40, -200])
    span = 1 << (p - 1)
    count = min(span, rng.randint(1, 1 << 14) * N * tau // rng.choice([1, 2, 5]))
    start = rng.randrange(0, span - count + 1)
    return slices.plan_arrays("exp", binade, fmt, pg, start, count), fmt, pg, binade, W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=10.0)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    from paper_1211_3056_b200 import hostgen
    from paper_1211_3056_b200.device import pack_columns_device

    rng = random.Random(a.seed)
    t_end = time.time() + 60 * a.minutes
    n_cfg = n_super = n_ok = n_fb = 0
    failures = []
    while time.time() < t_end:
        plan, fmt, pg, binade, W = random_plan(rng)
        if not len(plan) or pg.limbs > 12 or pg.frac_bits + pg.guard > 224:
            continue
        cfg = hostgen.make_cfg("exp", fmt, pg, binade, W)
        cols = (plan.bstart, plan.bcount, plan.n_p, plan.tau, plan.e_out)
        host = hostgen.pack_columns(cfg, *cols, 0)
        dev = pack_columns_device(cfg, *cols)
        ok = host[3] == hostgen.HRBH_OK
        same = np.array_equal(host[3], dev[3]) and all(
            np.array_equal(h[..., ok], d[..., ok]) for h, d in zip((host[0], host[1], host[2], host[4]),
                                                                (dev[0], dev[1], dev[2], dev[4])))
        n_cfg += 1
        n_super += len(plan)
        n_ok += int(ok.sum())
        n_fb += int((~ok).sum())
        if not same:
            failures.append({"p": fmt.precision, "eps": fmt.eps_bits, "binade": binade, "N": pg.N, "tau": pg.tau,
                             "delta": pg.delta, "limbs": pg.limbs, "F": pg.frac_bits, "guard": pg.guard, "W": W,
                             "start": int(plan.bstart[0])})
    print(json.dumps({"configurations": n_cfg, "super_domains": n_super, "generated": n_ok, "flagged": n_fb,
                      "mismatches": len(failures), "failures": failures[:10], "minutes": a.minutes,
                      "seed": a.seed}))


if __name__ == "__main__":
    main()
