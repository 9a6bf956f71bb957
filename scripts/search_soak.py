"""Search-core parity soak on the GPU (not part of the test suite): batches
of random and adversarial (a, b, eps, N) problems through the lockstep form
(hrb_search_verdicts, regular and unrolled) and the general cores
(hrb_search_batch, all four algorithms), compared with the oracle port of
the reference cores.  Prints one JSON summary.

    python scripts/search_soak.py --minutes 10 > gpurun_out/search_soak.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

ONE = 1 << 64


def adversarial(rng, n):
    """Vectorised form of tests/test_gpu_parity.py's _adversarial_problems:
    slopes near p/q with small q, tiny slopes, slopes near 1 and 2^63, near
    2^64/k; counts at the 32-bit edge."""
    kind = rng.integers(0, 8, n)
    a = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    q = rng.integers(2, 5000, n)
    p = (rng.random(n) * (q - 1)).astype(np.int64) + 1
    near = np.array([(ONE * int(pp) // int(qq)) % ONE for pp, qq in zip(p, q)], dtype=object)
    jit = rng.integers(-3, 4, n)
    k3 = rng.integers(2, 1 << 16, n)
    for i in np.nonzero(kind == 0)[0]:
        a[i] = np.uint64((near[i] + int(jit[i])) % ONE)
    a[kind == 1] = rng.integers(1, 1 << 20, int((kind == 1).sum()), dtype=np.uint64)
    a[kind == 2] = (np.uint64(0) - rng.integers(1, 1 << 20, int((kind == 2).sum()), dtype=np.uint64))
    for i in np.nonzero(kind == 3)[0]:
        a[i] = np.uint64((ONE // int(k3[i]) + int(jit[i]) % 5 - 2) % ONE)
    m4 = kind == 4
    a[m4] = (np.uint64(1 << 63) + rng.integers(0, 1 << 11, int(m4.sum()), dtype=np.uint64) - np.uint64(1 << 10))
    b = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    e = rng.integers(1, 1 << 40, n, dtype=np.uint64)
    Ns = np.array([1, 2, 3, 1 << 12, 1 << 15, (1 << 32) - 1, 1 << 32, (1 << 32) + 7], dtype=np.uint64)
    N = Ns[rng.integers(0, 8, n)]
    return a, b, e, N


def uniform(rng, n):
    a = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    b = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    e = np.uint64(1) << rng.integers(8, 50, n).astype(np.uint64)
    N = rng.integers(2, 1 << 16, n).astype(np.uint64)
    return a, b, e, N


def main():
    from paper_1211_3056_b200.device import search_batch_arrays, search_verdict_arrays

    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=10.0)
    ap.add_argument("--batch", type=int, default=1 << 20)
    ap.add_argument("--seed", type=int, default=20261017)
    a_ = ap.parse_args()
    oracle.build()
    rng = np.random.default_rng(a_.seed)
    t0 = time.time()
    stats = {"lockstep_problems": 0, "general_problems": 0, "mismatches": 0, "batches": 0}
    bad = []
    r = 0
    while time.time() - t0 < 60 * a_.minutes:
        gen = adversarial if r % 2 else uniform
        a, b, e, N = gen(rng, a_.batch)
        for name, code in (("regular", 2), ("regular_unrolled", 3)):
            ok, d, it = search_verdict_arrays(code, 64, a, b, e, N)
            wok, wd, wit, _, _ = oracle.search_batch(name, 1, ONE, a, b, e, N)
            m = (ok != wok) | (d != wd) | (it != wit)
            stats["lockstep_problems"] += len(a)
            if m.any():
                stats["mismatches"] += int(m.sum())
                bad.append({"form": "lockstep", "algo": name, "first": int(np.nonzero(m)[0][0])})
        if r % 4 == 0:  # the general cores (slower on the CPU side): a quarter of the batches
            for name, code, mode in (("lefevre", 0, 1), ("lefevre_swap", 1, 2), ("regular", 2, 1),
                                     ("regular_unrolled", 3, 1)):
                k = len(a) // 4
                ok, d, it, pl, ph = search_batch_arrays(code, mode, 64, a[:k], b[:k], e[:k], N[:k])
                wok, wd, wit, wpl, wph = oracle.search_batch(name, mode, ONE, a[:k], b[:k], e[:k], N[:k])
                m = (ok != wok) | (d != wd) | (it != wit) | (pl != wpl) | (ph.astype(np.uint64) != wph)
                stats["general_problems"] += k
                if m.any():
                    stats["mismatches"] += int(m.sum())
                    bad.append({"form": "general", "algo": name, "first": int(np.nonzero(m)[0][0])})
        stats["batches"] += 1
        r += 1
    stats["seconds"] = round(time.time() - t0, 1)
    stats["failures"] = bad[:20]
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
