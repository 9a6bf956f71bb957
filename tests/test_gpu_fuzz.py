"""Randomised parity sweep (fixed seeds): random function, binade, slice,
eps, domain size, super-domain shape, grid width F, word width W, split and
algorithm; the fused device funnel must equal the CPU oracle (itself pinned to
the reference by tests/golden) on failing ids, surviving subdomains and
candidates.  Configurations the reference itself would reject (error budget,
pad range) are skipped exactly as the host checks reject them."""

import os
import random

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

FUNCS = {"exp": (-3, 5), "log": (0, 6), "exp2": (-3, 5)}


def _config(rng):
    from paper_1211_3056_b200 import FpFormat, PhaseConfig, PipelineConfig, PolyGenConfig

    fn = rng.choice(sorted(FUNCS))
    binade = rng.randint(*FUNCS[fn])
    N = 1 << rng.randint(10, 15)
    tau = 1 << rng.randint(2, 9)
    mu = 1 << rng.randint(0, (tau.bit_length() - 1))
    split = rng.choice([2, 4, 8, 16])
    F = rng.choice([64, 96, 112, 128])
    W = rng.choice([64, 64, 64, 32])
    algo = rng.choice(["regular", "regular", "lefevre"])
    eps_bits = rng.randint(12, 36)
    pg = PolyGenConfig(tau=tau, N=N, mu=mu, nu=tau // mu, delta=2, limbs=8, frac_bits=F, guard=32)
    cfg = PipelineConfig(fn, FpFormat(53, eps_bits), pg, PhaseConfig(algo, phase2_split=split, N1=N), word_bits=W)
    count = 1 << rng.randint(20, 26)
    start = rng.randrange(0, (1 << 52) - count)
    return fn, binade, start, count, cfg, algo, split


@pytest.mark.parametrize("seed", list(range(24)))
def test_random_configuration_equals_oracle(seed):
    from paper_1211_3056_b200.device import DeviceSlice, FusedRunner
    from paper_1211_3056_b200.funnel import prepare_slice

    rng = random.Random(1000 + seed)
    fn, binade, start, count, cfg, algo, split = _config(rng)
    try:
        batch = prepare_slice(fn, binade, start, count, cfg, workers=min(8, os.cpu_count() or 1))
    except (ValueError, OverflowError) as exc:  # the reference raises here too (budget / pad / MPInt)
        pytest.skip(f"rejected on the host like the reference: {exc}")
    code = {"regular": 2, "lefevre": 0}[algo]
    fr = FusedRunner(DeviceSlice(batch), code, 1, split, sub_cap=batch.n_total * 2 * split + 1024,
                     cand_cap=1 << 22)
    fr.launch()
    r = fr.result()
    fails = oracle.phase1(batch, algo, 1)
    assert np.array_equal(r.fail_ids + np.uint64(batch.id0), fails), (fn, binade, start, count)
    rows = oracle.phase2(batch, algo, 1, split, fails)
    assert np.array_equal((r.sub_keys >> np.uint64(8)) + np.uint64(batch.id0), rows[0])
    assert np.array_equal(r.sub_keys & np.uint64(255), rows[1].astype(np.uint64))
    m, dist, dom = oracle.phase3(batch, rows)
    assert np.array_equal(r.cand_index, m) and np.array_equal(r.cand_dist, dist)
    assert np.array_equal(r.cand_dom + np.uint64(batch.id0), dom)
